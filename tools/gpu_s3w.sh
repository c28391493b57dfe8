#!/bin/bash
for i in 1 2; do
for c in C3 C2; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-scaling-config > /tmp/b.json 2>/dev/null
  python - /tmp/b.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
p = d["passes"]
print(d["config"]["workload"][:3], "%.3f ms" % d["value"], "frac %.3f" % d["roofline"]["frac"], " ".join("%s=%.3f" % (k, v["ms_per_step"]) for k, v in p.items() if k in ("sketch","power_xtq","power_xz","project")))
PY
done; done
