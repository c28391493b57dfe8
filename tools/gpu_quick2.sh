#!/bin/bash
# tests + device time of every config (no CPU baseline / e2e / scaling records)
O=gpurun_out/${1:-q}; mkdir -p $O
if [ "${2:-tests}" = tests ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
  tail -2 $O/pytest_gpu.log
fi
for c in C2 C3 C5 C4 C1; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-scaling-config > $O/bench_$c.json 2> $O/bench_$c.err
  python - $O/bench_$c.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
p = d["passes"]
print(d["config"]["workload"][:3], "%.3f ms" % d["value"], "frac %.3f" % d["roofline"]["frac"], "iters", d["iterations"],
      " ".join("%s=%.3f" % (k, v["ms_per_step"]) for k, v in p.items()))
PY
done
