#!/bin/bash
# round-2 benches: C3-C5 (faithful fp32) and C2, device + e2e; per-pass breakdown
for c in C3 C4 C5; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-scaling-config > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1])
print('$c', round(d['value'],2), 'e2e', round(d['e2e']['value'],1), 'frac', round(d['roofline']['frac'],3), d['iterations'])
print({k: round(v['ms_per_step'],2) for k,v in d['passes'].items()})"
done
