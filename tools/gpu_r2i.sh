#!/bin/bash
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_C2_i.json 2> gpurun_out/bench_C2_i.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_C2_i.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['parity']['pass'], d['gpu_launches'])
for k in ('scaling_config','scaling_config_C5'):
    s=d[k]; print(k, s['value'], s['roofline']['frac'], s['iterations'], s['parallelism'])"
tail -2 gpurun_out/bench_C2_i.err
