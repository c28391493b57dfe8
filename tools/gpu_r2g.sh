#!/bin/bash
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 1200 2>&1 | tail -5
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_C2_g.json 2> gpurun_out/bench_C2_g.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_C2_g.json').read().strip().splitlines()[-1])
print(d['value'], d['roofline']['bound'], d['roofline']['frac'], d['roofline']['hbm']['frac'], d['lu_roofline']['frac'], d['parity']['pass'], d['scaling_config']['roofline']['bound'], d['scaling_config']['roofline']['frac'])"
tail -3 gpurun_out/bench_C2_g.err
