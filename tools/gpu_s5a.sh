#!/bin/bash
# session 5: HEAD validation — full GPU tests, C2 bench + reference arm
O=gpurun_out/s5a; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
tail -5 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_C2.json 2> $O/bench_C2.err
timeout 900 python bench.py --impl reference > $O/bench_ref_C2.json 2> $O/bench_ref_C2.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/s5a/bench_C2.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e'], d['roofline']['frac'], d['parity']['pass'])
print({k:round(v['ms_per_step'],3) for k,v in d['passes'].items()})
PY
tail -c 600 $O/bench_ref_C2.json
