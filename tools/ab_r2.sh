#!/bin/bash
# A/B: big-LU occupancy (plu_coop minBlocks 1 vs 3), alternating
for lib in mb1 mb3 mb1 mb3; do
  RCPG_LIB=paper_1703_09074_b200/librcpg_$lib.so timeout 600 python bench.py --config C4 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e --no-scaling-config 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', round(d['value'],2), d['iterations'], {k: round(v['ms_per_step'],2) for k,v in d['passes'].items() if k in ('stab_w','thin_qr','omega','omega_overlapped','check_finite')})"
done
timeout 900 python bench.py --config C3 --steps 3 --warmup 1 --no-e2e --no-scaling-config 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C3', round(d['value'],2), d['iterations'], d['parity']['pass'], d['roofline']['frac'], {k: round(v['ms_per_step'],2) for k,v in d['passes'].items()})"
timeout 900 python bench.py --steps 5 --warmup 3 --no-scaling-config 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C2', round(d['value'],3), d['iterations'], d['parity']['pass'], d['roofline']['frac'], d['e2e']['value'], {k: round(v['ms_per_step'],3) for k,v in d['passes'].items()})"
