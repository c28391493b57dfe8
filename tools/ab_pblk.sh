# A/B of the fp32 sketch panel feed (RCPG_TC_PBLK=0 direct, 1 blocked raw, 2 blocked hi|lo)
timeout 600 python -m pytest tests/test_gpu_passes.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_pblk.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_pblk.log
for c in C3 C5 C4; do for m in 0 1 2; do
  echo "== $c PBLK=$m" >> gpurun_out/ab_pblk.txt
  RCPG_TC_PBLK=$m timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); p=d['passes']
print(round(d['value'],2), d['roofline']['frac'], {k:(round(p[k]['ms_per_step'],3), round(p[k]['gbs'] or 0)) for k in ('omega','sketch','power_xtq','power_xz','project')})" >> gpurun_out/ab_pblk.txt 2>&1
done; done
