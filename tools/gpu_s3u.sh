#!/bin/bash
O=gpurun_out/s3u; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_shard.py -x -q > $O/pytest_shard.log 2>&1; tail -3 $O/pytest_shard.log
for c in C3 C4 C5; do
  timeout 600 python bench.py --config $c --shard --steps 3 --warmup 1 --no-cpu-baseline --no-e2e --no-scaling-config > $O/shard_$c.json 2> $O/shard_$c.err
  python -c "import json,sys; d=json.loads(open('$O/shard_$c.json').read().strip().splitlines()[-1]); print('$c sharded N=1', d['value'], d['iterations'], d['relerr'], 'stab_w', d['passes']['stab_w']['ms_per_step'])"
done
