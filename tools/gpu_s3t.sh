#!/bin/bash
O=gpurun_out/s3t; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; tail -2 $O/pytest.log
timeout 600 python bench.py > $O/bench_C2.json 2> $O/bench_C2.err; tail -c 600 $O/bench_C2.json; echo
for c in C3 C5; do
  timeout 600 python bench.py --config $c --shard --steps 3 --warmup 1 --no-cpu-baseline --no-e2e --no-scaling-config > $O/shard_$c.json 2> $O/shard_$c.err
  python -c "import json,sys; d=json.loads(open('$O/shard_$c.json').read().strip().splitlines()[-1]); print('$c sharded N=1', d['value'], d['iterations'], d['relerr'], d['config']['parallelism'])"
done
