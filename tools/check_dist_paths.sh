O=gpurun_out/s5t; mkdir -p $O
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu-baseline > $O/torchrun_n1.json 2> $O/torchrun_n1.err; echo "torchrun rc=$?"
timeout 900 python bench.py --config C3 --shard --no-cpu-baseline --no-e2e --no-scaling-config --steps 2 > $O/c3_shard.json 2> $O/c3_shard.err; echo "c3 shard rc=$?"
timeout 900 python bench.py --config C5 --shard --no-cpu-baseline --no-e2e --no-scaling-config --steps 2 > $O/c5_shard.json 2> $O/c5_shard.err; echo "c5 shard rc=$?"
python - <<'PY'
import json
for f in ['torchrun_n1','c3_shard','c5_shard']:
    try:
        d=json.loads(open(f'gpurun_out/s5t/{f}.json').read().strip().splitlines()[-1])
        print(f, round(d['value'],3), d['config']['parallelism'], d['iterations'], round(d['relerr'],10), 'sc' , {k:(round(v.get('value',0),2) if isinstance(v,dict) and 'value' in v else v) for k,v in d.items() if k.startswith('scaling_config')})
    except Exception as e:
        print(f, 'ERR', e)
PY
for f in $O/*.err; do tail -n 3 $f; done
