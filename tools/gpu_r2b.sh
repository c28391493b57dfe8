#!/bin/bash
# round-2: full-size oracle fixtures (C1-C5) + GPU parity on the same inputs, then the C2 bench line
mkdir -p gpurun_out/golden
timeout 2400 python tools/make_fixtures.py C1 C2 C3 C4 C5 --out gpurun_out/golden > gpurun_out/fixtures.log 2> gpurun_out/fixtures.err
tail -c 4000 gpurun_out/fixtures.log; tail -5 gpurun_out/fixtures.err
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err
tail -c 3000 gpurun_out/bench_C2.json; tail -3 gpurun_out/bench_C2.err
