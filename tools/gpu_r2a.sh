#!/bin/bash
# round-2 check: parity suites + C4 stage diagnostics (faithful fp32, host Omega)
nvidia-smi --query-gpu=name,clocks.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_factor.py -x -q 2>&1 | tail -15
timeout 900 python tools/diag_parity.py --config C4 --omega-host > gpurun_out/diag_C4f.log 2>&1; tail -c 1500 gpurun_out/diag_C4f.log
