#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_bound.py tests/test_gpu_bcd.py -q -x 2>&1 | tail -25
