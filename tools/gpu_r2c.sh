#!/bin/bash
# round-2: the whole -m gpu suite (incl. full-size fixtures, bitwise LU/QR/Omega, mode-0 sharding)
timeout 3000 python -m pytest tests -m gpu -q -x --timeout 1200 2>&1 | tail -25
