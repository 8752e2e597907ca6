#!/bin/bash
# Development loop on the GPU box: parity tests, quick timings, marginal phase costs.
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -4
python scripts/quick_bench.py 26
python scripts/quick_bench.py 24
[ -n "$STOP" ] && MARKS=$STOP python scripts/stop_times.py 2>&1
true
