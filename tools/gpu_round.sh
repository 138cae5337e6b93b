#!/bin/bash
# One GPU session of the development loop: gpu tests, bench, per-level marginals.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/g_tests.log
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/g_bench.log 2>&1
timeout 300 python tools/tools_levels.py > gpurun_out/g_levels.log 2>&1
