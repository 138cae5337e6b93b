#!/bin/bash
# Full GPU check: pytest -m gpu, smoke, bench (default args).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -s 2>&1 | grep -v "^\s*$" | tail -40 > gpurun_out/full_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/full_bench.log 2>&1
