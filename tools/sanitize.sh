#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over tools/sanitize_run.py
# (run on the GPU box); summaries into gpurun_out/sanitize_<tool>.log
mkdir -p gpurun_out
export MGRX_FUSED_MIN_ELEMS=1
for t in memcheck racecheck synccheck initcheck; do
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $t --target-processes all --print-limit 20 \
    python tools/sanitize_run.py > gpurun_out/sanitize_$t.log 2>&1
  echo "$t rc=$?" >> gpurun_out/sanitize_$t.log
done
