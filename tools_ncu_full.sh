#!/bin/bash
# One ncu --set full capture of the named kernels (run on the GPU box).
# usage: tools_ncu_full.sh <regex> <count> <outname>
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/plain_full.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k "regex:$1" -c "$2" -o "gpurun_out/$3" $CMD > "gpurun_out/ncu_$3.log" 2>&1
