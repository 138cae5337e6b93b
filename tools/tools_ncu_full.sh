#!/bin/bash
# ncu --set full capture of one kernel launch (run on the GPU box).
# usage: tools_ncu_full.sh <regex> <skip> <outname> [more regex skip outname ...]
CMD="python tools/tools_step.py"
$CMD > gpurun_out/plain_full.log 2>&1 || exit 1
while [ $# -ge 3 ]; do
  ncu --set full --clock-control none --import-source on -k "regex:$1" -s "$2" -c 1 -o "gpurun_out/$3" $CMD > "gpurun_out/ncu_$3.log" 2>&1
  shift 3
done
