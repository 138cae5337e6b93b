#!/bin/bash
# Profiling helper run on the GPU box: plain run, then the ncu launch list
# (per-launch duration + DRAM bytes) of the same command (profiles/r0N_launches.md).
set -x
CMD="python tools/tools_step.py"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
