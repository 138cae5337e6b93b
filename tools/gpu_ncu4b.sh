#!/bin/bash
mkdir -p gpurun_out
python tools/level_kernels.py config4b > gpurun_out/l4b.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k "regex:kN_coef_load0" -s 0 -c 1 -o gpurun_out/c04b python tools/level_kernels.py config4b > gpurun_out/ncu_c04b.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:kN_rec_interp" -s 0 -c 1 -o gpurun_out/ri4b python tools/level_kernels.py config4b > gpurun_out/ncu_ri4b.log 2>&1
