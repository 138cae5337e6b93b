#!/bin/bash
# ncu --set full of the 4-D general-path kernels (config 4b), summarised on the box.
mkdir -p gpurun_out
python tools/level_kernels.py config4b > gpurun_out/l4b.log 2>&1 || exit 1
for k in ${KERNELS:-kN_coef_load0 kN_rec_interp}; do
  ncu --set full --clock-control none --import-source on -k "regex:$k" -s 0 -c 1 -o /tmp/n4b_$k python tools/level_kernels.py config4b > gpurun_out/ncu_$k.log 2>&1
done
python tools/tools_ncu_summary.py gpurun_out/ncu4b.md /tmp/n4b_*.ncu-rep
