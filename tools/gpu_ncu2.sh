#!/bin/bash
mkdir -p gpurun_out
python tools/tools_step.py > gpurun_out/plain2.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k "regex:k_f3_rec_plane" -s 9 -c 1 -o gpurun_out/recp9 python tools/tools_step.py > gpurun_out/ncu_recp9.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_f3_dec_plane" -s 5 -c 1 -o gpurun_out/decp9 python tools/tools_step.py > gpurun_out/ncu_decp9.log 2>&1
