#!/bin/bash
# Round profile bundle (GPU box): the ncu launch list of one eager step and
# ncu --set full captures of the level-9 kernels of the second step of
# tools/tools_step.py, after the plain run exits 0.  Launch order per step:
# dec_plane levels 9..5; rec_plane 5..9 (corrections forked coarse first);
# interp 5..9; row: 5 in decompose, 5 in recompose; col: 10 + 10.
mkdir -p gpurun_out
bash tools/tools_prof.sh
bash tools/tools_ncu_full.sh "k_f3_dec_plane" 5 decp "k_f3_rec_plane" 9 recp "k_f3_rec_interp" 9 interp \
  "k_f3_row" 10 row "k_f3_col" 20 col1 "k_quant_labels" 0 quant
python tools/tools_profiles.py gpurun_out/launches.csv r02 > gpurun_out/profiles_r02.log 2>&1
python tools/tools_ncu_summary.py gpurun_out/r02_ncu_full.md gpurun_out/decp.ncu-rep gpurun_out/recp.ncu-rep \
  gpurun_out/interp.ncu-rep gpurun_out/row.ncu-rep gpurun_out/col1.ncu-rep gpurun_out/quant.ncu-rep \
  > gpurun_out/summary_r02.log 2>&1
cp profiles/r02_launches.md profiles/traffic.json gpurun_out/ 2>/dev/null
rm -f gpurun_out/recp.ncu-rep gpurun_out/interp.ncu-rep gpurun_out/row.ncu-rep gpurun_out/col1.ncu-rep \
  gpurun_out/quant.ncu-rep
