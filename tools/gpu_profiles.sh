#!/bin/bash
# Round profile bundle (GPU box): the ncu launch list of one eager step and
# ncu --set full captures of the level-9 kernels, after the plain run exits 0.
mkdir -p gpurun_out
bash tools/tools_prof.sh
bash tools/tools_ncu_full.sh "k_f3_dec_plane" 2 decp "k_f3_rec_plane" 2 recp "k_f3_rec_interp" 2 interp \
  "k_f3_row" 4 row "k_f3_col" 8 col1 "k_quant_labels" 0 quant
# summaries here (ncu is on the box), keep only the dominant kernel's report
python tools/tools_profiles.py gpurun_out/launches.csv r02 > gpurun_out/profiles_r02.log 2>&1
python tools/tools_ncu_summary.py gpurun_out/r02_ncu_full.md gpurun_out/decp.ncu-rep gpurun_out/recp.ncu-rep \
  gpurun_out/interp.ncu-rep gpurun_out/row.ncu-rep gpurun_out/col1.ncu-rep gpurun_out/quant.ncu-rep \
  > gpurun_out/summary_r02.log 2>&1
cp profiles/r02_launches.md profiles/traffic.json gpurun_out/ 2>/dev/null
rm -f gpurun_out/recp.ncu-rep gpurun_out/interp.ncu-rep gpurun_out/row.ncu-rep gpurun_out/col1.ncu-rep \
  gpurun_out/quant.ncu-rep
