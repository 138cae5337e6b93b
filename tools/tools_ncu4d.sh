mkdir -p gpurun_out
CMD="python tools_step.py 288,115,69,69"
$CMD > gpurun_out/p4.log 2>&1 || exit 1
for k in kN_rec_interp kN_coef_load0; do
  ncu --set full --clock-control none --import-source on -k "regex:$k" -s 0 -c 1 -o gpurun_out/$k $CMD > gpurun_out/ncu_$k.log 2>&1
  ncu -i gpurun_out/$k.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${k}_src.csv 2>/dev/null
  ncu -i gpurun_out/$k.ncu-rep --page raw --csv > gpurun_out/${k}_raw.csv 2>/dev/null
done
