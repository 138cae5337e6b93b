#!/bin/bash
# A/B of env switches: tools/gpu_ab.sh "ENV=1" "ENV2=0" ... (empty string = baseline)
mkdir -p gpurun_out
: > gpurun_out/ab.log
for e in "$@"; do env $e timeout 300 python tools/dir_probe.py >> gpurun_out/ab.log 2>&1; done
