#!/bin/bash
# ncu --set full of the one-launch BatchNorm (first forward / backward launch
# of the ResNet-50 step) and of AlexNet's pool2 backward
set -u
mkdir -p gpurun_out/nb
for d in 0 1; do
  timeout 600 ncu --nvtx --nvtx-include "step/" --set full --import-source on --clock-control none \
    --kernel-name-base demangled -k "regex:bn_fused_kernel<.bool.$d>" -c 1 -o gpurun_out/nb/bn_fused_$d \
    python tools/profile_step.py resnet50_exec 32 > gpurun_out/nb/bn_$d.log 2>&1
  ncu -i gpurun_out/nb/bn_fused_$d.ncu-rep --page raw --csv > gpurun_out/nb/bn_fused_${d}_raw.csv 2>/dev/null
  ncu -i gpurun_out/nb/bn_fused_$d.ncu-rep --page details --csv > gpurun_out/nb/bn_fused_${d}_details.csv 2>/dev/null
  ncu -i gpurun_out/nb/bn_fused_$d.ncu-rep --page source --csv > gpurun_out/nb/bn_fused_${d}_source.csv 2>/dev/null
  rm -f gpurun_out/nb/bn_fused_$d.ncu-rep
done
timeout 600 ncu --nvtx --nvtx-include "step/" --set full --import-source on --clock-control none \
  -k regex:maxpool_bwd_nhwc -c 1 -o gpurun_out/nb/pool_bwd python tools/profile_step.py alexnet_exec 128 > gpurun_out/nb/pool.log 2>&1
ncu -i gpurun_out/nb/pool_bwd.ncu-rep --page details --csv > gpurun_out/nb/pool_bwd_details.csv 2>/dev/null
ncu -i gpurun_out/nb/pool_bwd.ncu-rep --page raw --csv > gpurun_out/nb/pool_bwd_raw.csv 2>/dev/null
rm -f gpurun_out/nb/pool_bwd.ncu-rep
ls -la gpurun_out/nb
