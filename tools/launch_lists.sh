#!/bin/bash
# step launch lists (ncu, cold-cache, serialised) of the ResNet-50 / Inception-V3 / VGG-16 steps on this build
set -u
O=gpurun_out/ll
mkdir -p $O
for m in "resnet50_exec 32" "inception_v3_exec 32" "vgg16_exec 64"; do
  set -- $m
  timeout 900 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/${1}_step_launches.csv python tools/profile_step.py $1 $2 > $O/${1}_ncu.log 2>&1
  echo "== $1"; python tools/launch_summary.py $O/${1}_step_launches.csv 2>/dev/null | head -14
done
