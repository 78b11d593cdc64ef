#!/bin/bash
# One GPU-box pass for the round's evidence (run via gpurun from the repo root):
# full GPU suite, smoke, both bench lines, the ResNet-50 step launch list and
# one ncu --set full capture of the BatchNorm backward apply kernel.
set -u
mkdir -p gpurun_out/prof
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest_exit=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 400 python bench.py > gpurun_out/bench_alex_full.log 2>&1
timeout 600 python bench.py --model resnet50_exec > gpurun_out/bench_resnet_full.log 2>&1
timeout 600 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none \
  --csv --log-file gpurun_out/prof/resnet50_step_launches.csv \
  python tools/profile_step.py resnet50_exec 32 > gpurun_out/prof/resnet50_step_ncu.log 2>&1
timeout 600 ncu --nvtx --nvtx-include "step/" --set full --import-source on --clock-control none \
  -k regex:bn_bwd_apply -c 1 -o gpurun_out/prof/bn_bwd_apply \
  python tools/profile_step.py resnet50_exec 32 > gpurun_out/prof/bn_ncu.log 2>&1
ncu -i gpurun_out/prof/bn_bwd_apply.ncu-rep --page raw --csv > gpurun_out/prof/bn_bwd_apply_raw.csv 2>/dev/null
ncu -i gpurun_out/prof/bn_bwd_apply.ncu-rep --page details --csv > gpurun_out/prof/bn_bwd_apply_details.csv 2>/dev/null
rm -f gpurun_out/prof/bn_bwd_apply.ncu-rep
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log
tail -1 gpurun_out/bench_alex_full.log | cut -c1-200; tail -1 gpurun_out/bench_resnet_full.log | cut -c1-200
