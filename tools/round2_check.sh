#!/bin/bash
# Round-2 evidence pass: full GPU suite, smoke, the 1-GPU bench lines, the
# ResNet-50 step launch list and ncu --set full captures of the one-launch
# BatchNorm (forward and backward, first launch of each in the step)
set -u
mkdir -p gpurun_out/r2/prof
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2/pytest_gpu.log 2>&1
tail -3 gpurun_out/r2/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2/smoke.log 2>&1; tail -2 gpurun_out/r2/smoke.log
for m in ${MODELS:-alexnet_exec resnet50_exec inception_v3_exec}; do
  timeout 600 python bench.py --model $m --steps 10 --warmup 5 --no-cpu-baseline > gpurun_out/r2/b_$m.jsonl 2> gpurun_out/r2/b_$m.err
  python tools/bench_calls.py gpurun_out/r2/b_$m.jsonl 2>/dev/null | head -3
done
timeout 600 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r2/prof/resnet50_step_launches.csv python tools/profile_step.py resnet50_exec 32 > gpurun_out/r2/prof/step_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/r2/prof/resnet50_step_launches.csv | head -12
for d in 0 1; do
  timeout 600 ncu --nvtx --nvtx-include "step/" --set full --import-source on --clock-control none \
    --kernel-name-base demangled -k "regex:bn_fused_kernel<.bool.$d>" -c 1 -o gpurun_out/r2/prof/bn_fused_$d \
    python tools/profile_step.py resnet50_exec 32 > gpurun_out/r2/prof/bn_$d.log 2>&1
  ncu -i gpurun_out/r2/prof/bn_fused_$d.ncu-rep --page raw --csv > gpurun_out/r2/prof/bn_fused_${d}_raw.csv 2>/dev/null
  ncu -i gpurun_out/r2/prof/bn_fused_$d.ncu-rep --page details --csv > gpurun_out/r2/prof/bn_fused_${d}_details.csv 2>/dev/null
  rm -f gpurun_out/r2/prof/bn_fused_$d.ncu-rep
done
ls -la gpurun_out/r2/prof
