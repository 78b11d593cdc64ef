#!/bin/bash
# bias-stream / prefetch check: affected tests, AlexNet bench, BN ncu captures
set -u
mkdir -p gpurun_out/r3/prof
timeout 900 python -m pytest tests/test_gpu_ops.py::test_colsum_matches_wgrad_bias tests/test_gpu_train.py tests/test_gpu_engine.py tests/test_gpu_dropin.py -m gpu -x -q > gpurun_out/r3/pytest.log 2>&1
tail -3 gpurun_out/r3/pytest.log
for m in alexnet_exec vgg16_exec; do
  timeout 600 python bench.py --model $m --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r3/b_$m.jsonl 2> gpurun_out/r3/b_$m.err
  python tools/bench_calls.py gpurun_out/r3/b_$m.jsonl 2>/dev/null | head -2
  python -c "import json;d=json.loads(open('gpurun_out/r3/b_$m.jsonl').readlines()[-1]);print('e2e',d['e2e']['value'],'value',d['value'])"
done
for d in 0 1; do
  timeout 600 ncu --nvtx --nvtx-include "step/" --set full --import-source on --clock-control none \
    --kernel-name-base demangled -k "regex:bn_fused_kernel<.bool.$d>" -c 1 -o gpurun_out/r3/prof/bn_fused_$d \
    python tools/profile_step.py resnet50_exec 32 > gpurun_out/r3/prof/bn_$d.log 2>&1
  ncu -i gpurun_out/r3/prof/bn_fused_$d.ncu-rep --page raw --csv > gpurun_out/r3/prof/bn_fused_${d}_raw.csv 2>/dev/null
  ncu -i gpurun_out/r3/prof/bn_fused_$d.ncu-rep --page details --csv > gpurun_out/r3/prof/bn_fused_${d}_details.csv 2>/dev/null
  rm -f gpurun_out/r3/prof/bn_fused_$d.ncu-rep
done
ls -la gpurun_out/r3/prof
