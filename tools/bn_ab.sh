#!/bin/bash
# BatchNorm A/B: the BN / ResNet / Inception GPU tests on the one-launch
# BatchNorm, then ResNet-50 and Inception-V3 bench lines with it on and off
set -u
mkdir -p gpurun_out/bn
timeout 900 python -m pytest tests/test_gpu_resnet.py tests/test_gpu_inception.py -m gpu -x -q > gpurun_out/bn/pytest.log 2>&1
tail -3 gpurun_out/bn/pytest.log
for m in ${MODELS:-resnet50_exec inception_v3_exec}; do
  for f in 1 0; do
    STZ_BN_FUSED=$f timeout 600 python bench.py --model $m --steps 10 --warmup 5 --no-cpu-baseline > gpurun_out/bn/b_${m}_$f.jsonl 2> gpurun_out/bn/b_${m}_$f.err
    echo "fused=$f"; python tools/bench_calls.py gpurun_out/bn/b_${m}_$f.jsonl | head -8
  done
done
