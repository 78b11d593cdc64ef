#!/bin/bash
# max-pool forward: op tests, per-call times tiled vs untiled, step A/B
set -u
mkdir -p gpurun_out/pool
timeout 600 python -m pytest tests/test_gpu_ops.py -m gpu -x -q -k maxpool > gpurun_out/pool/pytest_pool.txt 2>&1; tail -2 gpurun_out/pool/pytest_pool.txt
for t in 1 0; do
  for tag in pool2_fwd pool5_fwd pool2_bwd; do
    STZ_POOL_TILED=$t timeout 300 python tools/profile_op.py $tag 2>&1 | tail -1 | sed "s/^/tiled=$t /"
  done
done
VAR=STZ_POOL_TILED MODELS="${MODELS:-alexnet_exec}" TESTS="${TESTS:-tests/test_gpu_train.py}" bash tools/ab_env.sh
