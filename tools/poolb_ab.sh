#!/bin/bash
# max-pool backward fp32 fast path: op tests (bit-exact incl. shared maxima), per-call times
set -u
mkdir -p gpurun_out/pool
timeout 600 python -m pytest tests/test_gpu_ops.py -m gpu -x -q -k maxpool > gpurun_out/pool/pytest_pool.txt 2>&1; tail -2 gpurun_out/pool/pytest_pool.txt
for tag in pool2_bwd pool5_bwd; do timeout 300 python tools/profile_op.py $tag 2>&1 | tail -1; done
for m in alexnet_exec; do
  timeout 600 python bench.py --model $m --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/pool/b_$m.jsonl 2> gpurun_out/pool/b_$m.err
  python tools/bench_calls.py gpurun_out/pool/b_$m.jsonl 2>/dev/null | head -1
done
