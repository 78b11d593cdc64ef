#!/bin/bash
# quick GPU iteration: selected test files (TESTS), then 1-GPU bench lines (MODELS)
set -u
mkdir -p gpurun_out/q
timeout 1200 python -m pytest ${TESTS:-tests/test_gpu_train.py} -m gpu -x -q > gpurun_out/q/pytest.log 2>&1
tail -3 gpurun_out/q/pytest.log
for m in ${MODELS:-alexnet_exec}; do
  timeout 600 python bench.py --model $m --steps 10 --warmup 5 --no-cpu-baseline > gpurun_out/q/b_$m.jsonl 2> gpurun_out/q/b_$m.err
  python tools/bench_calls.py gpurun_out/q/b_$m.jsonl 2>/dev/null | head -9
done
