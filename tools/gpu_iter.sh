#!/bin/bash
# one GPU iteration: the GPU test suite, then the 1-GPU bench lines of the
# four models with their per-call summaries (gpurun_out/it/)
set -u
mkdir -p gpurun_out/it
python -m pytest tests -m gpu -x -q > gpurun_out/it/pytest.log 2>&1; tail -3 gpurun_out/it/pytest.log
for m in ${MODELS:-alexnet_exec resnet50_exec inception_v3_exec}; do
  python bench.py --model $m --steps 10 --warmup 5 --no-cpu-baseline > gpurun_out/it/b_$m.jsonl 2> gpurun_out/it/b_$m.err
  python tools/bench_calls.py gpurun_out/it/b_$m.jsonl
done
