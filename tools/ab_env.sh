#!/bin/bash
# A/B of an env knob (VAR, default STZ_WGRAD_STREAM) on 1-GPU bench lines
# (MODELS), after the train tests with the knob on
set -u
V=${VAR:-STZ_WGRAD_STREAM}
mkdir -p gpurun_out/ab
env $V=1 timeout 900 python -m pytest ${TESTS:-tests/test_gpu_train.py} -m gpu -x -q > gpurun_out/ab/pytest.log 2>&1
tail -2 gpurun_out/ab/pytest.log
for m in ${MODELS:-alexnet_exec}; do
  for f in 1 0; do
    env $V=$f timeout 600 python bench.py --model $m --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab/b_${m}_$f.jsonl 2> gpurun_out/ab/b_${m}_$f.err
    python -c "import json;d=json.loads(open('gpurun_out/ab/b_${m}_$f.jsonl').readlines()[-1]);print('$m $V=$f', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['ms_per_step'])"
  done
done
