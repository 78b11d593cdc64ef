#!/bin/bash
# FC-boundary (CHW-flat) max-pool in channel parts: tests, per-call times, step A/B
set -u
mkdir -p gpurun_out/pf
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_train.py tests/test_gpu_engine.py -m gpu -x -q > gpurun_out/pf/pytest.txt 2>&1; tail -2 gpurun_out/pf/pytest.txt
for p in 0 1; do
  for tag in pool12_fwd pool12_bwd; do
    STZ_POOL_FLAT_PARTS=$p timeout 300 python tools/profile_op.py $tag 2>&1 | tail -1 | sed "s/^/parts=$p /"
  done
done
for p in 0 1; do
  STZ_POOL_FLAT_PARTS=$p timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/pf/b_$p.jsonl 2> gpurun_out/pf/b_$p.err
  python -c "import json;d=json.loads(open('gpurun_out/pf/b_$p.jsonl').readlines()[-1]);print('parts=$p', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['ms_per_step'])"
done
