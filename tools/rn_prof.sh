#!/bin/bash
# ResNet-50 K=32 step: launch list (serialised, ncu) + bench line
set -u
mkdir -p gpurun_out/rp
python -m pytest tests/test_gpu_ops.py -m gpu -x -q -k "pack or strided" > gpurun_out/rp/pytest.log 2>&1; tail -2 gpurun_out/rp/pytest.log
python bench.py --model resnet50_exec --steps 10 --warmup 5 --no-cpu-baseline > gpurun_out/rp/bres.jsonl 2> gpurun_out/rp/bres.err
python tools/bench_calls.py gpurun_out/rp/bres.jsonl
python tools/profile_step.py resnet50_exec 32 > gpurun_out/rp/step_plain.log 2>&1 || exit 1
ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/rp/step_launches.csv python tools/profile_step.py resnet50_exec 32 > gpurun_out/rp/step_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/rp/step_launches.csv | head -40
