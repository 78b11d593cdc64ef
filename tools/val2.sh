mkdir -p gpurun_out/prof
timeout 600 python -m pytest tests/test_gpu_engine.py tests/test_gpu_resnet.py tests/test_gpu_ops.py -q -x 2>&1 | tail -3
timeout 300 python bench.py --model resnet50_exec > gpurun_out/bench_resnet_full.log 2>&1; tail -1 gpurun_out/bench_resnet_full.log | cut -c1-200
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_alex_full2.log 2>&1; tail -1 gpurun_out/bench_alex_full2.log | cut -c1-200
timeout 600 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/resnet50_step_launches.csv python tools/profile_step.py resnet50_exec 32 > gpurun_out/prof/resnet50_step_ncu.log 2>&1
