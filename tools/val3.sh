mkdir -p gpurun_out/prof
timeout 600 python -m pytest tests/test_gpu_engine.py tests/test_gpu_resnet.py -q -x 2>&1 | tail -2
timeout 300 python bench.py --model resnet50_exec > gpurun_out/bench_resnet_full.log 2>&1; tail -1 gpurun_out/bench_resnet_full.log | cut -c1-200
timeout 600 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/resnet50_step_launches.csv python tools/profile_step.py resnet50_exec 32 > gpurun_out/prof/resnet50_step_ncu.log 2>&1
timeout 600 ncu --nvtx --nvtx-include "step/" --set full --import-source on --clock-control none -k regex:bn_bwd_apply -s 20 -c 1 -o gpurun_out/prof/bn_bwd_apply python tools/profile_step.py resnet50_exec 32 > gpurun_out/prof/bn_ncu.log 2>&1
ncu -i gpurun_out/prof/bn_bwd_apply.ncu-rep --page raw --csv > gpurun_out/prof/bn_bwd_apply_raw.csv 2>/dev/null
ncu -i gpurun_out/prof/bn_bwd_apply.ncu-rep --page details --csv > gpurun_out/prof/bn_bwd_apply_details.csv 2>/dev/null
rm -f gpurun_out/prof/bn_bwd_apply.ncu-rep
