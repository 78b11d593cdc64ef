#!/bin/bash
# Round-2 closing evidence on one B200 (gpurun): full GPU suite, smoke, the
# default bench line (with its CPU baseline), the other models' 1-GPU lines,
# the AlexNet step launch list, and ncu --set full of the bench line's
# roofline kernel (conv3_dgrad), conv1's band kernels and the tiled pool bwd
set -u
O=gpurun_out/final
mkdir -p $O/prof
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; tail -2 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -2 $O/smoke.txt
timeout 900 python bench.py > $O/bench_alexnet_exec.jsonl 2> $O/bench_alexnet_exec.err
python tools/bench_calls.py $O/bench_alexnet_exec.jsonl 2>/dev/null | head -2
for m in resnet50_exec inception_v3_exec vgg16_exec; do
  timeout 600 python bench.py --model $m --steps 10 --warmup 5 --no-cpu-baseline > $O/bench_$m.jsonl 2> $O/bench_$m.err
  python tools/bench_calls.py $O/bench_$m.jsonl 2>/dev/null | head -1
done
timeout 600 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/prof/alexnet_step_launches.csv python tools/profile_step.py > $O/prof/step_ncu.log 2>&1
python tools/launch_summary.py $O/prof/alexnet_step_launches.csv 2>/dev/null | head -12
for tag in conv3_dgrad conv0_wgrad conv0_fwd pool2_bwd; do
  timeout 600 ncu --nvtx --nvtx-include "replay/" --set full --import-source on --clock-control none \
      -k regex:"tgemm|band|maxpool" -c 1 -o $O/prof/$tag python tools/profile_op.py $tag > $O/prof/${tag}_ncu.log 2>&1
  ncu -i $O/prof/$tag.ncu-rep --page raw --csv > $O/prof/${tag}_raw.csv 2>/dev/null
  ncu -i $O/prof/$tag.ncu-rep --page details --csv > $O/prof/${tag}_details.csv 2>/dev/null
  rm -f $O/prof/$tag.ncu-rep
done
ls -la $O/prof
