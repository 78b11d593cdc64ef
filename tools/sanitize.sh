#!/bin/bash
# compute-sanitizer over the step's kernels (one GPU): memcheck / racecheck /
# synccheck on tools/sanitize_step.py per model family, and memcheck on the
# multi-process peer-memory link + exchange (2 processes sharing cuda:0).
# Logs: gpurun_out/sanitizer_<tool>_<model>.log
set -u
OUT=gpurun_out
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for model in tiny_cnn tiny_resnet tiny_inception alexnet; do
    timeout 900 $CS --tool $tool --print-limit 20 --error-exitcode 9 \
      python tools/sanitize_step.py $model > $OUT/sanitizer_${tool}_${model}.log 2>&1
    echo "$tool $model rc=$?" | tee -a $OUT/sanitizer_summary.txt
    tail -3 $OUT/sanitizer_${tool}_${model}.log >> $OUT/sanitizer_summary.txt
  done
done
timeout 900 $CS --tool memcheck --target-processes all --print-limit 20 --error-exitcode 9 \
  python -m torch.distributed.run --nnodes=1 --nproc-per-node=3 --master-addr=127.0.0.1 \
  --master-port=29931 tools/dist_parity.py --n-conv 2 --n-fc 1 --iters 2 --micro 2 --same-gpu \
  > $OUT/sanitizer_memcheck_peer_2x1.log 2>&1
echo "memcheck peer 2:1 rc=$?" | tee -a $OUT/sanitizer_summary.txt
grep -E "PASS|FAIL|ERROR SUMMARY" $OUT/sanitizer_memcheck_peer_2x1.log | tail -5 >> $OUT/sanitizer_summary.txt
