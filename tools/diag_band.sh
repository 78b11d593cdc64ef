#!/bin/bash
# band-conv diagnostics: per-call time of conv1 forward / weight gradient with
# the kernel's debug variants (skip MMAs / stores / TMA loads), for a knob
# VAR (default STZ_BAND_THIN) off and on, then the knob's A/B on the step
set -u
V=${VAR:-STZ_BAND_THIN}
mkdir -p gpurun_out/diag
for e in 0 1; do
  env $V=$e STZ_DIAG=1 timeout 300 python tools/profile_op.py conv0_fwd > gpurun_out/diag/conv0_fwd_$e.txt 2>&1
  env $V=$e STZ_DIAG=1 timeout 300 python tools/profile_op.py conv0_fwd resnet50_exec 32 > gpurun_out/diag/rn_conv0_fwd_$e.txt 2>&1
done
for f in gpurun_out/diag/*_[01].txt; do echo "== $f"; grep "cluster=1" $f; tail -1 $f; done
VAR=$V MODELS="${MODELS:-alexnet_exec resnet50_exec}" TESTS="${TESTS:-tests/test_gpu_ops.py tests/test_gpu_resnet.py}" bash tools/ab_env.sh
