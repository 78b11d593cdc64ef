#!/bin/bash
# band weight-gradient diagnostics (debug variants: skip stores / MMAs / TMA),
# then the full GPU suite and smoke on this build
set -u
mkdir -p gpurun_out/diag
STZ_DIAG=1 timeout 300 python tools/profile_op.py conv0_wgrad > gpurun_out/diag/conv0_wgrad.txt 2>&1
STZ_DIAG=1 timeout 300 python tools/profile_op.py conv0_wgrad resnet50_exec 32 > gpurun_out/diag/rn_conv0_wgrad.txt 2>&1
for f in gpurun_out/diag/*wgrad.txt; do echo "== $f"; grep "cluster=1" $f; tail -1 $f; done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/diag/pytest_gpu_full.txt 2>&1
tail -2 gpurun_out/diag/pytest_gpu_full.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/diag/smoke.txt 2>&1; tail -2 gpurun_out/diag/smoke.txt
