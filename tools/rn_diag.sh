set -u
mkdir -p gpurun_out/rn
python -m pytest tests/test_gpu_resnet.py tests/test_gpu_inception.py tests/test_gpu_engine.py -m gpu -x -q > gpurun_out/bn_t.log 2>&1; tail -3 gpurun_out/bn_t.log
python bench.py --model resnet50_exec --steps 10 --warmup 5 --no-cpu-baseline > gpurun_out/bres.jsonl 2> gpurun_out/bres.err
python bench.py --model inception_v3_exec --steps 10 --warmup 5 --no-cpu-baseline > gpurun_out/binc.jsonl 2>> gpurun_out/bres.err
python tools/bench_calls.py gpurun_out/bres.jsonl gpurun_out/binc.jsonl
for t in r4b.conv6_fwd r5b.conv0_dgrad r7b.conv3_dgrad conv0_wgrad conv0_fwd r5b.conv3_wgrad; do
  echo "== $t"; STZ_DIAG=1 STZ_SWEEP=1 timeout 300 python tools/profile_op.py $t resnet50_exec 32 2>&1 | tail -25
done > gpurun_out/rn/diag.txt
timeout 600 ncu --nvtx --nvtx-include "replay/" --set full --import-source on --clock-control none -k regex:"tgemm" -c 1 -o gpurun_out/rn/conv6_fwd python tools/profile_op.py r4b.conv6_fwd resnet50_exec 32 > gpurun_out/rn/ncu.log 2>&1
ncu -i gpurun_out/rn/conv6_fwd.ncu-rep --page details --csv > gpurun_out/rn/conv6_fwd_details.csv 2>/dev/null
ncu -i gpurun_out/rn/conv6_fwd.ncu-rep --page raw --csv > gpurun_out/rn/conv6_fwd_raw.csv 2>/dev/null
rm -f gpurun_out/rn/conv6_fwd.ncu-rep
