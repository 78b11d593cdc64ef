#!/bin/bash
# first stride-1 conv on few channels packed 32 wide (TMA GEMM instead of the fallback):
# full GPU suite, then VGG-16 bench lines with STZ_FIRST_C32=1 / 0
set -u
O=gpurun_out/fc32
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; tail -2 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -2 $O/smoke.txt
for f in 1 0; do
  STZ_FIRST_C32=$f timeout 900 python bench.py --model vgg16_exec --steps 10 --warmup 3 --no-cpu-baseline > $O/b_vgg16_$f.jsonl 2> $O/b_vgg16_$f.err
  python -c "import json;d=json.loads(open('$O/b_vgg16_$f.jsonl').readlines()[-1]);print('vgg16 STZ_FIRST_C32=$f', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['ms_per_step']); c=d['roofline']['calls']; print({k:round(v['ms']*1000) for k,v in c.items() if k.startswith('conv0')})"
done
