#!/bin/bash
# multi-GPU pass (gpurun --gpus 4): the torchrun parity tests, then AlexNet
# bench lines at 2 (1:1) and 4 GPUs (3:1, 2:2) and ResNet-50 at 4 (3:1)
set -u
mkdir -p gpurun_out/multi
timeout 900 python -m pytest tests/test_gpu_dist.py -m gpu -x -q > gpurun_out/multi/pytest_dist.log 2>&1
tail -3 gpurun_out/multi/pytest_dist.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 500 $R --nproc-per-node 2 --master-port 29521 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/multi/bench_alex_2.log 2>&1
timeout 500 $R --nproc-per-node 4 --master-port 29522 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/multi/bench_alex_4_31.log 2>&1
timeout 500 $R --nproc-per-node 4 --master-port 29523 bench.py --gpus 4 --fc-workers 2 --steps 20 --warmup 5 > gpurun_out/multi/bench_alex_4_22.log 2>&1
timeout 500 $R --nproc-per-node 4 --master-port 29524 bench.py --gpus 4 --model resnet50_exec --steps 10 --warmup 3 > gpurun_out/multi/bench_resnet_4.log 2>&1
for f in gpurun_out/multi/bench_*.log; do echo $f; tail -1 $f | python -c "import json,sys
try:
  d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['ms_per_step'], (d.get('nvlink') or {}).get('exchange_GBps'))
except Exception as e: print('no json', e)"; done
