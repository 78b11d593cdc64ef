#!/bin/bash
# ResNet kinds over one process per GPU (run via gpurun --gpus 4): parity of
# tiny_resnet at 1:1, 3:1, 2:2 against the oracle, and ResNet-50 bench lines.
set -u
mkdir -p gpurun_out/multi
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 $R --nproc-per-node 2 --master-port 29511 tools/dist_parity.py 1 1 tiny_resnet 4 > gpurun_out/multi/parity_11.log 2>&1
timeout 300 $R --nproc-per-node 4 --master-port 29512 tools/dist_parity.py 3 1 tiny_resnet 4 > gpurun_out/multi/parity_31.log 2>&1
timeout 300 $R --nproc-per-node 4 --master-port 29513 tools/dist_parity.py 2 2 tiny_resnet 4 > gpurun_out/multi/parity_22.log 2>&1
timeout 400 $R --nproc-per-node 2 --master-port 29514 bench.py --gpus 2 --model resnet50_exec --steps 10 --warmup 3 > gpurun_out/multi/bench_resnet_2.log 2>&1
timeout 400 $R --nproc-per-node 4 --master-port 29515 bench.py --gpus 4 --model resnet50_exec --steps 10 --warmup 3 > gpurun_out/multi/bench_resnet_4.log 2>&1
grep -h "PASS\|FAIL\|Error" gpurun_out/multi/parity_*.log | head
for f in gpurun_out/multi/bench_resnet_*.log; do tail -1 $f | cut -c1-250; done
