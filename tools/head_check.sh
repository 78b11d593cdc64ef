#!/bin/bash
# last check of HEAD: full GPU suite, smoke, the default bench line
set -u
O=gpurun_out/head
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; tail -2 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -2 $O/smoke.txt
timeout 900 python bench.py > $O/bench_alexnet_exec.jsonl 2> $O/bench_alexnet_exec.err
python tools/bench_calls.py $O/bench_alexnet_exec.jsonl 2>/dev/null | head -2
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.jsonl 2> $O/bench_reference.err
tail -c 400 $O/bench_reference.jsonl
