for f in 0 1; do for m in alexnet_exec resnet50_exec; do
STZ_FIXUP=$f python bench.py --model $m --steps 10 --warmup 5 --no-cpu-baseline > gpurun_out/fx_${m}_$f.jsonl 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/fx_${m}_$f.jsonl').readline());print('fixup=$f', '$m', round(d['value'],1), round(d['ms_per_step'],3))"
done; done
