#!/bin/bash
# Regenerate the committed ncu evidence for the current build (run on a GPU
# box via gpurun; results land in gpurun_out/prof/, then copy to profiles/).
#   1. launch list of one co-located AlexNet K=128 step (cold cache, serialised)
#   2. ncu --set full of the GEMM behind each top ABI call (NVTX-isolated replay)
set -u
OUT=gpurun_out/prof
mkdir -p "$OUT"
python tools/profile_step.py > "$OUT/step_plain.log" 2>&1 || exit 1
ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$OUT/step_launches.csv" python tools/profile_step.py > "$OUT/step_ncu.log" 2>&1
for tag in "$@"; do
  python tools/profile_op.py "$tag" > "$OUT/${tag}_plain.log" 2>&1 || continue
  ncu --nvtx --nvtx-include "replay/" --set full --import-source on --clock-control none \
      -k regex:"tgemm|band" -c 1 -o "$OUT/$tag" python tools/profile_op.py "$tag" > "$OUT/${tag}_ncu.log" 2>&1
  ncu -i "$OUT/$tag.ncu-rep" --page raw --csv > "$OUT/${tag}_raw.csv" 2>/dev/null
  ncu -i "$OUT/$tag.ncu-rep" --page details --csv > "$OUT/${tag}_details.csv" 2>/dev/null
  ncu -i "$OUT/$tag.ncu-rep" --page source --csv --print-source sass > "$OUT/${tag}_source.csv" 2>/dev/null
  rm -f "$OUT/$tag.ncu-rep"
done
