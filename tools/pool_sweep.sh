#!/bin/bash
# tiled max-pool backward: shared-memory budget x block size sweep (per-call times)
set -u
for kb in 24 48 96 160; do for t in 128 256 512; do
  for tag in pool2_bwd pool5_bwd; do
    STZ_POOL_KB=$kb STZ_POOL_THREADS=$t timeout 300 python tools/profile_op.py $tag 2>&1 | tail -1 | sed "s/^/kb=$kb thr=$t /"
  done
done; done
