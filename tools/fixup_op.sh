for t in conv3_fwd conv2_wgrad conv4_dgrad; do for f in 0 1; do
  echo "== $t fixup=$f"; STZ_FIXUP=$f STZ_AUTOTUNE=0 STZ_TRACE=1 timeout 300 python tools/profile_op.py $t alexnet_exec 128 2>&1 | grep -E "stz\]|ms" | tail -4
done; done
