"""Accumulation-precision probe: FC forward y = x @ W with growing K through
both GEMM cores vs a float64 reference; reports max rel error and the mean
signed error (a truncating accumulator shows up as a bias toward zero)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1812_10624_b200 import _lib, tensor_core as tc
lib = _lib.load()
rng = np.random.Generator(np.random.PCG64(0))
M, N = 128, 128
for positive in (False, True):
    for K in (64, 512, 2048, 8192, 32768):
        x = rng.standard_normal((M, K)).astype(np.float32)
        w = rng.standard_normal((K, N)).astype(np.float32)
        if positive:
            x, w = np.abs(x), np.abs(w)
        ref = x.astype(np.float64) @ w.astype(np.float64)
        row = []
        for impl, kps in ((0, 0), (0, 64), (2, 0), (1, 0)):
            lib.stz_set_gemm_impl(impl); lib.stz_set_max_k_per_split(kps)
            y, _ = tc.forward(tc.FullyConnected(K, N), [torch.from_numpy(w).cuda(), torch.zeros(N).cuda()], torch.from_numpy(x).cuda())
            yy = y.cpu().numpy().astype(np.float64)
            err = yy - ref
            scale = np.abs(ref).max()
            row.append(f"impl{impl}/kps{kps}: max {np.abs(err).max()/scale:.2e} bias {err.mean()/scale:+.2e}")
        print(f"pos={positive} K={K:6d} | " + " | ".join(row), flush=True)
lib.stz_set_gemm_impl(0); lib.stz_set_max_k_per_split(0)
