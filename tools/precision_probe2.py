"""Where does the tcgen05 error come from?  Inputs exactly representable in
bf16 (so the 3-way split is exact and only b0*b0 is non-zero): any error is
the hardware's product-sum / accumulation."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1812_10624_b200 import _lib, tensor_core as tc
lib = _lib.load()
rng = np.random.Generator(np.random.PCG64(1))
M, N = 128, 128
def bf16(a):
    b = a.astype(np.float32).view(np.uint32)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return b.view(np.float32)
for kind in ("bf16-exact positive", "bf16-exact signed", "bf16-exact positive, same exponent"):
    for K in (16, 32, 64, 256, 1024, 4096):
        if "same exponent" in kind:
            x = bf16(1.0 + rng.random((M, K)).astype(np.float32)); w = bf16(1.0 + rng.random((K, N)).astype(np.float32))
        else:
            x = bf16(rng.standard_normal((M, K))); w = bf16(rng.standard_normal((K, N)))
            if "positive" in kind: x, w = np.abs(x), np.abs(w)
        ref = x.astype(np.float64) @ w.astype(np.float64)
        row = []
        for impl, kps in ((0, 0), (0, 32), (1, 0)):
            lib.stz_set_gemm_impl(impl); lib.stz_set_max_k_per_split(kps)
            y, _ = tc.forward(tc.FullyConnected(K, N), [torch.from_numpy(w).cuda(), torch.zeros(N).cuda()], torch.from_numpy(x).cuda())
            err = y.cpu().numpy().astype(np.float64) - ref
            # error in units of fp32 ulp of the exact result
            ulp = np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64)
            row.append(f"impl{impl}/kps{kps}: maxulp {np.abs(err/ulp).max():7.1f} meanulp {np.mean(err/ulp):+7.2f}")
        print(f"{kind:36s} K={K:5d} | " + " | ".join(row), flush=True)
lib.stz_set_gemm_impl(0); lib.stz_set_max_k_per_split(0)
