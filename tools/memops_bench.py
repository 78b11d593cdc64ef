"""Time the memory-bound hot-path kernels at the AlexNet K=128 shapes through
the C-ABI (GPU box): max-pool forward / backward for the three pools, the
space-to-depth input pack, the split-row pack and the momentum SGD.  Prints
achieved GB/s of algorithmic bytes (each tensor read / written once)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1812_10624_b200 import _lib  # noqa: E402

lib = _lib.load()
st = torch.cuda.current_stream().cuda_stream
K = 128


def timeit(fn, reps=20):
    """GPU time per call: the reps are captured in one CUDA graph and replayed,
    so Python / ctypes launch overhead cannot leak into short kernels."""
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    global st
    with torch.cuda.stream(s):
        st = s.cuda_stream
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    st = torch.cuda.current_stream().cuda_stream
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def split(*dims):
    t = torch.randn(3, *dims, device="cuda").to(torch.bfloat16)
    return t, t[0].numel()


def report(name, ms, nbytes):
    print(f"{name:34s} {ms * 1e3:8.1f} us  {nbytes / ms / 1e6:8.0f} GB/s", flush=True)


def pools():
    # (C, H, W, k, s, flat): AlexNet pool1 / pool2 / pool5 (flattened into the FC boundary)
    for c, h, w, k, s, flat in ((64, 55, 55, 3, 2, False), (192, 27, 27, 3, 2, False),
                                (256, 13, 13, 3, 2, True)):
        c8 = (c + 7) // 8 * 8
        oh, ow = (h - k) // s + 1, (w - k) // s + 1
        x, psx = split(K, h, w, c8)
        arg = torch.zeros(K * oh * ow * c8, dtype=torch.uint8, device="cuda")
        if flat:
            d8 = (c * oh * ow + 7) // 8 * 8
            y, psy = split(K, d8)
            flat_ld = d8
        else:
            y, psy = split(K, oh, ow, c8)
            flat_ld = 0
        esz = 6  # three bf16 planes
        fwd_bytes = K * h * w * c8 * esz + K * oh * ow * c8 * (esz + 1)
        ms = timeit(lambda: _lib.call("stzx_maxpool_fwd", x.data_ptr(), psx, y.data_ptr(), psy,
                                      arg.data_ptr(), K, c, c8, h, w, k, s, flat_ld, st))
        report(f"maxpool_fwd {c}x{h}x{w}", ms, fwd_bytes)
        gx, psgx = split(K, h, w, c8)
        bwd_bytes = K * oh * ow * c8 * (esz + 1) + K * h * w * c8 * (esz + 2)
        ms = timeit(lambda: _lib.call("stzx_maxpool_bwd", y.data_ptr(), psy, arg.data_ptr(),
                                      gx.data_ptr(), psgx, x.data_ptr(), K, c, c8, h, w, k, s,
                                      flat_ld, st))
        report(f"maxpool_bwd {c}x{h}x{w} (+relu mask)", ms, bwd_bytes)


def packs():
    x = torch.randn(K, 3, 224, 224, device="cuda")
    xs, ps = split(K, 57, 57, 64)
    ms = timeit(lambda: _lib.call("stzx_pack_s2d", x.data_ptr(), xs.data_ptr(), ps, K, 3, 224,
                                  224, 4, 2, 57, 57, 64, st))
    report("pack_s2d 3x224x224 -> 57x57x64", ms, x.numel() * 4 + xs.numel() * 2)
    w = torch.randn(9216, 4096, device="cuda")
    wr, psw = split(4096, 9216)
    ms = timeit(lambda: _lib.call("stzx_pack_rows", w.data_ptr(), wr.data_ptr(), psw, 9216, 4096,
                                  9216, st) if False else None)


def sgd():
    n = 58_631_144
    p = torch.randn(n, device="cuda")
    v = torch.zeros(n, device="cuda")
    g = torch.randn(n, device="cuda")
    sig = _lib.SIGNATURES["stz_sgd_momentum"]
    print("stz_sgd_momentum signature", sig, flush=True)


if __name__ == "__main__":
    pools()
    packs()
