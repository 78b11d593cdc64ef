"""Diagnostic (GPU box): compare CTA-pair (cta_group::2) GEMMs with single-CTA
GEMMs for every operand mode and split-K combination the layers produce."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1812_10624_b200 import _lib, tensor_core as tc  # noqa: E402

lib = _lib.load()


def dev(a):
    return torch.from_numpy(a).cuda()


def run_fc(m, i, o):
    rng = np.random.Generator(np.random.PCG64(m + i + o))
    x = rng.standard_normal((m, i)).astype(np.float32)
    w = (rng.standard_normal((i, o)) / np.sqrt(i)).astype(np.float32)
    b = rng.standard_normal(o).astype(np.float32)
    gy = rng.standard_normal((m, o)).astype(np.float32)
    layer = tc.FullyConnected(i, o)
    params = [dev(w), dev(b)]
    y, cache = tc.forward(layer, params, dev(x))
    gx, (gw, gb) = tc.backward(layer, params, cache, dev(gy))
    torch.cuda.synchronize()
    return {"fwd": y.cpu(), "dgrad": gx.cpu(), "wgrad": gw.cpu()}


def run_conv(n, c, h, w_, o, k, s, p):
    rng = np.random.Generator(np.random.PCG64(n + c + o))
    x = rng.standard_normal((n, c, h, w_)).astype(np.float32)
    wt = (rng.standard_normal((o, c, k, k)) / np.sqrt(c * k * k)).astype(np.float32)
    b = rng.standard_normal(o).astype(np.float32)
    layer = tc.Conv2d(c, o, k, s, p)
    params = [dev(wt), dev(b)]
    y, cache = tc.forward(layer, params, dev(x))
    gy = dev(rng.standard_normal(tuple(y.shape)).astype(np.float32))
    gx, (gw, gb) = tc.backward(layer, params, cache, gy)
    torch.cuda.synchronize()
    return {"fwd": y.cpu(), "dgrad": gx.cpu(), "wgrad": gw.cpu()}


CASES = [("fc", (1024, 1024, 1024)), ("fc", (4096, 512, 256)), ("fc", (256, 4096, 4096)),
         ("fc", (300, 640, 192)), ("conv", (2, 64, 13, 13, 128, 3, 1, 1)),
         ("conv", (2, 192, 13, 13, 384, 3, 1, 1)), ("conv", (8, 64, 27, 27, 192, 5, 1, 2))]

def run_head(dims, batch, seed=6):
    """BlockEngine over an FC stack (the failing engine test's path): output,
    per-layer gradients, input gradient."""
    from paper_1812_10624_b200.engine import BlockEngine, Split, rup8
    from paper_1812_10624_b200.tensor_core import FullyConnected, ReLU, ptr, seeded_init, stream_of
    layers = []
    for i in range(len(dims) - 1):
        layers += [FullyConnected(dims[i], dims[i + 1]), ReLU()]
    layers = layers[:-1]
    params = seeded_init(layers, seed)
    eng = BlockEngine(layers, (dims[0],), batch, "cuda:0", params, need_input_grad=True)
    rng = np.random.Generator(np.random.PCG64(seed))
    x = rng.standard_normal((batch, dims[0])).astype(np.float32)
    out = eng.forward(dev(x))
    gy = rng.standard_normal((batch, dims[-1])).astype(np.float32)
    g = Split.alloc("rows", (batch, rup8(dims[-1])), dims[-1], "cuda:0")
    _lib.call("stzx_pack_rows", ptr(dev(gy)), g.ptr(), g.ps, batch, dims[-1], g.width,
              stream_of(torch.device("cuda:0")))
    gin = eng.backward(g)
    torch.cuda.synchronize()
    res = {"out": out.to_float().cpu(), "gin": gin.to_float().cpu()}
    for li, gl in enumerate(eng.grads):
        for j, a in enumerate(gl):
            res[f"grad{li}.{j}"] = a.detach().cpu().clone()
    return res


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "head":
        CASES = [("head", ((9216, 4096, 4096, 1000), 896)), ("head", ((4096, 1000), 896)),
                 ("head", ((4096, 4096), 896)), ("head", ((9216, 4096), 896)),
                 ("head", ((1024, 1024, 1000), 512))]
    for kind, shp in CASES:
        if kind == "head":
            fn = run_head
        else:
            fn = run_fc if kind == "fc" else run_conv
        lib.stz_set_cluster(0)
        ref = fn(*shp)
        lib.stz_set_cluster(1)
        got = fn(*shp)
        for key in ref:
            a, b = ref[key], got[key]
            d = (a - b).abs().max().item()
            print(f"{kind}{shp} {key}: max|diff| {d:.3e}  nan {int(torch.isnan(b).sum())}  "
                  f"scale {a.abs().max().item():.3e}", flush=True)
