"""GPU cost of running the AlexNet CONV block as m micro-batches instead of one
K=128 batch (each variant captured in a CUDA graph, so host launch overhead is
excluded): the efficiency price micro-batch pipelining has to beat."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1812_10624_b200 import _lib  # noqa: E402
from paper_1812_10624_b200.engine import BlockEngine, Split, rup8  # noqa: E402
from paper_1812_10624_b200.model_partition import builtin_model, split  # noqa: E402
from paper_1812_10624_b200.tensor_core import seeded_init  # noqa: E402

_lib.load()
dev = torch.device("cuda:0")
K = 128
spec = builtin_model("alexnet_exec", K)
part = split(spec)
cut = part.split_index
params = seeded_init(spec.layers, 3)[:cut]
eng = BlockEngine(part.conv_block, tuple(spec.input_shape), K, dev, params,
                  need_input_grad=False)
x = torch.randn(K, *spec.input_shape, device=dev)
a = eng.out_shape[0] if len(eng.out_shape) == 1 else None
gy = Split.alloc("rows", (K, rup8(9216)), 9216, dev)
gy.storage.normal_()


def run(m):
    kb = K // m
    for j in range(m):
        eng.forward(x, rows=(j * kb, (j + 1) * kb))
    for j in range(m):
        eng.backward(gy, rows=(j * kb, (j + 1) * kb), accumulate=j > 0)


for m in (1, 2, 4, 8):
    run(m)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            run(m)
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"micro={m}: conv block fwd+bwd {e0.elapsed_time(e1) / 10:.3f} ms", flush=True)
