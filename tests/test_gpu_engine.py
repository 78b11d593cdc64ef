"""BlockEngine (the fused hot path on split-plane tensors) vs the oracle at
the block level: forward output, parameter-gradient sums and the block input
gradient, for the layer stacks the bench runs (AlexNet conv1 as
space-to-depth, TMA im2col convs, pool -> flatten -> FC boundary).

Tolerance: conftest.gemm_tol(K) of the longest contraction in the stack
(rel_err of the tensor max); the input gradient of a block crosses every GEMM
of the chain, so it gets that x (number of GEMM layers)."""

import numpy as np
import pytest
import torch

import stanza_oracle as orc
from conftest import gemm_tol

pytestmark = pytest.mark.gpu
TOL = 3e-6


def _longest_contraction(layers, in_shape, batch):
    """Largest K over the stack's forward, input-gradient and weight-gradient
    GEMMs."""
    from paper_1812_10624_b200.tensor_core import (Concat, Conv2d, FullyConnected, Residual,
                                                    out_shape)
    shape, kmax = tuple(in_shape), 1
    for l in layers:
        nxt = out_shape(l, shape)
        if isinstance(l, Residual):
            kmax = max(kmax, _longest_contraction(l.body, shape, batch),
                       _longest_contraction(l.shortcut, shape, batch))
        elif isinstance(l, Concat):
            kmax = max([kmax] + [_longest_contraction(br, shape, batch) for br in l.branches])
        elif isinstance(l, FullyConnected):
            kmax = max(kmax, l.in_dim, l.out_dim, batch)
        elif isinstance(l, Conv2d):
            kk = l.kh * l.kw
            kmax = max(kmax, l.in_ch * kk, l.out_ch * kk, batch * nxt[1] * nxt[2])
        shape = nxt
    return kmax


TIE = 1e-5   # |pre-activation| <= TIE * max|.|: a ReLU decision fp32 rounding may flip


def _device_act(eng, i):
    """Op i's output on the device, in the oracle's layout (rows / NCHW)."""
    a = eng._act(i)
    f = a.to_float()
    if a.layout == "rows":
        return f[:, :a.logical].cpu().numpy()
    return f[..., :a.logical].permute(0, 3, 1, 2).cpu().numpy()


def _oracle_forward_tie_aware(tl, params, x, dev_pos):
    """orc.block_forward, layer by layer, except that a ReLU whose
    pre-activation is within TIE of zero takes the device's decision: both
    sides are correct to fp32 rounding there, and one flipped unit would
    otherwise perturb a whole weight-gradient row far beyond TOL."""
    caches = []
    for i, (layer, p) in enumerate(zip(tl, params)):
        z = x
        x, c = orc.block_forward([layer], [p], x)
        c = c[0]
        if layer[0] == "relu":
            tie = np.abs(z) <= TIE * float(np.abs(z).max())
            if tie.any():
                c = np.where(tie, dev_pos[i], c)
        caches.append(c)
    return x, caches


def _bn_fed_biases(layers):
    """(layer, tensor) positions of conv biases that feed a BatchNorm, inside
    residual rows too (tensor index within the row)."""
    from paper_1812_10624_b200.tensor_core import (BatchNorm2d, Concat, Conv2d, Residual,
                                                    param_shapes)
    out = set()

    def scan(seq, li, t0):
        t = t0
        for j, l in enumerate(seq):
            if isinstance(l, Concat):
                for br in l.branches:
                    t = scan(br, li, t)
                continue
            if isinstance(l, Conv2d) and j + 1 < len(seq) and isinstance(seq[j + 1], BatchNorm2d):
                out.add((li, t + 1))
            t += len(param_shapes(l))
        return t
    for li, l in enumerate(layers):
        if isinstance(l, Residual):
            scan(l.shortcut, li, scan(l.body, li, 0))
        elif isinstance(l, Concat):
            t = 0
            for br in l.branches:
                t = scan(br, li, t)
        elif isinstance(l, Conv2d) and li + 1 < len(layers) and \
                isinstance(layers[li + 1], BatchNorm2d):
            out.add((li, 1))
    return out


def _run(layers, in_shape, batch, need_input_grad, seed):
    from paper_1812_10624_b200.tensor_core import Conv2d, FullyConnected
    from paper_1812_10624_b200.tensor_core import Concat, Residual

    def _depth(seq):
        return sum(_depth(l.body) + _depth(l.shortcut) if isinstance(l, Residual)
                   else max(_depth(b) for b in l.branches) if isinstance(l, Concat)
                   else isinstance(l, (Conv2d, FullyConnected)) for l in seq)
    depth = max(1, _depth(layers))
    tol = gemm_tol(_longest_contraction(layers, in_shape, batch))
    from paper_1812_10624_b200.engine import BlockEngine
    from paper_1812_10624_b200.tensor_core import as_tuple, seeded_init
    params = seeded_init(layers, seed)
    eng = BlockEngine(layers, in_shape, batch, "cuda:0", params,
                      need_input_grad=need_input_grad)
    rng = np.random.Generator(np.random.PCG64(seed))
    x = rng.standard_normal((batch, *in_shape)).astype(np.float32)
    out = eng.forward(torch.from_numpy(x).cuda())
    dev_pos = {i: _device_act(eng, i) > 0 for i, l in enumerate(layers) if type(l).__name__ == "ReLU"}
    oshape = eng.out_shape
    gy = rng.standard_normal((batch, *oshape)).astype(np.float32)
    # feed gy in the engine's layout: rows for a flat output
    from paper_1812_10624_b200 import _lib
    from paper_1812_10624_b200.engine import Split, rup8
    from paper_1812_10624_b200.tensor_core import ptr, stream_of
    if out.layout == "rows":
        g = Split.alloc("rows", (batch, rup8(oshape[0])), oshape[0], "cuda:0")
        _lib.call("stzx_pack_rows", ptr(torch.from_numpy(gy).cuda()), g.ptr(), g.ps, batch,
                  oshape[0], g.width, stream_of(torch.device("cuda:0")))
        got = out.to_float()[:, :oshape[0]]
    else:
        c, h, w = oshape
        g = Split.alloc("nhwc", (batch, h, w, rup8(c)), c, "cuda:0")
        _lib.call("stzx_pack_nchw", ptr(torch.from_numpy(gy).cuda()), g.ptr(), g.ps, batch, c, h,
                  w, g.width, stream_of(torch.device("cuda:0")))
        got = out.to_float()[..., :c].permute(0, 3, 1, 2)
    gin = eng.backward(g)
    torch.cuda.synchronize()
    tl = [as_tuple(l) for l in layers]
    ry, caches = _oracle_forward_tie_aware(tl, params, x, dev_pos)
    rgx, rgrads = orc.block_backward(tl, params, caches, gy)
    assert orc.rel_err(got.cpu().numpy(), ry) <= tol
    noise = _bn_fed_biases(layers)
    for li, (gl, rl) in enumerate(zip(eng.grads, rgrads)):
        for ti, (a, b) in enumerate(zip(gl, rl)):
            if (li, ti) in noise:
                # a conv bias feeding a BatchNorm: its true gradient is 0 (BN
                # removes any per-channel shift), both sides hold rounding noise
                scale = max(float(np.abs(r).max()) for r in rl)
                assert float(np.abs(a.cpu().numpy()).max()) <= 1e-4 * scale, f"layer {li}.{ti}"
                continue
            assert orc.rel_err(a.cpu().numpy(), b) <= tol, f"layer {li}.{ti}"
    if need_input_grad:
        if len(in_shape) == 1:
            got_gx = gin.to_float()[:, :in_shape[0]]
        else:
            c, h, w = in_shape
            got_gx = gin.to_float()[..., :c].permute(0, 3, 1, 2)
        assert orc.rel_err(got_gx.cpu().numpy(), rgx) <= tol * depth
    return eng


def test_alexnet_conv1_space_to_depth(clusters):
    from paper_1812_10624_b200.tensor_core import Conv2d, MaxPool2d, ReLU
    eng = _run([Conv2d(3, 64, 11, 4, 2), ReLU(), MaxPool2d(3, 2)], (3, 224, 224), 2, False, 1)
    assert eng.ops[0].s2d == (3, 64, 57, 57)


@pytest.mark.parametrize("side", [64, 224], ids=["64px", "224px"])
def test_resnet_stem_space_to_depth(clusters, side):
    """ResNet-50's 7x7/2 stem as a stride-1 4x4 conv over 2x2 space-to-depth
    blocks (12 real of 32 channels)."""
    from paper_1812_10624_b200.tensor_core import Conv2d, MaxPool2d, ReLU
    eng = _run([Conv2d(3, 64, 7, 2, 3), ReLU(), MaxPool2d(3, 2)], (3, side, side), 2, False, 1)
    assert eng.ops[0].s2d == (4, 32, side // 2 + 3, side // 2 + 3)


def test_alexnet_conv2_to_pool_tma(clusters):
    from paper_1812_10624_b200.tensor_core import Conv2d, MaxPool2d, ReLU
    _run([Conv2d(64, 192, 5, 1, 2), ReLU(), MaxPool2d(3, 2)], (64, 27, 27), 2, True, 2)


def test_alexnet_conv5_pool_flatten_boundary(clusters):
    from paper_1812_10624_b200.tensor_core import Conv2d, Flatten, MaxPool2d, ReLU
    _run([Conv2d(256, 256, 3, 1, 1), ReLU(), MaxPool2d(3, 2), Flatten()], (256, 13, 13), 3, True,
         3)


def test_vgg_stage_conv_conv_pool(clusters):
    from paper_1812_10624_b200.tensor_core import Conv2d, MaxPool2d, ReLU
    _run([Conv2d(64, 128, 3, 1, 1), ReLU(), Conv2d(128, 128, 3, 1, 1), ReLU(), MaxPool2d(2, 2)],
         (64, 28, 28), 2, True, 4)


def test_flatten_without_pool_relayout():
    from paper_1812_10624_b200.tensor_core import Conv2d, Flatten, FullyConnected, ReLU
    _run([Conv2d(8, 16, 3, 1, 1), ReLU(), Flatten(), FullyConnected(16 * 6 * 6, 24), ReLU()],
         (8, 6, 6), 4, True, 5)


def test_fc_head_alexnet_shapes(clusters):
    """FC head at the 7:1 FC worker's batch (M = 896): fc 9216->4096->4096->1000."""
    from paper_1812_10624_b200.tensor_core import FullyConnected, ReLU
    _run([FullyConnected(9216, 4096), ReLU(), FullyConnected(4096, 4096), ReLU(),
          FullyConnected(4096, 1000)], (9216,), 896, True, 6)


@pytest.mark.parametrize("schedule", ["accumulate", "dgrad_then_wgrad"])
def test_micro_batches_match_full_batch(schedule):
    """Micro-batched passes (the pipelined step's building blocks) give the
    full-batch results: forward rows, per-micro-batch backward with gradient
    accumulation, or the FC worker's dgrad-per-micro-batch then one
    full-batch wgrad.  Sums differ only in fp32 order."""
    from paper_1812_10624_b200.engine import BlockEngine, Split, rup8
    from paper_1812_10624_b200.tensor_core import (Conv2d, Flatten, FullyConnected, MaxPool2d,
                                                    ReLU, seeded_init)
    from paper_1812_10624_b200 import _lib
    from paper_1812_10624_b200.tensor_core import ptr, stream_of
    layers = [Conv2d(16, 32, 3, 1, 1), ReLU(), MaxPool2d(2, 2), Flatten(),
              FullyConnected(32 * 4 * 4, 40), ReLU(), FullyConnected(40, 24)]
    batch, m = 8, 4
    kb = batch // m
    params = seeded_init(layers, 9)
    rng = np.random.Generator(np.random.PCG64(9))
    x = torch.from_numpy(rng.standard_normal((batch, 16, 8, 8)).astype(np.float32)).cuda()
    gy_h = rng.standard_normal((batch, 24)).astype(np.float32)

    def run(micro):
        eng = BlockEngine(layers, (16, 8, 8), batch, "cuda:0", params, need_input_grad=True)
        g = Split.alloc("rows", (batch, rup8(24)), 24, "cuda:0")
        _lib.call("stzx_pack_rows", ptr(torch.from_numpy(gy_h).cuda()), g.ptr(), g.ps, batch, 24,
                  g.width, stream_of(torch.device("cuda:0")))
        if not micro:
            out = eng.forward(x).to_float()
            gin = eng.backward(g).to_float()
        else:
            outs, gins = [], []
            for j in range(m):
                outs.append(eng.forward(x, rows=(j * kb, (j + 1) * kb)).to_float())
            for j in range(m):
                rows = (j * kb, (j + 1) * kb)
                if schedule == "accumulate":
                    gins.append(eng.backward(g, rows=rows, accumulate=j > 0).to_float())
                else:
                    gins.append(eng.backward(g, rows=rows, phase="dgrad").to_float())
            if schedule == "dgrad_then_wgrad":
                eng.backward(phase="wgrad")
            out, gin = torch.cat(outs), torch.cat(gins)
        torch.cuda.synchronize()
        return out.cpu().numpy(), gin.cpu().numpy(), eng.grad_flat.cpu().numpy()

    full, micro = run(False), run(True)
    for a, b in zip(full, micro):
        assert orc.rel_err(b, a) <= 1e-6


# -- ResNet-trunk kinds (oracle-defined, parity unpinned) --------

RESNET_STRIDED = [  # (layers factory, in_shape, batch): ResNet-50 stage-4 shapes at 64x64
    ("proj1x1s2", lambda m: [m.Conv2d(1024, 2048, 1, 2)], (1024, 4, 4), 2),
    ("proj1x1s2_relu_in", lambda m: [m.Conv2d(64, 256, 3, 1, 1), m.ReLU(), m.Conv2d(256, 512, 1, 2)],
     (64, 15, 15), 2),
    ("c3x3s2", lambda m: [m.Conv2d(512, 512, 3, 2, 1)], (512, 4, 4), 2),
    ("c3x3s2_c64", lambda m: [m.Conv2d(64, 64, 3, 2, 1)], (64, 16, 16), 2),
    ("c1x1_reduce", lambda m: [m.Conv2d(256, 64, 1)], (256, 14, 14), 2),
    ("c1x1_expand_relu", lambda m: [m.Conv2d(64, 256, 1), m.ReLU(), m.Conv2d(256, 64, 1)],
     (64, 28, 28), 2),
    ("bn_relu", lambda m: [m.BatchNorm2d(256), m.ReLU()], (256, 7, 7), 4),
    ("bn_large", lambda m: [m.BatchNorm2d(64)], (64, 56, 56), 2),
    ("gap_flatten", lambda m: [m.GlobalAvgPool2d(), m.Flatten()], (2048, 2, 2), 3),
]


@pytest.mark.parametrize("case", RESNET_STRIDED, ids=lambda c: c[0])
def test_resnet_pieces(case):
    from paper_1812_10624_b200 import tensor_core as m
    _, make, shape, batch = case
    _run(make(m), shape, batch, True, 7)


def test_resnet_stage4_first_block():
    from paper_1812_10624_b200 import tensor_core as m
    body = (m.Conv2d(1024, 512, 1), m.BatchNorm2d(512), m.ReLU(), m.Conv2d(512, 512, 3, 2, 1),
            m.BatchNorm2d(512), m.ReLU(), m.Conv2d(512, 2048, 1), m.BatchNorm2d(2048))
    short = (m.Conv2d(1024, 2048, 1, 2), m.BatchNorm2d(2048))
    _run([m.Residual(body, short)], (1024, 4, 4), 2, True, 8)
