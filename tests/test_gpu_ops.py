"""Per-layer parity on the B200: the C-ABI kernels vs the reference's own
outputs (golden fixtures) and vs the CPU oracle on fresh seeded inputs.

Tolerances (rel_err = max|a-b| / max(|a|,|b|), the reference's own metric,
tests/oracles.py): conv / FC contractions run on the tcgen05 BF16x6 core
(fp32-class) against the reference's float64 accumulation; each is checked
at conftest.gemm_tol(K) for its contraction length K (3e-6 up to K = 800,
half the worst-case accumulator-truncation bound beyond).  Max-pool, ReLU
and SGD are bit-exact; the float64 softmax / bias-sum paths agree within
1e-7.
"""

import numpy as np
import pytest
import torch

import golden_io
import stanza_oracle as orc
from conftest import gemm_tol

pytestmark = pytest.mark.gpu

DEV = "cuda:0"
GEMM_TOL = 3e-6


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def host(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy()


@pytest.fixture(scope="module")
def ops():
    return golden_io.ops()


@pytest.fixture(scope="module")
def tc():
    from paper_1812_10624_b200 import tensor_core
    return tensor_core


@pytest.mark.parametrize("case", ["c3s1p1", "c3s2p0", "c5s1p2", "c11s4p2", "c3s1p0_odd"])
def test_conv_golden(ops, tc, producer, case):
    g = ops[f"conv_{case}"]
    c, o, k, s, p = (int(v) for v in g["cfg"][:5])
    layer = tc.Conv2d(c, o, k, s, p)
    params = [dev(g["w"]), dev(g["b"])]
    y, cache = tc.forward(layer, params, dev(g["x"]))
    assert orc.rel_err(host(y), g["y"]) <= GEMM_TOL
    gx, (gw, gb) = tc.backward(layer, params, cache, dev(g["gy"]))
    assert orc.rel_err(host(gx), g["gx"]) <= GEMM_TOL
    assert orc.rel_err(host(gw), g["gw"]) <= GEMM_TOL
    assert orc.rel_err(host(gb), g["gb"]) <= 1e-7


@pytest.mark.parametrize("case", ["p2s2", "p3s2", "p3s2_ties"])
def test_maxpool_golden_bit_exact(ops, tc, case):
    g = ops[f"pool_{case}"]
    k, s = (int(v) for v in g["cfg"])
    layer = tc.MaxPool2d(k, s)
    y, cache = tc.forward(layer, [], dev(g["x"]))
    np.testing.assert_array_equal(host(y), g["y"])
    np.testing.assert_array_equal(host(cache[0]), g["arg"])
    gx, _ = tc.backward(layer, [], cache, dev(g["gy"]))
    np.testing.assert_array_equal(host(gx), g["gx"])


@pytest.mark.parametrize("case", ["fc_small", "fc_mid"])
def test_fc_golden(ops, tc, producer, case):
    g = ops[case]
    i, o = g["w"].shape
    layer = tc.FullyConnected(i, o)
    params = [dev(g["w"]), dev(g["b"])]
    y, cache = tc.forward(layer, params, dev(g["x"]))
    assert orc.rel_err(host(y), g["y"]) <= GEMM_TOL
    gx, (gw, gb) = tc.backward(layer, params, cache, dev(g["gy"]))
    assert orc.rel_err(host(gx), g["gx"]) <= GEMM_TOL
    assert orc.rel_err(host(gw), g["gw"]) <= GEMM_TOL
    assert orc.rel_err(host(gb), g["gb"]) <= 1e-7


@pytest.mark.parametrize("case", ["ce_10", "ce_1000"])
def test_softmax_ce_golden(ops, tc, case):
    g = ops[case]
    layer = tc.SoftmaxCrossEntropy()
    loss, cache = tc.forward(layer, [], dev(g["z"]), labels=g["labels"])
    gz, _ = tc.backward(layer, [], cache, None)
    assert orc.rel_err(host(loss), g["loss"]) <= 1e-7
    assert orc.rel_err(host(gz), g["g"]) <= 1e-7


def test_sgd_golden_bit_exact(ops, tc):
    g = ops["sgd"]
    w, v = dev(g["w"]), dev(g["v"])
    opt = tc.OptimizerState(lr=float(g["lr"]), momentum=float(g["mu"]), velocity=[[v]])
    tc.sgd_step([[w]], [[dev(g["g"])]], int(g["n"]), opt)
    np.testing.assert_array_equal(host(w), g["w1"])
    np.testing.assert_array_equal(host(v), g["v1"])


def test_relu_kat(tc):
    x = dev(np.array([[-1.0, 0.0, 2.0]], np.float32))
    y, cache = tc.forward(tc.ReLU(), [], x)
    np.testing.assert_array_equal(host(y), [[0.0, 0.0, 2.0]])
    gx, _ = tc.backward(tc.ReLU(), [], cache, torch.ones_like(x))
    np.testing.assert_array_equal(host(gx), [[0.0, 0.0, 1.0]])


def test_hand_arithmetic(tc):
    """Reference KATs (test_tensor_core.py:46-70) through the CUDA path."""
    layer = tc.Conv2d(1, 1, 2)
    y, _ = tc.forward(layer, [dev(np.array([[[[1.0, 0.0], [0.0, 1.0]]]], np.float32)),
                              dev(np.array([0.5], np.float32))],
                      dev(np.array([[[[1.0, 2.0], [3.0, 4.0]]]], np.float32)))
    assert host(y)[0, 0, 0, 0] == pytest.approx(5.5)
    fc = tc.FullyConnected(2, 2)
    y, _ = tc.forward(fc, [dev(np.array([[1.0, 2.0], [3.0, 4.0]], np.float32)),
                           dev(np.array([0.5, -0.5], np.float32))],
                      dev(np.array([[1.0, 1.0]], np.float32)))
    np.testing.assert_allclose(host(y), [[4.5, 5.5]])
    y, _ = tc.forward(tc.MaxPool2d(2, 2), [],
                      dev(np.arange(16, dtype=np.float32).reshape(1, 1, 4, 4)))
    np.testing.assert_array_equal(host(y)[0, 0], [[5, 7], [13, 15]])


CONV_SHAPES = [  # (N, C, H, W, O, k, s, p) incl. AlexNet-like layer shapes at small batch
    (2, 3, 35, 35, 16, 11, 4, 2),
    (2, 64, 27, 27, 192, 5, 1, 2),
    (2, 192, 13, 13, 384, 3, 1, 1),
    (1, 384, 13, 13, 256, 3, 1, 1),
    (3, 5, 9, 7, 33, 3, 2, 1),
    (1, 3, 224, 224, 64, 11, 4, 2),
    (2, 64, 13, 13, 128, 3, 1, 1),
    (2, 128, 9, 9, 192, 3, 1, 1),
    (1, 256, 6, 6, 40, 3, 1, 1),
    (2, 32, 12, 12, 64, 3, 2, 1),
]


@pytest.mark.parametrize("shape", CONV_SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_conv_vs_oracle(tc, producer, clusters, shape):
    _conv_case(tc, shape)


STRIDED_CONV_SHAPES = [  # input gradient as s*s phase sub-convolutions (O8 % 32 == 0)
    (2, 64, 56, 56, 128, 3, 2, 1), (2, 32, 15, 15, 64, 3, 2, 1), (1, 32, 14, 13, 96, 5, 2, 2),
    (2, 64, 17, 17, 32, 3, 2, 0), (1, 48, 20, 20, 64, 7, 3, 3), (2, 32, 11, 11, 64, 2, 2, 0),
    (1, 32, 10, 10, 64, 2, 3, 0), (1, 40, 23, 23, 64, 7, 2, 3)]


@pytest.mark.parametrize("shape", STRIDED_CONV_SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_strided_conv_phases_vs_oracle(tc, shape):
    _conv_case(tc, shape)


def _conv_case(tc, shape):
    n, c, h, w, o, k, s, p = shape
    rng = np.random.Generator(np.random.PCG64(hash(shape) & 0xFFFF))
    x = rng.standard_normal((n, c, h, w)).astype(np.float32)
    wt = (rng.standard_normal((o, c, k, k)) / np.sqrt(c * k * k)).astype(np.float32)
    b = rng.standard_normal(o).astype(np.float32)
    ry, xp = orc.conv_forward(x, wt, b, s, p)
    gy = rng.standard_normal(ry.shape).astype(np.float32)
    rgx, rgw, rgb = orc.conv_backward(xp, wt, gy, s, p)
    layer = tc.Conv2d(c, o, k, s, p)
    params = [dev(wt), dev(b)]
    y, cache = tc.forward(layer, params, dev(x))
    assert orc.rel_err(host(y), ry) <= gemm_tol(c * k * k)
    gx, (gw, gb) = tc.backward(layer, params, cache, dev(gy))
    assert orc.rel_err(host(gx), rgx) <= gemm_tol(o * k * k)
    assert orc.rel_err(host(gw), rgw) <= gemm_tol(n * ry.shape[2] * ry.shape[3])
    assert orc.rel_err(host(gb), rgb) <= 1e-7


FC_SHAPES = [(8, 256, 128), (8, 128, 10), (128, 9216, 512), (896, 4096, 1000), (100, 200, 300),
             (5, 11, 7), (33, 1024, 4096)]


@pytest.mark.parametrize("shape", FC_SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_fc_vs_oracle(tc, producer, clusters, shape):
    _fc_case(tc, shape)


def _fc_case(tc, shape):
    m, i, o = shape
    rng = np.random.Generator(np.random.PCG64(m * 7919 + i * 31 + o))
    x = rng.standard_normal((m, i)).astype(np.float32)
    w = (rng.standard_normal((i, o)) / np.sqrt(i)).astype(np.float32)
    b = rng.standard_normal(o).astype(np.float32)
    gy = rng.standard_normal((m, o)).astype(np.float32)
    layer = tc.FullyConnected(i, o)
    params = [dev(w), dev(b)]
    y, cache = tc.forward(layer, params, dev(x))
    assert orc.rel_err(host(y), orc.fc_forward(x, w, b)) <= gemm_tol(i)
    gx, (gw, gb) = tc.backward(layer, params, cache, dev(gy))
    rgx, rgw, rgb = orc.fc_backward(x, w, gy)
    assert orc.rel_err(host(gx), rgx) <= gemm_tol(o)
    assert orc.rel_err(host(gw), rgw) <= gemm_tol(m)
    assert orc.rel_err(host(gb), rgb) <= 1e-7


@pytest.mark.parametrize("k,s,shape", [(3, 2, (4, 64, 55, 55)), (2, 2, (2, 8, 16, 16)),
                                       (3, 2, (2, 256, 13, 13)), (3, 2, (2, 16, 56, 57)),
                                       (2, 2, (3, 8, 17, 15)), (3, 2, (2, 192, 27, 27))])
def test_maxpool_vs_oracle_bit_exact(tc, k, s, shape):
    rng = np.random.Generator(np.random.PCG64(k * 100 + shape[1]))
    x = rng.standard_normal(shape).astype(np.float32)
    ry, arg = orc.maxpool_forward(x, k, s)
    gy = rng.standard_normal(ry.shape).astype(np.float32)
    rgx = orc.maxpool_backward(arg, x.shape, gy, k, s)
    y, cache = tc.forward(tc.MaxPool2d(k, s), [], dev(x))
    np.testing.assert_array_equal(host(y), ry)
    gx, _ = tc.backward(tc.MaxPool2d(k, s), [], cache, dev(gy))
    np.testing.assert_array_equal(host(gx), rgx)


@pytest.mark.parametrize("shape", [(2, 64, 55, 55), (2, 24, 27, 27)])
def test_maxpool_backward_shared_maxima_bit_exact(tc, shape):
    """3x3/2 pooling with a spike on every (even, even) pixel: each spike is
    the argmax of up to four overlapping windows, so most gradient cells sum
    three or four contributions (the float64 re-sum of the tiled kernel)."""
    rng = np.random.Generator(np.random.PCG64(shape[1] * 7 + shape[2]))
    x = rng.standard_normal(shape).astype(np.float32)
    x[:, :, ::2, ::2] += 8.0
    ry, arg = orc.maxpool_forward(x, 3, 2)
    gy = (rng.standard_normal(ry.shape) * np.exp2(rng.integers(-30, 30, ry.shape))).astype(
        np.float32)
    rgx = orc.maxpool_backward(arg, x.shape, gy, 3, 2)
    y, cache = tc.forward(tc.MaxPool2d(3, 2), [], dev(x))
    np.testing.assert_array_equal(host(y), ry)
    gx, _ = tc.backward(tc.MaxPool2d(3, 2), [], cache, dev(gy))
    np.testing.assert_array_equal(host(gx), rgx)


TILE_CONFIGS = [(64, 1, 1), (96, 1, 1), (128, 1, 1), (192, 1, 1), (128, 2, 1), (192, 2, 1),
                (256, 2, 1), (64, 1, 3), (128, 2, 4), (192, 1, 2), (256, 2, 5)]


@pytest.fixture(params=TILE_CONFIGS, ids=lambda t: "bn%d-cl%d-sp%d" % t)
def tile(request, lib):
    """Force every (width, pair, split-K) configuration the cost model can pick."""
    assert lib.stz_set_tile(*request.param) == 0
    yield request.param
    lib.stz_set_tile(0, 0, 0)


@pytest.fixture(params=[1, 0], ids=["fixup", "reduce-pass"])
def fixup(request, lib):
    """Split-K sums in the GEMM (last split of each tile) or in a separate pass."""
    lib.stz_set_fixup(request.param)
    yield request.param
    lib.stz_set_fixup(0)


@pytest.mark.parametrize("shape", [(300, 640, 1000), (896, 1024, 384), (257, 200, 96)],
                         ids=lambda s: "x".join(map(str, s)))
def test_fc_every_tile_config(tc, tile, fixup, shape):
    _fc_case(tc, shape)


@pytest.mark.parametrize("shape", [(2, 64, 13, 13, 384, 3, 1, 1), (3, 96, 9, 9, 256, 3, 1, 1),
                                   (2, 32, 15, 15, 192, 5, 1, 2)],
                         ids=lambda s: "x".join(map(str, s)))
def test_conv_every_tile_config(tc, tile, fixup, shape):
    _conv_case(tc, shape)


VALID_CONV_SHAPES = [  # stride 1: the shifted-window (band) path, forward and input gradient
    (2, 64, 15, 15, 64, 3, 1, 0), (2, 32, 20, 17, 192, 5, 1, 0), (1, 64, 57, 57, 64, 3, 1, 0),
    (3, 96, 9, 11, 128, 3, 1, 0), (2, 32, 8, 8, 40, 1, 1, 0), (1, 64, 31, 31, 64, 5, 1, 0),
    (2, 64, 27, 27, 64, 5, 1, 2), (2, 192, 13, 13, 64, 3, 1, 1), (1, 32, 20, 21, 48, 3, 1, 1),
    (2, 96, 15, 15, 32, 5, 1, 2), (1, 256, 9, 9, 64, 5, 1, 2)]


@pytest.fixture(params=[1, 2, 0], ids=["band", "band-padded", "im2col"])
def band(request, lib):
    """Run with the shifted-window conv (unpadded only / padded too) and with
    the im2col GEMM; restore the default after."""
    lib.stz_set_band(request.param)
    yield request.param
    lib.stz_set_band(1)


@pytest.mark.parametrize("shape", VALID_CONV_SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_valid_conv_band_vs_oracle(tc, band, shape):
    _conv_case(tc, shape)


@pytest.fixture(params=[(64, 1, 1), (64, 1, 3)], ids=["bn64-sp1", "bn64-sp3"])
def halves(request, lib):
    """Thin tiles as two 128-row halves per CTA (stz_set_mh(2)): one 256-row A
    box, one B stage shared by both halves' TMEM accumulators."""
    assert lib.stz_set_tile(*request.param) == 0
    assert lib.stz_set_mh(2) == 0
    yield request.param
    lib.stz_set_mh(0)
    lib.stz_set_tile(0, 0, 0)


@pytest.mark.parametrize("shape", [(2, 64, 27, 27, 192, 5, 1, 2), (2, 64, 13, 13, 64, 3, 1, 1),
                                   (3, 96, 9, 9, 40, 3, 1, 1), (1, 3, 224, 224, 64, 11, 4, 2)],
                         ids=lambda s: "x".join(map(str, s)))
def test_conv_two_halves(tc, producer, halves, shape):
    _conv_case(tc, shape)


@pytest.mark.parametrize("shape", [(300, 640, 64), (896, 1024, 40), (257, 200, 96)],
                         ids=lambda s: "x".join(map(str, s)))
def test_fc_two_halves(tc, producer, halves, shape):
    _fc_case(tc, shape)


@pytest.mark.parametrize("shapes", [
    [(64, 3, 7, 7, 8, 64), (256, 64, 1, 1, 64, 256), (128, 128, 3, 3, 128, 128)],
    [(33, 5, 3, 3, 8, 40), (40, 70, 1, 7, 72, 40), (1000, 48, 5, 5, 48, 1000)],
    [(16, 3, 11, 11, 8, 32), (64, 17, 7, 1, 24, 64)]], ids=["resnet", "ragged", "wide-taps"])
def test_pack_conv_w_multi_matches_single(lib, shapes):
    """The tiled multi-job weight pack writes exactly what the per-layer pack
    writes (forward and flipped input-gradient operands, padded channels 0)."""
    from paper_1812_10624_b200 import _lib
    rng = np.random.Generator(np.random.PCG64(len(shapes)))
    jobs, outs = [], []
    for o, c, kh, kw, c8, o8 in shapes:
        w = torch.tensor(rng.standard_normal((o, c, kh, kw)).astype(np.float32), device="cuda")
        kk = kh * kw
        wf = torch.full((3, o * kk * c8), 7, dtype=torch.int16, device="cuda")
        wd = torch.full((3, c * kk * o8), 7, dtype=torch.int16, device="cuda")
        rf, rd = wf.clone(), wd.clone()
        _lib.call("stzx_pack_conv2_w", w.data_ptr(), rf.data_ptr(), rf.shape[1], rd.data_ptr(),
                  rd.shape[1], o, c, kh, kw, c8, o8, None)
        jobs.append(_lib.ConvPack(w.data_ptr(), wf.data_ptr(), wd.data_ptr(), wf.shape[1],
                                  wd.shape[1], o, c, kh, kw, c8, o8))
        outs.append((w, wf, wd, rf, rd))
    arr = (_lib.ConvPack * len(jobs))(*jobs)
    _lib.call("stzx_pack_conv_w_multi", arr, len(jobs), None)
    torch.cuda.synchronize()
    for w, wf, wd, rf, rd in outs:
        assert torch.equal(wf, rf)
        assert torch.equal(wd, rd)


@pytest.mark.parametrize("accumulate", [0, 1], ids=["batch", "accumulate"])
@pytest.mark.parametrize("shape", [(128, 1024, 1000), (37, 200, 96), (256, 640, 4096),
                                   (128, 9216, 512)], ids=lambda s: "x".join(map(str, s)))
def test_fc_wgrad_sgd_matches_unfused(lib, shape, accumulate):
    """The momentum step in the FC weight-gradient epilogue (one FC worker)
    leaves w, v, the split-plane copy and the bias exactly as the unfused
    weight gradient followed by the flat-block update."""
    from paper_1812_10624_b200 import _lib
    m, i, o = shape
    i8, o8 = -(-i // 8) * 8, -(-o // 8) * 8
    rng = np.random.Generator(np.random.PCG64(m + i + o + accumulate))
    t = lambda *s: torch.tensor(rng.standard_normal(s).astype(np.float32), device=DEV)
    x, g = t(m, i), t(m, o)
    xp = torch.zeros((3, m, i8), dtype=torch.bfloat16, device=DEV)
    gp = torch.zeros((3, m, o8), dtype=torch.bfloat16, device=DEV)
    _lib.call("stzx_pack_rows", x.data_ptr(), xp.data_ptr(), xp[0].numel(), m, i, i8, None)
    _lib.call("stzx_pack_rows", g.data_ptr(), gp.data_ptr(), gp[0].numel(), m, o, o8, None)
    w, v, wb, vb = t(i, o), t(i, o), t(o), t(o)
    gw0, gb0 = t(i, o), t(o)
    lr, mu, n = 0.05, 0.9, m
    from paper_1812_10624_b200.tensor_core import inv_batch
    ws = torch.empty(256 << 20, dtype=torch.uint8, device=DEV)

    # unfused: gradient, then the update with the fused plane repack
    gw, gb = (gw0.clone(), gb0.clone()) if accumulate else (torch.zeros_like(gw0),
                                                           torch.zeros_like(gb0))
    w1, v1, wb1, vb1 = w.clone(), v.clone(), wb.clone(), vb.clone()
    p1 = torch.zeros((3, i, o8), dtype=torch.bfloat16, device=DEV)
    _lib.call("stzx_fc_wgrad", xp.data_ptr(), xp[0].numel(), gp.data_ptr(), gp[0].numel(),
              gw.data_ptr(), gb.data_ptr(), accumulate, m, i, i8, o, o8, ws.data_ptr(),
              ws.numel(), None)
    rs = _lib.range_array([(0, i * o, p1.data_ptr(), p1[0].numel(), o, o8)])
    _lib.call("stz_sgd_momentum_pack", w1.data_ptr(), v1.data_ptr(), gw.data_ptr(), i * o, lr,
              mu, inv_batch(n), rs, 1, None)
    _lib.call("stz_sgd_momentum_pack", wb1.data_ptr(), vb1.data_ptr(), gb.data_ptr(), o, lr, mu,
              inv_batch(n), _lib.range_array([]), 0, None)

    # fused
    w2, v2, wb2, vb2 = w.clone(), v.clone(), wb.clone(), vb.clone()
    gw2, gb2 = gw0.clone(), gb0.clone()
    p2 = torch.zeros_like(p1)
    _lib.call("stzx_fc_wgrad_sgd", xp.data_ptr(), xp[0].numel(), gp.data_ptr(), gp[0].numel(),
              w2.data_ptr(), v2.data_ptr(), p2.data_ptr(), p2[0].numel(), wb2.data_ptr(),
              vb2.data_ptr(), gw2.data_ptr(), gb2.data_ptr(), accumulate, m, i, i8, o, o8, lr,
              mu, inv_batch(n), ws.data_ptr(), ws.numel(), None)
    torch.cuda.synchronize()
    for a, b in [(w1, w2), (v1, v2), (wb1, wb2), (vb1, vb2), (gb, gb2)]:
        assert torch.equal(a, b)
    assert torch.equal(p1.view(torch.int16), p2.view(torch.int16))
    assert torch.equal(gw2, gw0)          # the weight gradient itself is never stored


@pytest.mark.parametrize("shape", [(387200, 64), (128, 4096), (37, 1000), (1000, 13)],
                         ids=lambda s: "x".join(map(str, s)))
def test_colsum_matches_wgrad_bias(lib, shape):
    """stzx_colsum (the bias gradient issued on its own stream) writes exactly
    the column sums the weight-gradient entry writes (float64, fixed order),
    and accumulates like it."""
    from paper_1812_10624_b200 import _lib
    r, n = shape
    n8 = -(-n // 8) * 8
    rng = np.random.Generator(np.random.PCG64(r + n))
    g = torch.tensor(rng.standard_normal((r, n)).astype(np.float32), device=DEV)
    gp = torch.zeros((3, r, n8), dtype=torch.bfloat16, device=DEV)
    _lib.call("stzx_pack_rows", g.data_ptr(), gp.data_ptr(), gp[0].numel(), r, n, n8, None)
    ws = torch.empty(64 << 20, dtype=torch.uint8, device=DEV)
    ref = np.asarray(g.cpu().numpy(), np.float64).sum(axis=0).astype(np.float32)
    out = torch.full((n,), 0.5, device=DEV)
    _lib.call("stzx_colsum", gp.data_ptr(), gp[0].numel(), r, n, n8, out.data_ptr(), 0,
              ws.data_ptr(), ws.numel(), None)
    assert orc.rel_err(host(out), ref) <= 1e-7
    x = torch.zeros((r, 8), device=DEV)
    xp = torch.zeros((3, r, 8), dtype=torch.bfloat16, device=DEV)
    gw = torch.zeros((8, n), device=DEV)
    gb = torch.zeros((n,), device=DEV)
    _lib.call("stzx_fc_wgrad", xp.data_ptr(), xp[0].numel(), gp.data_ptr(), gp[0].numel(),
              gw.data_ptr(), gb.data_ptr(), 0, r, 8, 8, n, n8, ws.data_ptr(), ws.numel(), None)
    assert torch.equal(out, gb)
    _lib.call("stzx_colsum", gp.data_ptr(), gp[0].numel(), r, n, n8, out.data_ptr(), 1,
              ws.data_ptr(), ws.numel(), None)
    torch.cuda.synchronize()
    assert torch.equal(out, gb + gb)
