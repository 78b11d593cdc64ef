"""Inception-V3 kinds, CPU side: the oracle's
asymmetric conv, padded average pool and channel concat against finite
differences and against independent formulations (the reference has no such
kinds, so the oracle is checked against calculus, not reference outputs),
and the host-side specs (shapes, init order, partition)."""

import numpy as np
import pytest

import stanza_oracle as orc

F64 = np.float64


def _fd(f, x, g, idx, eps=1e-3, tol=2e-2):
    for i in idx:
        xp, xm = x.copy(), x.copy()
        xp.flat[i] += eps
        xm.flat[i] -= eps
        num = (f(xp) - f(xm)) / (2 * eps)
        assert abs(num - g.flat[i]) <= tol * max(1.0, abs(num)), (i, num, g.flat[i])


@pytest.mark.parametrize("k,p", [((1, 7), (0, 3)), ((7, 1), (3, 0)), ((1, 3), (0, 1)),
                                 ((3, 1), (1, 0)), ((2, 5), (1, 2))])
def test_rect_conv_matches_square_embedding_and_fd(k, p):
    """A kh x kw conv equals the square conv whose kernel is zero outside
    the kh x kw window (with matching padding), and its backward matches
    finite differences."""
    rng = np.random.default_rng(3)
    kh, kw = k
    ph, pw = p
    x = rng.standard_normal((2, 4, 6, 7)).astype(np.float32)
    w = rng.standard_normal((5, 4, kh, kw)).astype(np.float32)
    b = rng.standard_normal(5).astype(np.float32)
    y, xp = orc.conv_forward(x, w, b, 1, (ph, pw))
    assert y.shape == (2, 5, 6 + 2 * ph - kh + 1, 7 + 2 * pw - kw + 1)
    # direct float64 reference
    xpad = np.pad(x.astype(F64), ((0, 0), (0, 0), (ph, ph), (pw, pw)))
    ref = np.zeros(y.shape, F64) + b.astype(F64)[None, :, None, None]
    for i in range(kh):
        for j in range(kw):
            ref += np.einsum("nchw,oc->nohw", xpad[:, :, i:i + y.shape[2], j:j + y.shape[3]],
                             w[:, :, i, j].astype(F64))
    np.testing.assert_allclose(y, ref.astype(np.float32), rtol=1e-6, atol=1e-6)
    gy = rng.standard_normal(y.shape).astype(np.float32)
    gx, gw, gb = orc.conv_backward(xp, w, gy, 1, (ph, pw))
    assert gx.shape == x.shape
    loss_x = lambda v: float((orc.conv_forward(v.astype(np.float32), w, b, 1, (ph, pw))[0]  # noqa
                              .astype(F64) * gy).sum())
    loss_w = lambda v: float((orc.conv_forward(x, v.astype(np.float32), b, 1, (ph, pw))[0]  # noqa
                              .astype(F64) * gy).sum())
    _fd(loss_x, x.astype(F64), gx, range(0, x.size, 13), eps=1e-2)
    _fd(loss_w, w.astype(F64), gw, range(0, w.size, 7), eps=1e-2)
    np.testing.assert_allclose(gb, gy.astype(F64).sum(axis=(0, 2, 3)), rtol=1e-6)


@pytest.mark.parametrize("k,s,p", [(3, 1, 1), (3, 2, 1), (2, 2, 0), (3, 2, 0)])
def test_avgpool_forward_backward(k, s, p):
    rng = np.random.default_rng(4)
    x = rng.standard_normal((2, 3, 7, 6)).astype(np.float32)
    y = orc.avgpool_forward(x, k, s, p)
    xpad = np.pad(x.astype(F64), ((0, 0), (0, 0), (p, p), (p, p)))
    oh, ow = y.shape[2], y.shape[3]
    ref = np.zeros(y.shape)
    for i in range(oh):
        for j in range(ow):
            ref[:, :, i, j] = xpad[:, :, i * s:i * s + k, j * s:j * s + k].sum(axis=(2, 3)) / (k * k)
    np.testing.assert_allclose(y, ref.astype(np.float32), rtol=1e-6)
    gy = rng.standard_normal(y.shape).astype(np.float32)
    gx = orc.avgpool_backward(x.shape, gy, k, s, p)
    # linear op: the backward is the exact transpose
    lhs = float((y.astype(F64) * gy).sum())
    rhs = float((x.astype(F64) * gx.astype(F64)).sum())
    assert abs(lhs - rhs) <= 1e-5 * max(1.0, abs(lhs))


def test_concat_block_backward_matches_finite_differences():
    """A module with four branches (1x1; 1x1 -> 1x3; avgpool -> 1x1; a nested
    concat of 1x3 / 3x1) on the same input."""
    br = ((("conv", 4, 3, 1, 1, 0),),
          (("conv", 4, 2, 1, 1, 0), ("relu",), ("conv", 2, 3, (1, 3), 1, (0, 1))),
          (("avgpool", 3, 1, 1), ("conv", 4, 2, 1, 1, 0)),
          (("concat", ((("conv", 4, 2, (1, 3), 1, (0, 1)),),
                       (("conv", 4, 2, (3, 1), 1, (1, 0)),))),))
    layers = [("concat", br)]
    assert orc.out_shape(layers[0], (4, 5, 5)) == (12, 5, 5)
    params = orc.seeded_init(layers, 7)
    assert [p.shape for p in params[0]] == [s for s in orc.param_shapes(layers[0])]
    rng = np.random.default_rng(5)
    x = rng.standard_normal((2, 4, 5, 5)).astype(np.float32)
    y, caches = orc.block_forward(layers, params, x)
    w = rng.standard_normal(y.shape).astype(np.float32)
    gx, grads = orc.block_backward(layers, params, caches, w)

    def loss_x(v):
        yy, _ = orc.block_forward(layers, params, v.astype(np.float32))
        return float((yy.astype(F64) * w).sum())
    _fd(loss_x, x.astype(F64), gx, range(0, x.size, 11), eps=1e-3, tol=5e-2)
    for ti in range(len(params[0])):
        t = params[0][ti]

        def loss_p(v, ti=ti):
            p2 = [list(params[0])]
            p2[0][ti] = v.astype(np.float32).reshape(t.shape)
            yy, _ = orc.block_forward(layers, p2, x)
            return float((yy.astype(F64) * w).sum())
        _fd(loss_p, t.astype(F64), grads[0][ti], range(0, t.size, max(1, t.size // 3)),
            eps=1e-3, tol=5e-2)


def test_inception_specs():
    from paper_1812_10624_b200 import model_partition as mp
    from paper_1812_10624_b200.tensor_core import as_tuple, out_shape, seeded_init
    full = mp.inception_v3()
    part = mp.split(full)
    assert part.boundary_activations == 2048 and part.fc_params == 2049 * 1000
    shape = full.input_shape
    seen = []
    for l in full.layers:
        shape = out_shape(l, shape)
        seen.append(shape)
    assert (192, 35, 35) in seen and (768, 17, 17) in seen and (1280, 8, 8) in seen
    assert (2048, 8, 8) in seen
    tiny = mp.tiny_inception()
    layers = [as_tuple(l) for l in tiny.layers]
    a = seeded_init(tiny.layers, 3)
    b = orc.seeded_init(layers, 3)
    for ra, rb in zip(a, b):
        assert len(ra) == len(rb)
        for u, v in zip(ra, rb):
            np.testing.assert_array_equal(u, v)
    assert mp.split(tiny).split_index == orc.split_index(layers)
    for l, t in zip(tiny.layers, layers):
        assert orc.param_shapes(t) == [tuple(s) for s in __import__(
            "paper_1812_10624_b200.tensor_core", fromlist=["x"]).param_shapes(l)]


def test_concat_and_avgpool_shape_errors():
    from paper_1812_10624_b200.tensor_core import AvgPool2d, Concat, Conv2d, ShapeMismatch, out_shape
    with pytest.raises(ShapeMismatch):
        out_shape(Concat(((Conv2d(4, 8, 1),), (Conv2d(4, 8, 3, 2),))), (4, 5, 5))
    with pytest.raises(ShapeMismatch):
        out_shape(AvgPool2d(3, 1, 2), (4, 5, 5))
    assert out_shape(Conv2d(4, 8, 1, 1, 0, 7, 3), (4, 5, 5)) == (8, 5, 5)
