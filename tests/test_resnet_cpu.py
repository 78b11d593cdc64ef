"""ResNet-trunk kinds, CPU side: the oracle's
BatchNorm / global-pool / residual backward against finite differences (the
reference has no such kinds, so the oracle is checked against calculus, not
against reference outputs), init and partition of the host-side specs."""

import numpy as np
import pytest

import stanza_oracle as orc

F64 = np.float64


def _fd_check(f, x, g_analytic, idx, eps=1e-2, tol=2e-2):
    for i in idx:
        xp, xm = x.copy(), x.copy()
        xp.flat[i] += eps
        xm.flat[i] -= eps
        num = (f(xp) - f(xm)) / (2 * eps)
        assert abs(num - g_analytic.flat[i]) <= tol * max(1.0, abs(num)), (i, num,
                                                                           g_analytic.flat[i])


def test_bn_backward_matches_finite_differences():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((3, 4, 5, 5)).astype(np.float32) * 2 + 1
    gamma = rng.uniform(0.5, 1.5, 4).astype(np.float32)
    beta = rng.standard_normal(4).astype(np.float32)
    w = rng.standard_normal(x.shape)        # loss = sum(w * y)

    def loss(xx, gg=gamma, bb=beta):
        y, _ = orc.bn_forward(xx.astype(np.float32), gg, bb, 1e-5)
        return float((y.astype(F64) * w).sum())

    y, cache = orc.bn_forward(x, gamma, beta, 1e-5)
    gx, dg, db = orc.bn_backward(cache, gamma, w.astype(np.float32))
    _fd_check(loss, x, gx, range(0, x.size, 7))
    _fd_check(lambda g: loss(x, g.astype(np.float32)), gamma.astype(F64), dg, range(4))
    _fd_check(lambda b: loss(x, gamma, b.astype(np.float32)), beta.astype(F64), db, range(4))
    # normalised output: zero mean, unit variance per channel (before the affine)
    xhat = cache[0]
    np.testing.assert_allclose(xhat.mean(axis=(0, 2, 3)), 0, atol=1e-12)
    np.testing.assert_allclose(xhat.var(axis=(0, 2, 3)), 1, rtol=1e-3)


def test_gap_and_residual_backward_match_finite_differences():
    layers, shape = orc.tiny_resnet_layers()
    cut = orc.split_index(layers)
    front = layers[:cut]
    params = orc.seeded_init(front, 5)
    x = np.random.default_rng(1).standard_normal((4, *shape)).astype(np.float32)
    out, caches = orc.block_forward(front, params, x)
    w = np.random.default_rng(2).standard_normal(out.shape).astype(np.float32)
    _, grads = orc.block_backward(front, params, caches, w)

    # perturb weights of each residual block's first conv (the stem sits in
    # front of a max-pool whose window switches make the difference quotient
    # converge too slowly for a bounded test)
    for li in [i for i, l in enumerate(front) if l[0] == "residual"]:
        t = params[li][0]
        g = grads[li][0]

        def loss(v, li=li):
            p2 = [list(r) for r in params]
            p2[li][0] = v.astype(np.float32).reshape(t.shape)
            y, _ = orc.block_forward(front, p2, x)
            return float((y.astype(F64) * w).sum())
        _fd_check(loss, t.astype(F64), g, range(0, t.size, max(1, t.size // 5)), eps=1e-3,
                  tol=5e-2)


def test_resnet_specs_match_oracle_layers_and_init():
    from paper_1812_10624_b200.model_partition import resnet, split, tiny_resnet
    from paper_1812_10624_b200.tensor_core import as_tuple, seeded_init
    for spec, (layers, shape) in ((tiny_resnet(), orc.tiny_resnet_layers()),
                                  (resnet(), orc.resnet_layers())):
        assert [as_tuple(l) for l in spec.layers] == layers
        assert tuple(spec.input_shape) == shape
        part = split(spec)
        assert part.split_index == orc.split_index(layers)
    a = seeded_init(tiny_resnet().layers, 3)
    b = orc.seeded_init(orc.tiny_resnet_layers()[0], 3)
    for ra, rb in zip(a, b):
        assert len(ra) == len(rb)
        for u, v in zip(ra, rb):
            np.testing.assert_array_equal(u, v)
    p50 = split(resnet())
    # torchvision ResNet-50 has 25,557,032 parameters; + 53 conv biases here
    assert (p50.conv_params, p50.fc_params, p50.boundary_activations) == (23_534_592, 2_049_000,
                                                                         2048)


def test_residual_shape_errors():
    from paper_1812_10624_b200.tensor_core import (BatchNorm2d, Conv2d, Residual, ShapeMismatch,
                                                   out_shape)
    with pytest.raises(ShapeMismatch):
        out_shape(Residual((Conv2d(8, 16, 1),), ()), (8, 4, 4))     # identity 8 != 16 channels
    with pytest.raises(ShapeMismatch):
        out_shape(BatchNorm2d(4), (8, 4, 4))
    assert out_shape(Residual((Conv2d(8, 16, 3, 2, 1),), (Conv2d(8, 16, 1, 2),)),
                     (8, 5, 5)) == (16, 3, 3)
