"""The CPU oracle against the reference's own outputs (golden fixtures made
by oracle/make_golden.py from /root/reference) and known-answer tests."""

import numpy as np
import pytest

import golden_io
import stanza_oracle as orc


@pytest.fixture(scope="module")
def ops():
    return golden_io.ops()


@pytest.mark.parametrize("case", ["c3s1p1", "c3s2p0", "c5s1p2", "c11s4p2", "c3s1p0_odd"])
def test_conv_matches_reference(ops, case):
    g = ops[f"conv_{case}"]
    s, p = int(g["cfg"][3]), int(g["cfg"][4])
    y, xp = orc.conv_forward(g["x"], g["w"], g["b"], s, p)
    gx, gw, gb = orc.conv_backward(xp, g["w"], g["gy"], s, p)
    for a, b in ((y, g["y"]), (gx, g["gx"]), (gw, g["gw"]), (gb, g["gb"])):
        assert orc.rel_err(a, b) <= 1e-7


@pytest.mark.parametrize("case", ["p2s2", "p3s2", "p3s2_ties"])
def test_maxpool_bit_exact(ops, case):
    g = ops[f"pool_{case}"]
    k, s = (int(v) for v in g["cfg"])
    y, arg = orc.maxpool_forward(g["x"], k, s)
    np.testing.assert_array_equal(y, g["y"])
    np.testing.assert_array_equal(arg.astype(np.uint8), g["arg"])
    np.testing.assert_array_equal(orc.maxpool_backward(arg, g["x"].shape, g["gy"], k, s), g["gx"])


@pytest.mark.parametrize("case", ["fc_small", "fc_mid"])
def test_fc_matches_reference(ops, case):
    g = ops[case]
    assert orc.rel_err(orc.fc_forward(g["x"], g["w"], g["b"]), g["y"]) <= 1e-7
    for a, b in zip(orc.fc_backward(g["x"], g["w"], g["gy"]), (g["gx"], g["gw"], g["gb"])):
        assert orc.rel_err(a, b) <= 1e-7


@pytest.mark.parametrize("case", ["ce_10", "ce_1000"])
def test_softmax_ce_bit_exact(ops, case):
    g = ops[case]
    loss, p = orc.softmax_ce_forward(g["z"], g["labels"])
    np.testing.assert_array_equal(loss, g["loss"])
    np.testing.assert_array_equal(orc.softmax_ce_backward(p, g["labels"]), g["g"])


def test_sgd_bit_exact(ops):
    g = ops["sgd"]
    w, v = [[g["w"].copy()]], [[g["v"].copy()]]
    orc.sgd_update(w, [[g["g"]]], v, int(g["n"]), float(g["lr"]), float(g["mu"]))
    np.testing.assert_array_equal(w[0][0], g["w1"])
    np.testing.assert_array_equal(v[0][0], g["v1"])


@pytest.mark.parametrize("case", ["tiny_1x1", "tiny_2x1", "tiny_4x2", "tiny_3x2", "tiny_7x1",
                                  "tiny32_2x1", "mlp_2x1"])
def test_layer_separated_train_bit_exact(case):
    g = golden_io.train()[f"train_{case}"]
    if case.startswith("mlp"):
        layers, shape = orc.tiny_mlp_layers()
    else:
        layers, shape = orc.tiny_cnn_layers(32 if case.startswith("tiny32") else 16)
    mk = orc.batch_fn(shape, int(g["batch_k"]), int(g["data_seed"]))
    p, v, losses = orc.layer_separated_train(layers, int(g["batch_k"]), int(g["n_conv"]),
                                             int(g["n_fc"]), int(g["iters"]), int(g["seed"]),
                                             mk, cut=int(g["cut"]))
    ref_p, ref_v = golden_io.nested_state(g)
    assert orc.max_param_dev(p, ref_p) == 0.0
    assert orc.max_param_dev(v, ref_v) == 0.0
    np.testing.assert_array_equal(losses, g["losses"])


def test_hand_arithmetic():
    """Reference KATs (test_tensor_core.py:46-87, :199-207)."""
    y, _ = orc.conv_forward(np.array([[[[1, 2], [3, 4]]]], np.float32),
                            np.array([[[[1, 0], [0, 1]]]], np.float32),
                            np.array([0.5], np.float32), 1, 0)
    assert y[0, 0, 0, 0] == pytest.approx(5.5)
    np.testing.assert_allclose(orc.fc_forward(np.ones((1, 2), np.float32),
                                              np.array([[1, 2], [3, 4]], np.float32),
                                              np.array([0.5, -0.5], np.float32)), [[4.5, 5.5]])
    y, _ = orc.maxpool_forward(np.arange(16, dtype=np.float32).reshape(1, 1, 4, 4), 2, 2)
    np.testing.assert_array_equal(y[0, 0], [[5, 7], [13, 15]])
    loss, p = orc.softmax_ce_forward(np.zeros((1, 2), np.float32), np.array([0]))
    assert loss[0] == pytest.approx(np.log(2.0), rel=1e-6)
    np.testing.assert_allclose(orc.softmax_ce_backward(p, np.array([0])), [[-0.5, 0.5]])
    w, v = [[np.array([2.0], np.float32)]], [[np.zeros(1, np.float32)]]
    orc.sgd_update(w, [[np.array([4.0], np.float32)]], v, 4, 0.1, 0.9)
    assert w[0][0][0] == pytest.approx(1.9, rel=1e-6)
    orc.sgd_update(w, [[np.array([4.0], np.float32)]], v, 4, 0.1, 0.9)
    assert w[0][0][0] == pytest.approx(1.71, rel=1e-6)


def test_conv_gradients_finite_difference():
    rng = np.random.Generator(np.random.PCG64(0))
    x = rng.standard_normal((1, 2, 5, 5)).astype(np.float32)
    w = rng.standard_normal((3, 2, 3, 3)).astype(np.float32)
    b = np.zeros(3, np.float32)
    y, xp = orc.conv_forward(x, w, b, 2, 1)
    proj = rng.standard_normal(y.shape)
    gx, gw, _ = orc.conv_backward(xp, w, proj.astype(np.float32), 2, 1)
    eps = 1e-3
    for arr, grad in ((x, gx), (w, gw)):
        flat, gflat = arr.reshape(-1), grad.reshape(-1)
        for i in range(0, flat.size, 7):
            old = flat[i]
            flat[i] = old + eps
            hi = (orc.conv_forward(x, w, b, 2, 1)[0] * proj).sum()
            flat[i] = old - eps
            lo = (orc.conv_forward(x, w, b, 2, 1)[0] * proj).sum()
            flat[i] = old
            assert (hi - lo) / (2 * eps) == pytest.approx(gflat[i], rel=2e-2, abs=2e-3)
