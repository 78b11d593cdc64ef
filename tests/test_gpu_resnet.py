"""ResNet-trunk kinds on the B200 vs the CPU oracle.

The reference has no BatchNorm / residual / global-pool layers, so these
checks compare the CUDA path with the oracle's own definition of them
(oracle/stanza_oracle.py bn_forward, bn_backward, gap_*, "residual"):
parity UNPINNED by any reference output.  Bar: the reference's 1e-5
max_param_dev after N layer-separated iterations, losses within 1e-5.
"""

import numpy as np
import pytest
import torch

import stanza_oracle as orc

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _worst(a, b, n=6):
    """(dev, layer, tensor, max|ref|) of the n worst tensors (for messages)."""
    rows = []
    for li, (ra, rb) in enumerate(zip(a, b)):
        for ti, (x, y) in enumerate(zip(ra, rb)):
            rows.append((orc.rel_err(x, y), li, ti, float(np.abs(y).max(initial=0))))
    return sorted(rows, reverse=True)[:n]


def _run(spec, nc, nf, iters, lr=0.05, seed=3, dseed=7, classes=10, **kw):
    from paper_1812_10624_b200.stanza_runtime import StanzaCluster
    from paper_1812_10624_b200.tensor_core import as_tuple
    mk = orc.batch_fn(spec.input_shape, spec.batch_k, dseed, classes=classes)
    res = StanzaCluster(spec, n_conv=nc, n_fc=nf, batch_fn=mk, lr=lr, momentum=0.9, seed=seed,
                        device="cuda:0", **kw).train(iters)
    torch.cuda.synchronize()
    ref = orc.layer_separated_train([as_tuple(l) for l in spec.layers], spec.batch_k, nc, nf,
                                    iters, seed, mk, lr=lr)
    return res, ref


@pytest.mark.parametrize("nc,nf", [(1, 1), (2, 1), (3, 2)])
def test_tiny_resnet_matches_oracle(lib, nc, nf):
    """Strided stem (space-to-depth) + BN + ReLU + pool, projection shortcuts
    at stride 1 and 2, an identity block, global pool, FC head.  With n_c > 1
    co-located the trunk runs all workers' batches in one pass and BatchNorm
    must still normalise per worker (group = K)."""
    from paper_1812_10624_b200.model_partition import tiny_resnet
    res, (ref_p, ref_v, ref_l) = _run(tiny_resnet(), nc, nf, 4)
    assert orc.max_param_dev(res.state.params, ref_p) <= TOL
    # velocities: the biases of convs that feed a BatchNorm have gradients that
    # are pure rounding noise (BN removes any per-channel shift), so compare
    # against the largest velocity instead of per tensor
    vmax = max(float(np.abs(t).max()) for row in ref_v for t in row)
    vdev = max(float(np.abs(np.asarray(a, np.float64) - b).max())
               for ra, rb in zip(res.state.velocities, ref_v) for a, b in zip(ra, rb))
    assert vdev <= 1e-5 * vmax
    np.testing.assert_allclose(res.losses, ref_l, rtol=TOL)


def test_resnet50_structure_matches_oracle(lib):
    """The full ResNet-50 layer list (16 bottleneck blocks, 2048-wide
    boundary, 1000 classes) on 64x64 inputs, K = 2, one iteration; every conv
    shape class of the 224x224 model (7x7/2 stem as space-to-depth, 1x1,
    3x3/1, 3x3/2, 1x1/2 projections) on the TMA and cp.async paths.

    This configuration is ill-conditioned for elementwise comparison: in the
    oracle alone, a 1e-7 relative perturbation of the initial parameters
    moves the first step's gradient by 2% of its largest entry and the BN
    betas by up to 18% (a beta's gradient is a sum that cancels almost
    exactly, since the following BatchNorm's backward removes the mean; a
    channel that is constant over K*H*W = 8 values turns rounding into O(1)
    normalised values).  So the bar here is the loss (rtol 1e-5) and the
    update direction: cosine over the whole gradient vector >= 0.999 (the
    oracle against itself under 1e-7 parameter perturbations: 0.99981 and
    0.99994 for two perturbation seeds; the GPU measured 0.99973);
    exact per-block parity at these shapes is test_gpu_engine.py's
    test_resnet_stage4_first_block / test_resnet_pieces."""
    from paper_1812_10624_b200.model_partition import resnet
    res, (ref_p, ref_v, ref_l) = _run(resnet(batch_k=2, side=64), 1, 1, 1, lr=0.005,
                                      classes=1000)
    np.testing.assert_allclose(res.losses, ref_l, rtol=TOL)
    a = np.concatenate([np.ravel(t) for row in res.state.velocities for t in row]).astype(np.float64)
    b = np.concatenate([np.ravel(t) for row in ref_v for t in row]).astype(np.float64)
    assert np.isfinite(a).all()
    cos = float(a @ b / (np.linalg.norm(a) * np.linalg.norm(b)))
    assert cos >= 0.999, cos


def test_tiny_resnet_deterministic_and_graph(lib):
    """Two runs are bit-identical, and the CUDA-graph replay of the step
    (what bench.py times) gives the eager step's parameters bit for bit."""
    from paper_1812_10624_b200.model_partition import tiny_resnet
    from paper_1812_10624_b200.stanza_runtime import StanzaCluster
    spec = tiny_resnet()
    mk = orc.batch_fn(spec.input_shape, spec.batch_k, 11)

    def make():
        return StanzaCluster(spec, n_conv=2, n_fc=1, batch_fn=mk, lr=0.05, seed=4,
                             device="cuda:0")

    a, b = make().train(3), make().train(3)
    for la, lb in zip(a.state.params, b.state.params):
        for x, y in zip(la, lb):
            np.testing.assert_array_equal(x, y)
    eager, graphed = make(), make()
    for c in (eager, graphed):            # one eager step each (sets kernel attributes)
        c.load_batch(0)
        c.step()
    x, y = eager.x.clone(), eager.labels.clone()
    g = graphed.capture(x, y)
    for _ in range(2):
        eager.step(x=x, labels=y)
        g.replay()
    torch.cuda.synchronize()
    for la, lb in zip(eager.state().params, graphed.state().params):
        for u, v in zip(la, lb):
            np.testing.assert_array_equal(u, v)


def test_bn_micro_batches_rejected(lib):
    from paper_1812_10624_b200.model_partition import ConfigError, tiny_resnet
    from paper_1812_10624_b200.stanza_runtime import StanzaCluster
    spec = tiny_resnet()
    with pytest.raises(ConfigError):
        StanzaCluster(spec, n_conv=1, n_fc=1, batch_fn=orc.batch_fn(spec.input_shape, 4, 1),
                      lr=0.05, device="cuda:0", micro_batches=2)
