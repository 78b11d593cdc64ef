"""Generate the golden fixtures under tests/golden from the REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    python oracle/make_golden.py

It imports the unmodified reference package read-only
(PYTHONPATH=/root/reference/pkg/src), runs its numeric core and its
StanzaCluster on small seeded inputs, and stores inputs + outputs as
compressed npz files.  It also runs oracle/stanza_oracle.py on the same
inputs and refuses to write anything unless the restatement matches the
reference (bit-exact on integer/role data, <= 1e-6 relative on floats).
The fixtures travel with the repo; /root/reference does not.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
OUT = os.path.join(REPO, "tests", "golden")
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")
sys.path.insert(0, HERE)

import stanza_oracle as orc  # noqa: E402
from stanza import tensor_core as tc  # noqa: E402
from stanza.model_partition import (builtin_model, executable_spec,  # noqa: E402
                                    mlp_split, split, tiny_cnn, tiny_mlp)
from stanza.stanza_runtime import StanzaCluster, plan_groups  # noqa: E402
from trainers import make_batch_fn, reference_train  # noqa: E402

_KIND = {
    tc.Conv2d: lambda l: ("conv", l.in_ch, l.out_ch, l.kernel, l.stride, l.padding),
    tc.MaxPool2d: lambda l: ("maxpool", l.kernel, l.stride),
    tc.Flatten: lambda l: ("flatten",),
    tc.FullyConnected: lambda l: ("fc", l.in_dim, l.out_dim),
    tc.ReLU: lambda l: ("relu",),
    tc.SoftmaxCrossEntropy: lambda l: ("softmax_ce",),
}


def as_tuples(layers):
    return [_KIND[type(l)](l) for l in layers]


def check(name, a, b, tol=1e-6):
    err = orc.rel_err(a, b)
    if err > tol:
        raise SystemExit(f"oracle disagrees with reference on {name}: {err:.3e}")
    return err


def digest(arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.float32).tobytes())
    return h.hexdigest()


def op_vectors():
    """Per-layer forward/backward vectors from tensor_core.forward/backward."""
    rng = np.random.Generator(np.random.PCG64(20181224))
    out = {}
    conv_cases = [  # (name, C, O, k, s, p, N, H, W)
        ("c3s1p1", 3, 8, 3, 1, 1, 2, 9, 9),
        ("c3s2p0", 2, 3, 3, 2, 0, 2, 7, 7),
        ("c5s1p2", 4, 6, 5, 1, 2, 2, 8, 8),
        ("c11s4p2", 3, 5, 11, 4, 2, 1, 31, 31),
        ("c3s1p0_odd", 5, 7, 3, 1, 0, 3, 6, 5),
    ]
    for name, c, o, k, s, p, n, h, w in conv_cases:
        layer = tc.Conv2d(c, o, k, s, p)
        params = tc.seeded_init([layer], 11)[0]
        x = rng.standard_normal((n, c, h, w)).astype(np.float32)
        y, cache = tc.forward(layer, params, x)
        gy = rng.standard_normal(y.shape).astype(np.float32)
        gx, (gw, gb) = tc.backward(layer, params, cache, gy)
        oy, ocache = orc.conv_forward(x, params[0], params[1], s, p)
        ogx, ogw, ogb = orc.conv_backward(ocache, params[0], gy, s, p)
        for tag, a, b in (("y", y, oy), ("gx", gx, ogx), ("gw", gw, ogw), ("gb", gb, ogb)):
            check(f"conv {name} {tag}", a, b)
        out[f"conv_{name}"] = dict(cfg=np.array([c, o, k, s, p, n, h, w]), x=x,
                                   w=params[0], b=params[1], y=y, gy=gy, gx=gx,
                                   gw=gw, gb=gb)
    for name, k, s, shape in (("p2s2", 2, 2, (2, 3, 8, 8)),
                              ("p3s2", 3, 2, (2, 3, 13, 13)),
                              ("p3s2_ties", 3, 2, (1, 2, 9, 9))):
        layer = tc.MaxPool2d(k, s)
        if name.endswith("ties"):
            x = rng.integers(-2, 3, size=shape).astype(np.float32)
        else:
            x = rng.standard_normal(shape).astype(np.float32)
        y, cache = tc.forward(layer, [], x)
        gy = rng.standard_normal(y.shape).astype(np.float32)
        gx, _ = tc.backward(layer, [], cache, gy)
        oy, arg = orc.maxpool_forward(x, k, s)
        ogx = orc.maxpool_backward(arg, x.shape, gy, k, s)
        check(f"pool {name} y", y, oy, 0.0)
        check(f"pool {name} gx", gx, ogx, 0.0)
        out[f"pool_{name}"] = dict(cfg=np.array([k, s]), x=x, y=y, arg=cache[0].astype(np.uint8),
                                   gy=gy, gx=gx)
    for name, m, i, o in (("fc_small", 5, 11, 7), ("fc_mid", 33, 257, 130)):
        layer = tc.FullyConnected(i, o)
        params = tc.seeded_init([layer], 5)[0]
        x = rng.standard_normal((m, i)).astype(np.float32)
        y, cache = tc.forward(layer, params, x)
        gy = rng.standard_normal(y.shape).astype(np.float32)
        gx, (gw, gb) = tc.backward(layer, params, cache, gy)
        check(f"{name} y", y, orc.fc_forward(x, *params))
        for tag, a, b in zip(("gx", "gw", "gb"), (gx, gw, gb),
                             orc.fc_backward(x, params[0], gy)):
            check(f"{name} {tag}", a, b)
        out[name] = dict(x=x, w=params[0], b=params[1], y=y, gy=gy, gx=gx, gw=gw, gb=gb)
    for name, m, c in (("ce_10", 6, 10), ("ce_1000", 4, 1000)):
        z = (rng.standard_normal((m, c)) * 3).astype(np.float32)
        labels = rng.integers(0, c, m)
        loss, cache = tc.forward(tc.SoftmaxCrossEntropy(), [], z, labels=labels)
        g, _ = tc.backward(tc.SoftmaxCrossEntropy(), [], cache, None)
        ol, probs = orc.softmax_ce_forward(z, labels)
        check(f"{name} loss", loss, ol, 0.0)
        check(f"{name} grad", g, orc.softmax_ce_backward(probs, labels), 0.0)
        out[name] = dict(z=z, labels=labels, loss=loss, g=g)
    # momentum SGD, exact fp32 op order
    w = rng.standard_normal(1000).astype(np.float32)
    v = rng.standard_normal(1000).astype(np.float32)
    g = rng.standard_normal(1000).astype(np.float32)
    params = [[w.copy()]]
    opt = tc.OptimizerState(lr=0.05, momentum=0.9, velocity=[[v.copy()]])
    tc.sgd_step(params, [[g]], 28, opt)
    ow, ov = [[w.copy()]], [[v.copy()]]
    orc.sgd_update(ow, [[g]], ov, 28, 0.05, 0.9)
    check("sgd w", params[0][0], ow[0][0], 0.0)
    check("sgd v", opt.velocity[0][0], ov[0][0], 0.0)
    out["sgd"] = dict(w=w, v=v, g=g, n=np.array(28), lr=np.array(0.05),
                      mu=np.array(0.9), w1=params[0][0], v1=opt.velocity[0][0])
    return out


def train_vectors():
    """StanzaCluster runs (the hot path) on tiny models."""
    out = {}
    cases = [  # (name, spec factory, n_conv, n_fc, iters, seed, data_seed, boundary)
        ("tiny_1x1", lambda: tiny_cnn(), 1, 1, 10, 3, 7, None),
        ("tiny_2x1", lambda: tiny_cnn(), 2, 1, 8, 5, 11, None),
        ("tiny_4x2", lambda: tiny_cnn(), 4, 2, 8, 5, 11, None),
        ("tiny_3x2", lambda: tiny_cnn(), 3, 2, 8, 5, 11, None),
        ("tiny_7x1", lambda: tiny_cnn(), 7, 1, 4, 3, 7, None),
        ("tiny32_2x1", lambda: tiny32(), 2, 1, 5, 3, 7, None),
        ("mlp_2x1", lambda: tiny_mlp(), 2, 1, 6, 6, 4, 4),
    ]
    for name, factory, nc, nf, iters, seed, dseed, boundary in cases:
        spec = factory()
        cluster = StanzaCluster(spec, n_conv=nc, n_fc=nf,
                                batch_fn=make_batch_fn(spec, dseed), lr=0.05,
                                momentum=0.9, seed=seed, boundary=boundary)
        res = cluster.train(iters)
        layers = as_tuples(spec.layers)
        cut = cluster.partition.split_index
        op, ov, ol = orc.layer_separated_train(
            layers, spec.batch_k, nc, nf, iters, seed,
            orc.batch_fn(spec.input_shape, spec.batch_k, dseed), cut=cut)
        dev = orc.max_param_dev(res.state.params, op)
        if dev != 0.0:
            raise SystemExit(f"oracle cluster {name} deviates {dev:.3e} from reference")
        if not np.allclose(res.losses, ol, rtol=1e-12, atol=0):
            raise SystemExit(f"oracle losses {name} deviate")
        rp, _, _ = reference_train(spec, nc, iters, seed=seed, data_seed=dseed)
        item = dict(n_conv=np.array(nc), n_fc=np.array(nf), iters=np.array(iters),
                    seed=np.array(seed), data_seed=np.array(dseed), cut=np.array(cut),
                    batch_k=np.array(spec.batch_k), losses=np.array(res.losses),
                    single_dev=np.array(orc.max_param_dev(rp, res.state.params)))
        for li, layer in enumerate(res.state.params):
            for ti, t in enumerate(layer):
                item[f"p{li}_{ti}"] = t
                item[f"v{li}_{ti}"] = res.state.velocities[li][ti]
        out[f"train_{name}"] = item
        print(f"  {name}: oracle == reference (bit-exact), single-node dev "
              f"{float(item['single_dev']):.2e}")
    return out


def tiny32():
    s = tiny_cnn()
    layers = list(s.layers)
    layers[7] = tc.FullyConnected(1024, 128)
    return executable_spec("tiny_cnn32", layers, input_shape=(3, 32, 32), batch_k=4)


def meta_vectors():
    """Role maps, cuts, counts, init and batch digests for the big configs."""
    groups = {f"{nc}x{nf}": plan_groups(nc, nf)
              for nc in range(1, 9) for nf in range(1, nc + 1)}
    for key, g in groups.items():
        nc, nf = map(int, key.split("x"))
        if orc.plan_groups(nc, nf) != g:
            raise SystemExit(f"plan_groups restatement differs at {key}")
    specs = {}
    for name, (layers, shape) in (("alexnet", orc.alexnet_layers()),
                                  ("vgg16", orc.vgg16_layers())):
        ref_layers = []
        for l in layers:
            ref_layers.append({"conv": lambda l: tc.Conv2d(*l[1:]),
                               "maxpool": lambda l: tc.MaxPool2d(*l[1:]),
                               "flatten": lambda l: tc.Flatten(),
                               "fc": lambda l: tc.FullyConnected(*l[1:]),
                               "relu": lambda l: tc.ReLU(),
                               "softmax_ce": lambda l: tc.SoftmaxCrossEntropy()}[l[0]](l))
        spec = executable_spec(name, ref_layers, input_shape=shape, batch_k=1)
        part = split(spec)
        ref_init = tc.seeded_init(spec.layers, 3)
        flat_ref = [t for layer in ref_init for t in layer]
        ora_init = orc.seeded_init(layers, 3)
        flat_ora = [t for layer in ora_init for t in layer]
        if digest(flat_ref) != digest(flat_ora):
            raise SystemExit(f"seeded_init restatement differs for {name}")
        bx, by = make_batch_fn(spec, 7)(0, 1)
        ox, oy = orc.batch_fn(shape, 1, 7)(0, 1)
        if digest([bx]) != digest([ox]) or not np.array_equal(by, oy):
            raise SystemExit(f"batch restatement differs for {name}")
        specs[name] = dict(split_index=part.split_index, conv_params=part.conv_params,
                           fc_params=part.fc_params,
                           boundary_activations=part.boundary_activations,
                           init_seed3_sha256=digest(flat_ref),
                           batch_seed7_it0_w1_sha256=digest([bx]),
                           batch_seed7_it0_w1_labels=[int(v) for v in by])
    mlp = mlp_split(tiny_mlp(), 4)
    specs["tiny_mlp_b4"] = dict(split_index=4, conv_params=mlp.conv_params,
                                fc_params=mlp.fc_params,
                                boundary_activations=mlp.boundary_activations)
    tiny = split(tiny_cnn())
    specs["tiny_cnn"] = dict(split_index=tiny.split_index, conv_params=tiny.conv_params,
                             fc_params=tiny.fc_params,
                             boundary_activations=tiny.boundary_activations)
    prof = builtin_model("alexnet")
    specs["alexnet_profile"] = dict(params_total=prof.params_total,
                                    params_conv=prof.params_conv,
                                    boundary_activations=prof.boundary_activations)
    return dict(plan_groups=groups, specs=specs)


def main():
    os.makedirs(OUT, exist_ok=True)
    print("per-op vectors ...")
    ops = op_vectors()
    np.savez_compressed(os.path.join(OUT, "ops.npz"),
                        **{f"{k}__{f}": v for k, d in ops.items() for f, v in d.items()})
    print("training runs ...")
    tr = train_vectors()
    np.savez_compressed(os.path.join(OUT, "train.npz"),
                        **{f"{k}__{f}": v for k, d in tr.items() for f, v in d.items()})
    print("role maps / specs / digests ...")
    with open(os.path.join(OUT, "meta.json"), "w") as fh:
        json.dump(meta_vectors(), fh, indent=1, sort_keys=True)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
