"""CPU oracle for the Stanza layer-separated training step.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package may import this
module: it is the checker the parity tests, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg compare against.
It is a numpy restatement of the reference algorithm (stanza-sim 0.1.0,
``/root/reference/pkg/src/stanza``), written from its semantics:

* storage is float32, every contraction accumulates in float64 and rounds
  once to float32 (``tensor_core.py:3-8``);
* backward passes return gradient SUMS over the batch; the single division
  by the global batch happens inside the momentum step
  (``tensor_core.py:366-388``).

Parity is pinned: ``oracle/make_golden.py`` runs the reference itself in the
build container and stores its outputs under ``tests/golden``;
``tests/test_oracle.py`` checks this restatement against those fixtures and
against the reference's own known-answer tests.

Layers are plain tuples so this module depends on nothing but numpy:

    ("conv", in_ch, out_ch, kernel, stride, pad)
    ("maxpool", kernel, stride)
    ("flatten",)
    ("fc", in_dim, out_dim)
    ("relu",)
    ("softmax_ce",)

SURVEY.md §8f row 4 adds the layer kinds of the ResNet trunk.  The
reference has no such kinds (``tensor_core.py:37-74``), so their semantics
are defined HERE (training-mode BatchNorm over each call's batch, global
average pooling, post-activation residual blocks); parity for them is
UNPINNED -- no reference output exists to check this restatement against:

    ("bn", channels, eps)             gamma, beta [C]; init 1 / 0 (no RNG draw)
    ("gap",)                          (C, H, W) -> (C, 1, 1)
    ("residual", body, shortcut)      relu(body(x) + shortcut(x)); shortcut
                                      () is the identity; params = body's
                                      then shortcut's, one flat row

and those of the Inception-V3 trunk (same status: defined here, unpinned):

    ("conv", C, O, (kh, kw), s, (ph, pw))   asymmetric kernel / padding
                                      (1xn, nx1); W [O, C, kh, kw]
    ("avgpool", kernel, stride, pad)  zero-padded average pool, every window
                                      divided by kernel^2 (padding counted)
    ("concat", branches)              branches: tuple of layer tuples, each
                                      applied to the same input; outputs
                                      concatenated along channels in branch
                                      order; params = every branch's in order,
                                      one flat row; the input gradient is the
                                      fp32 left fold of the branches' input
                                      gradients in branch order
"""

from __future__ import annotations

import random

import numpy as np

F32 = np.float32
F64 = np.float64


# ---------------------------------------------------------------------------
# per-layer math (tensor_core.py:153-301)
# ---------------------------------------------------------------------------

def _conv_out_hw(h, w, k, s, p):
    kh, kw = _pair(k)
    ph, pw = _pair(p)
    return (h + 2 * ph - kh) // s + 1, (w + 2 * pw - kw) // s + 1


def _pair(v):
    return (int(v[0]), int(v[1])) if isinstance(v, (tuple, list)) else (int(v), int(v))


def conv_forward(x, w, b, stride, pad):
    """Conv2d forward, tensor_core.py:161-181.

    Zero-padded input, one float64 contraction per kernel tap (kh, kw)
    accumulated in tap order, bias added in float64, one fp32 rounding.
    Returns (y, padded input) -- the padded input is the backward cache.
    ``pad`` may be (ph, pw) and W [O, C, kh, kw] rectangular (Inception kinds).
    """
    o, c, kh_, kw_ = w.shape
    ph, pw = _pair(pad)
    xp = np.pad(x, ((0, 0), (0, 0), (ph, ph), (pw, pw))) if (ph or pw) else x
    n, _, hp, wp = xp.shape
    oh = (hp - kh_) // stride + 1
    ow = (wp - kw_) // stride + 1
    xd = xp.astype(F64)
    wd = w.astype(F64)
    acc = np.zeros((n, o, oh, ow), F64)
    for kh in range(kh_):
        for kw in range(kw_):
            tap = xd[:, :, kh:kh + stride * oh:stride, kw:kw + stride * ow:stride]
            # sum over input channels for this tap: [n,c,h,w] x [o,c] -> [n,o,h,w]
            acc += np.einsum("nchw,oc->nohw", tap, wd[:, :, kh, kw])
    acc += b.astype(F64)[None, :, None, None]
    return acc.astype(F32), xp


def conv_backward(xp, w, gy, stride, pad):
    """Conv2d backward, tensor_core.py:242-261.

    Returns (gx, gw, gb): input gradient (padding cropped), weight-gradient
    sum, bias-gradient sum, each computed in float64 and rounded once.
    """
    o, c, kh_, kw_ = w.shape
    ph, pw = _pair(pad)
    _, _, hp, wp = xp.shape
    oh, ow = gy.shape[2], gy.shape[3]
    gd = gy.astype(F64)
    xd = xp.astype(F64)
    wd = w.astype(F64)
    gw = np.zeros(wd.shape, F64)
    gxp = np.zeros(xd.shape, F64)
    for kh in range(kh_):
        for kw in range(kw_):
            tap = xd[:, :, kh:kh + stride * oh:stride, kw:kw + stride * ow:stride]
            gw[:, :, kh, kw] = np.einsum("nohw,nchw->oc", gd, tap)
            gxp[:, :, kh:kh + stride * oh:stride, kw:kw + stride * ow:stride] += \
                np.einsum("nohw,oc->nchw", gd, wd[:, :, kh, kw])
    gb = gd.sum(axis=(0, 2, 3))
    gx = gxp[:, :, ph:hp - ph, pw:wp - pw]
    return gx.astype(F32), gw.astype(F32), gb.astype(F32)


def maxpool_forward(x, k, s):
    """MaxPool2d forward, tensor_core.py:183-198.

    Window candidates are enumerated kh-major / kw-minor; the FIRST maximum
    wins (numpy argmax).  Returns (y, argmax index in [0, k*k)).
    """
    n, c, h, w = x.shape
    oh = (h - k) // s + 1
    ow = (w - k) // s + 1
    cand = np.stack([x[:, :, kh:kh + s * oh:s, kw:kw + s * ow:s]
                     for kh in range(k) for kw in range(k)], axis=-1)
    arg = cand.argmax(axis=-1)
    y = np.take_along_axis(cand, arg[..., None], axis=-1)[..., 0]
    return y, arg


def maxpool_backward(arg, x_shape, gy, k, s):
    """MaxPool2d backward, tensor_core.py:263-276: the output gradient goes to
    the argmax cell; overlapping windows accumulate in float64."""
    oh, ow = arg.shape[2], arg.shape[3]
    gx = np.zeros(x_shape, F64)
    gd = gy.astype(F64)
    for kh in range(k):
        for kw in range(k):
            hit = arg == kh * k + kw
            gx[:, :, kh:kh + s * oh:s, kw:kw + s * ow:s] += np.where(hit, gd, 0.0)
    return gx.astype(F32)


def avgpool_forward(x, k, s, p):
    """AvgPool2d (Inception kinds): zero padding p, window sum in float64
    (kh-major), divided by k*k (padding counted), one fp32 rounding."""
    xp = np.pad(x, ((0, 0), (0, 0), (p, p), (p, p))).astype(F64) if p else x.astype(F64)
    n, c, hp, wp = xp.shape
    oh, ow = (hp - k) // s + 1, (wp - k) // s + 1
    acc = np.zeros((n, c, oh, ow), F64)
    for kh in range(k):
        for kw in range(k):
            acc += xp[:, :, kh:kh + s * oh:s, kw:kw + s * ow:s]
    return (acc / (k * k)).astype(F32)


def avgpool_backward(x_shape, gy, k, s, p):
    """Each input cell receives the sum over the windows covering it of
    g / (k*k), in float64, rounded once."""
    n, c, h, w = x_shape
    oh, ow = gy.shape[2], gy.shape[3]
    gxp = np.zeros((n, c, h + 2 * p, w + 2 * p), F64)
    gd = gy.astype(F64) / (k * k)
    for kh in range(k):
        for kw in range(k):
            gxp[:, :, kh:kh + s * oh:s, kw:kw + s * ow:s] += gd
    return gxp[:, :, p:p + h, p:p + w].astype(F32)


def fc_forward(x, w, b):
    """FullyConnected forward, tensor_core.py:205-211; W is [in, out]."""
    return (x.astype(F64) @ w.astype(F64) + b.astype(F64)).astype(F32)


def fc_backward(x, w, gy):
    """FullyConnected backward, tensor_core.py:282-289 -> (gx, gW, gb)."""
    gd = gy.astype(F64)
    gx = gd @ w.astype(F64).T
    gw = x.astype(F64).T @ gd
    gb = gd.sum(axis=0)
    return gx.astype(F32), gw.astype(F32), gb.astype(F32)


def relu_forward(x):
    """ReLU, tensor_core.py:213-214 (mask = x > 0)."""
    return np.maximum(x, 0), x > 0


def relu_backward(mask, gy):
    """ReLU backward, tensor_core.py:291-293."""
    return np.where(mask, gy, 0).astype(F32)


def softmax_ce_forward(z, labels):
    """SoftmaxCrossEntropy forward, tensor_core.py:216-228.

    Max-subtracted float64 softmax; per-sample loss -log p[label] rounded
    to fp32.  Returns (losses, probs64).
    """
    zd = z.astype(F64)
    zd = zd - zd.max(axis=1, keepdims=True)
    e = np.exp(zd)
    p = e / e.sum(axis=1, keepdims=True)
    rows = np.arange(z.shape[0])
    return (-np.log(p[rows, labels])).astype(F32), p


def softmax_ce_backward(p, labels):
    """Gradient of the per-batch loss SUM wrt logits: p - onehot
    (tensor_core.py:295-299; no 1/n)."""
    g = p.copy()
    g[np.arange(len(labels)), labels] -= 1.0
    return g.astype(F32)


def bn_forward(x, gamma, beta, eps):
    """BatchNorm2d forward, training mode (not in the reference; §8f row 4).

    Batch statistics over (N, H, W) in float64 (two-pass, biased variance),
    xhat = (x - mean) * rstd, y = xhat * gamma + beta rounded once to fp32.
    eps is taken at float32 precision (the value the C ABI receives).
    Returns (y, cache) with cache = (xhat64, rstd64, m).
    """
    xd = x.astype(F64)
    m = x.shape[0] * x.shape[2] * x.shape[3]
    mean = xd.mean(axis=(0, 2, 3))
    var = ((xd - mean[None, :, None, None]) ** 2).mean(axis=(0, 2, 3))
    rstd = 1.0 / np.sqrt(var + float(F32(eps)))
    xhat = (xd - mean[None, :, None, None]) * rstd[None, :, None, None]
    y = xhat * gamma.astype(F64)[None, :, None, None] + beta.astype(F64)[None, :, None, None]
    return y.astype(F32), (xhat, rstd, m)


def bn_backward(cache, gamma, gy):
    """BatchNorm2d backward of the loss SUM -> (gx, dgamma, dbeta):
    gx = (gamma * rstd / m) * ((m * g - sum g) - xhat * sum(g * xhat)),
    everything float64, rounded once."""
    xhat, rstd, m = cache
    gd = gy.astype(F64)
    sg = gd.sum(axis=(0, 2, 3))
    sgx = (gd * xhat).sum(axis=(0, 2, 3))
    coef = (gamma.astype(F64) * rstd) / m
    inner = (m * gd - sg[None, :, None, None]) - xhat * sgx[None, :, None, None]
    gx = coef[None, :, None, None] * inner
    return gx.astype(F32), sgx.astype(F32), sg.astype(F32)


def gap_forward(x):
    """Global average pool (C, H, W) -> (C, 1, 1): float64 sum / (H*W)."""
    hw = x.shape[2] * x.shape[3]
    return (x.astype(F64).sum(axis=(2, 3), keepdims=True) / hw).astype(F32)


def gap_backward(x_shape, gy):
    """Each input cell receives g / (H*W) (float64 quotient, rounded once)."""
    hw = x_shape[2] * x_shape[3]
    return np.broadcast_to((gy.astype(F64) / hw).astype(F32), x_shape).copy()


def _split_rows(layers, flat):
    """Cut one residual row's flat tensor list into per-sub-layer lists."""
    out, off = [], 0
    for l in layers:
        n = len(param_shapes(l))
        out.append(list(flat[off:off + n]))
        off += n
    return out


# ---------------------------------------------------------------------------
# shapes, init, blocks
# ---------------------------------------------------------------------------

def param_shapes(layer):
    """tensor_core.py:81-88: conv W [O,C,k,k] + b [O]; FC W [in,out] + b [out]."""
    if layer[0] == "conv":
        _, cin, cout, k, _, _ = layer
        kh, kw = _pair(k)
        return [(cout, cin, kh, kw), (cout,)]
    if layer[0] == "fc":
        return [(layer[1], layer[2]), (layer[2],)]
    if layer[0] == "bn":
        return [(layer[1],), (layer[1],)]
    if layer[0] == "residual":
        return [s for l in layer[1] + layer[2] for s in param_shapes(l)]
    if layer[0] == "concat":
        return [s for br in layer[1] for l in br for s in param_shapes(l)]
    return []


def fan_in(layer):
    if layer[0] == "conv":
        kh, kw = _pair(layer[3])
        return layer[1] * kh * kw
    return layer[1]


def out_shape(layer, shape):
    """Per-sample output shape (tensor_core.py:103-140), no validation."""
    kind = layer[0]
    if kind == "conv":
        _, _, cout, k, s, p = layer
        oh, ow = _conv_out_hw(shape[1], shape[2], k, s, p)
        return (cout, oh, ow)
    if kind == "maxpool":
        _, k, s = layer
        return (shape[0], (shape[1] - k) // s + 1, (shape[2] - k) // s + 1)
    if kind == "avgpool":
        _, k, s, p = layer
        return (shape[0], (shape[1] + 2 * p - k) // s + 1, (shape[2] + 2 * p - k) // s + 1)
    if kind == "concat":
        outs = []
        for br in layer[1]:
            sh = shape
            for l in br:
                sh = out_shape(l, sh)
            outs.append(sh)
        return (sum(o[0] for o in outs), outs[0][1], outs[0][2])
    if kind == "flatten":
        return (int(np.prod(shape)),)
    if kind == "fc":
        return (layer[2],)
    if kind in ("relu", "bn"):
        return shape
    if kind == "gap":
        return (shape[0], 1, 1)
    if kind == "residual":
        for l in layer[1]:
            shape = out_shape(l, shape)
        return shape
    return ()


def _init_layer(gen, layer):
    if layer[0] == "bn":
        return [np.ones(layer[1], F32), np.zeros(layer[1], F32)]
    if layer[0] == "residual":
        return [t for l in layer[1] + layer[2] for t in _init_layer(gen, l)]
    if layer[0] == "concat":
        return [t for br in layer[1] for l in br for t in _init_layer(gen, l)]
    ts = []
    for shp in param_shapes(layer):
        bound = float(np.sqrt(1.0 / fan_in(layer)))
        ts.append(gen.uniform(-bound, bound, size=shp).astype(F32))
    return ts


def seeded_init(layers, seed):
    """tensor_core.py:332-346: one PCG64(seed) stream, U(-s, s) drawn in float64
    then rounded, s = sqrt(1/fan_in), weight before bias, layer order.  (§8f
    kinds: BatchNorm gamma 1 / beta 0 without a draw; a residual block draws
    for its body then its shortcut.)"""
    gen = np.random.Generator(np.random.PCG64(seed))
    return [_init_layer(gen, layer) for layer in layers]


def block_forward(layers, params, x, labels=None):
    """Forward through a layer list, keeping per-layer caches
    (tensor_core.py:304-311)."""
    caches = []
    for layer, p in zip(layers, params):
        kind = layer[0]
        if kind == "conv":
            x, cache = conv_forward(x, p[0], p[1], layer[4], layer[5])
        elif kind == "maxpool":
            shape = x.shape
            x, arg = maxpool_forward(x, layer[1], layer[2])
            cache = (arg, shape)
        elif kind == "flatten":
            cache = x.shape
            x = np.ascontiguousarray(x).reshape(x.shape[0], -1)
        elif kind == "fc":
            cache = x
            x = fc_forward(x, p[0], p[1])
        elif kind == "relu":
            x, cache = relu_forward(x)
        elif kind == "softmax_ce":
            x, probs = softmax_ce_forward(x, labels)
            cache = (probs, labels)
        elif kind == "bn":
            x, cache = bn_forward(x, p[0], p[1], layer[2])
        elif kind == "gap":
            cache = x.shape
            x = gap_forward(x)
        elif kind == "avgpool":
            cache = x.shape
            x = avgpool_forward(x, layer[1], layer[2], layer[3])
        elif kind == "concat":
            outs, bcaches, off, bparams = [], [], 0, []
            for br in layer[1]:
                nb = len(param_shapes(("concat", (br,))))
                pb = _split_rows(br, p[off:off + nb])
                off += nb
                yb, cb = block_forward(br, pb, x)
                outs.append(yb)
                bcaches.append(cb)
                bparams.append(pb)
            cache = (bcaches, bparams, [o.shape[1] for o in outs])
            x = np.concatenate(outs, axis=1)
        elif kind == "residual":
            body, short = layer[1], layer[2]
            pb, ps = _split_rows(body, p), _split_rows(short, p[len(param_shapes(("residual", body, ()))):])
            yb, cb = block_forward(body, pb, x)
            ys, cs = block_forward(short, ps, x) if short else (x, None)
            x, mask = relu_forward(yb + ys)
            cache = (cb, cs, mask, pb, ps)
        else:
            raise TypeError(kind)
        caches.append(cache)
    return x, caches


def block_backward(layers, params, caches, gy, need_input_grad=True):
    """Backward through a layer list (tensor_core.py:314-325).

    Returns (grad wrt block input, per-layer [gW, gb] sums).
    """
    grads = [[] for _ in layers]
    for i in range(len(layers) - 1, -1, -1):
        layer, cache = layers[i], caches[i]
        kind = layer[0]
        if kind == "conv":
            gy, gw, gb = conv_backward(cache, params[i][0], gy, layer[4], layer[5])
            grads[i] = [gw, gb]
        elif kind == "maxpool":
            arg, shape = cache
            gy = maxpool_backward(arg, shape, gy, layer[1], layer[2])
        elif kind == "flatten":
            gy = np.ascontiguousarray(gy).reshape(cache)
        elif kind == "fc":
            gy, gw, gb = fc_backward(cache, params[i][0], gy)
            grads[i] = [gw, gb]
        elif kind == "relu":
            gy = relu_backward(cache, gy)
        elif kind == "softmax_ce":
            gy = softmax_ce_backward(*cache)
        elif kind == "bn":
            gy, dg, db = bn_backward(cache, params[i][0], gy)
            grads[i] = [dg, db]
        elif kind == "gap":
            gy = gap_backward(cache, gy)
        elif kind == "avgpool":
            gy = avgpool_backward(cache, gy, layer[1], layer[2], layer[3])
        elif kind == "concat":
            bcaches, bparams, widths = cache
            c0, gx, flat = 0, None, []
            for br, cb, pb, cw in zip(layer[1], bcaches, bparams, widths):
                gxb, gb = block_backward(br, pb, cb, np.ascontiguousarray(gy[:, c0:c0 + cw]))
                c0 += cw
                gx = gxb if gx is None else (gx + gxb).astype(F32)
                flat += [t for row in gb for t in row]
            gy = gx
            grads[i] = flat
        elif kind == "residual":
            body, short = layer[1], layer[2]
            cb, cs, mask, pb, ps = cache
            g = relu_backward(mask, gy)
            gxb, gb = block_backward(body, pb, cb, g)
            if short:
                gxs, gs = block_backward(short, ps, cs, g)
            else:
                gxs, gs = g, []
            gy = gxb + gxs
            grads[i] = [t for row in gb + gs for t in row]
    return gy, grads


def sgd_update(params, grad_sums, velocities, n, lr, mu):
    """Momentum SGD from gradient sums, tensor_core.py:366-388.

    float32 throughout, in this exact order: v *= mu; v += g * (1/n);
    w -= lr * v, with 1/n itself an fp32 quotient.
    """
    inv_n = F32(1.0) / F32(n)
    lr32, mu32 = F32(lr), F32(mu)
    for lp, lg, lv in zip(params, grad_sums, velocities):
        for w, g, v in zip(lp, lg, lv):
            v *= mu32
            v += g * inv_n
            w -= lr32 * v


# ---------------------------------------------------------------------------
# model cut and role map (model_partition.py:144-195, stanza_runtime.py:41-56)
# ---------------------------------------------------------------------------

def split_index(layers):
    """model_partition.py:144-173: the cut follows the last MaxPool/Flatten
    that precedes the first FC layer.  None when there is no such cut."""
    first_fc = next((i for i, l in enumerate(layers) if l[0] == "fc"), None)
    if first_fc is None:
        return None
    for i in range(first_fc - 1, -1, -1):
        if layers[i][0] in ("maxpool", "flatten"):
            return i + 1
    return None


def equal_split(total, parts):
    """ps_runtime.py:27-32: near-equal shards, remainder to the first ones."""
    q, r = divmod(total, parts)
    return [q + 1 if i < r else q for i in range(parts)]


def plan_groups(n_conv, n_fc):
    """stanza_runtime.py:41-56: contiguous CONV->FC assignment."""
    if n_conv < 1 or n_fc < 1 or n_fc > n_conv:
        raise ValueError((n_conv, n_fc))
    out = []
    for j, size in enumerate(equal_split(n_conv, n_fc)):
        out += [j] * size
    return out


# ---------------------------------------------------------------------------
# synthetic batches (harness.py:180-197, tests/trainers.py:13-24)
# ---------------------------------------------------------------------------

def batch_fn(input_shape, batch_k, data_seed, classes=10):
    """Per-(iteration, worker) N(0,1) fp32 images and uniform int labels drawn
    from PCG64([seed, iteration, worker])."""
    def make(iteration, worker):
        gen = np.random.Generator(np.random.PCG64([data_seed, iteration, worker]))
        x = gen.standard_normal((batch_k, *input_shape)).astype(F32)
        y = gen.integers(0, classes, size=batch_k)
        return x, y
    return make


# ---------------------------------------------------------------------------
# allreduce summation order (collectives.py:1-24, :78-157; tests/oracles.py)
# ---------------------------------------------------------------------------

def _surplus_donors(n, seed):
    """collectives.py:78-103: which ranks fold into which core donor."""
    core = 1 << (n.bit_length() - 1)
    if core == n:
        return list(range(n)), {}
    pick = random.Random(seed)
    extra = sorted(pick.sample(range(n), n - core))
    core_ranks = [r for r in range(n) if r not in set(extra)]
    donor_slots = pick.sample(range(core), len(extra))
    return core_ranks, {s: core_ranks[d] for s, d in zip(extra, donor_slots)}


def allreduce_sum(values, seed):
    """Canonical fp32 sum every member of the reference's recursive-doubling
    allreduce returns: surplus members fold into their donor (lower rank
    first), then an aligned binary tree over the core in rank order."""
    n = len(values)
    if n == 1:
        return values[0].copy()
    core_ranks, donors = _surplus_donors(n, seed)
    acc = {r: values[r].astype(F32) for r in core_ranks}
    for s, d in donors.items():
        acc[d] = values[s] + acc[d] if s < d else acc[d] + values[s]
    level = [acc[r] for r in core_ranks]
    while len(level) > 1:
        level = [level[i] + level[i + 1] for i in range(0, len(level), 2)]
    return level[0]


def _flat(nested):
    ts = [t for layer in nested for t in layer]
    return np.concatenate([t.ravel() for t in ts]) if ts else np.zeros(0, F32)


def _unflat(vec, like):
    out, off = [], 0
    for layer in like:
        row = []
        for t in layer:
            row.append(vec[off:off + t.size].reshape(t.shape))
            off += t.size
        out.append(row)
    return out


# ---------------------------------------------------------------------------
# training loops
# ---------------------------------------------------------------------------

def single_node_train(layers, batch_k, n_workers, iterations, seed, make_batch,
                      lr=0.05, mu=0.9):
    """One-node full-batch momentum SGD over the concatenation of all
    workers' batches in worker order (tests/trainers.py:36-55,
    harness.py:440-463).  Returns (params, velocities, losses)."""
    params = seeded_init(layers, seed)
    vel = [[np.zeros_like(t) for t in layer] for layer in params]
    n = n_workers * batch_k
    losses = []
    for it in range(iterations):
        parts = [make_batch(it, w) for w in range(n_workers)]
        x = np.concatenate([p[0] for p in parts])
        y = np.concatenate([p[1] for p in parts])
        out, caches = block_forward(layers, params, x, labels=y)
        _, grads = block_backward(layers, params, caches, None)
        losses.append(float(out.sum()) / n)
        sgd_update(params, grads, vel, n, lr, mu)
    return params, vel, losses


def layer_separated_train(layers, batch_k, n_conv, n_fc, iterations, seed,
                          make_batch, lr=0.05, mu=0.9, cut=None,
                          state=None, start_iteration=0):
    """BSP layer-separated iteration, stanza_runtime.py:352-375.

    CONV worker i runs layers[:cut] on batch (it, i); FC worker j runs
    layers[cut:] on the concatenation of its members' activations in
    ascending CONV index and returns rows [pos*K, (pos+1)*K) to member pos;
    each group sums its gradient vectors in the reference's canonical
    allreduce order (seed*1_000_003 + it, stanza_runtime.py:59-61) and every
    replica applies sgd_update with n = n_conv * K.
    Returns (params, velocities, losses) for replica conv0 + fc0.
    """
    if cut is None:
        cut = split_index(layers)
    conv_to_fc = plan_groups(n_conv, n_fc)
    members = [[i for i, j in enumerate(conv_to_fc) if j == f] for f in range(n_fc)]
    if state is None:
        full = seeded_init(layers, seed)
        vel = [[np.zeros_like(t) for t in layer] for layer in full]
    else:
        full, vel = state
        full = [[t.copy() for t in layer] for layer in full]
        vel = [[t.copy() for t in layer] for layer in vel]
    conv_p, fc_p = full[:cut], full[cut:]
    conv_v, fc_v = vel[:cut], vel[cut:]
    front, back = layers[:cut], layers[cut:]
    n = n_conv * batch_k
    losses = []
    for step in range(iterations):
        it = start_iteration + step
        acts, labs, caches = [], [], []
        for i in range(n_conv):
            x, y = make_batch(it, i)
            a, c = block_forward(front, conv_p, x)
            acts.append(a)
            labs.append(np.asarray(y, dtype=F32).astype(np.int64))
            caches.append(c)
        boundary = [None] * n_conv
        fc_vecs, loss_sum = [], 0.0
        for f in range(n_fc):
            xs = np.concatenate([acts[i] for i in members[f]])
            ys = np.concatenate([labs[i] for i in members[f]])
            out, fcache = block_forward(back, fc_p, xs, labels=ys)
            gx, g = block_backward(back, fc_p, fcache, None)
            fc_vecs.append(_flat(g))
            loss_sum += float(out.sum())
            for pos, i in enumerate(members[f]):
                boundary[i] = gx[pos * batch_k:(pos + 1) * batch_k]
        conv_vecs = []
        for i in range(n_conv):
            _, g = block_backward(front, conv_p, caches[i], boundary[i])
            conv_vecs.append(_flat(g))
        ar_seed = seed * 1_000_003 + it
        conv_sum = allreduce_sum(conv_vecs, ar_seed)
        fc_sum = allreduce_sum(fc_vecs, ar_seed) if n_fc > 1 else fc_vecs[0]
        sgd_update(conv_p, _unflat(conv_sum, conv_p), conv_v, n, lr, mu)
        sgd_update(fc_p, _unflat(fc_sum, fc_p), fc_v, n, lr, mu)
        losses.append(loss_sum / n)
    return conv_p + fc_p, conv_v + fc_v, losses


def rel_err(a, b):
    """Per-tensor max|a-b| / max(|a|,|b|) (tests/oracles.py, rel_err)."""
    a = np.asarray(a, F64)
    b = np.asarray(b, F64)
    scale = max(np.abs(a).max(initial=0.0), np.abs(b).max(initial=0.0), 1e-8)
    return float(np.abs(a - b).max(initial=0.0) / scale)


def max_param_dev(a, b):
    """tests/trainers.py:58-60: worst per-tensor relative deviation."""
    return max(rel_err(x, y) for la, lb in zip(a, b) for x, y in zip(la, lb))


# ---------------------------------------------------------------------------
# executable model stacks (model_partition.py:311-330)
# ---------------------------------------------------------------------------

def tiny_cnn_layers(side=16):
    """tiny_cnn (model_partition.py:311-319); side=32 is the A=1024 variant."""
    a = 16 * (side // 4) * (side // 4)
    return [("conv", 3, 8, 3, 1, 1), ("relu",), ("maxpool", 2, 2),
            ("conv", 8, 16, 3, 1, 1), ("relu",), ("maxpool", 2, 2),
            ("flatten",), ("fc", a, 128), ("relu",), ("fc", 128, 10),
            ("softmax_ce",)], (3, side, side)


def tiny_mlp_layers():
    """tiny_mlp (model_partition.py:322-330)."""
    return [("fc", 64, 48), ("relu",), ("fc", 48, 48), ("relu",),
            ("fc", 48, 96), ("relu",), ("fc", 96, 10), ("softmax_ce",)], (64,)


def alexnet_layers():
    """Single-tower AlexNet in the reference grammar."""
    return [("conv", 3, 64, 11, 4, 2), ("relu",), ("maxpool", 3, 2),
            ("conv", 64, 192, 5, 1, 2), ("relu",), ("maxpool", 3, 2),
            ("conv", 192, 384, 3, 1, 1), ("relu",),
            ("conv", 384, 256, 3, 1, 1), ("relu",),
            ("conv", 256, 256, 3, 1, 1), ("relu",), ("maxpool", 3, 2),
            ("flatten",), ("fc", 9216, 4096), ("relu",),
            ("fc", 4096, 4096), ("relu",), ("fc", 4096, 1000),
            ("softmax_ce",)], (3, 224, 224)


def resnet_layers(blocks=(3, 4, 6, 3), widths=(64, 128, 256, 512), side=224, stem=64,
                  expansion=4, classes=1000, stem_kernel=7, eps=1e-5):
    """Post-activation bottleneck ResNet (ResNet-50 with the defaults) in the
    tuple grammar (§8f row 4).  The reference's MaxPool2d has no padding, so
    the stem pool is an unpadded 3x3/2 (112 -> 55; the stages then give 28,
    14, 7).  Conv layers keep their bias (the reference's Conv2d always has
    one)."""
    layers = [("conv", 3, stem, stem_kernel, 2, stem_kernel // 2), ("bn", stem, eps), ("relu",),
              ("maxpool", 3, 2)]
    cin = stem
    for si, (n, w) in enumerate(zip(blocks, widths)):
        for b in range(n):
            s = 2 if (b == 0 and si > 0) else 1
            cout = w * expansion
            body = (("conv", cin, w, 1, 1, 0), ("bn", w, eps), ("relu",),
                    ("conv", w, w, 3, s, 1), ("bn", w, eps), ("relu",),
                    ("conv", w, cout, 1, 1, 0), ("bn", cout, eps))
            short = ((("conv", cin, cout, 1, s, 0), ("bn", cout, eps))
                     if (s != 1 or cin != cout) else ())
            layers.append(("residual", body, short))
            cin = cout
    layers += [("gap",), ("flatten",), ("fc", cin, classes), ("softmax_ce",)]
    return layers, (3, side, side)


def tiny_resnet_layers():
    """Two bottleneck stages on 16x16 inputs (parity-sized, §8f row 4):
    strided stem (space-to-depth on the GPU), a projection shortcut in each
    stage (stride 1, then stride 2), and an identity block."""
    return resnet_layers(blocks=(2, 1), widths=(8, 16), side=16, stem=8, expansion=2,
                         classes=10, stem_kernel=3)


def vgg16_layers():
    """VGG-16 in the reference grammar."""
    layers, cin = [], 3
    for stage in ((64, 64), (128, 128), (256, 256, 256), (512, 512, 512),
                  (512, 512, 512)):
        for cout in stage:
            layers += [("conv", cin, cout, 3, 1, 1), ("relu",)]
            cin = cout
        layers.append(("maxpool", 2, 2))
    layers += [("flatten",), ("fc", 25088, 4096), ("relu",), ("fc", 4096, 4096),
               ("relu",), ("fc", 4096, 1000), ("softmax_ce",)]
    return layers, (3, 224, 224)
