"""Layer kinds and the per-layer operator contract, on the B200.

Drop-in for the reference's numeric core (/root/reference/pkg/src/stanza/
tensor_core.py): the same layer dataclasses and field names, the same
``forward(layer, params, x, labels=None) -> (y, cache)`` /
``backward(layer, params, cache, gy) -> (gx, [gW, gb])`` contract
(gradients are batch SUMS), ``seeded_init`` and ``sgd_step`` -- but tensors
are CUDA ``torch.Tensor``s in the reference layouts and every op is a call
into the sm_100a C ABI (include/stanza_b200.h).  There is no CPU path.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Sequence, Union

import numpy as np
import torch

from . import _lib

FLOAT = np.float32


class ShapeMismatch(ValueError):
    """Input shape is incompatible with the layer (tensor_core.py:25-26)."""


class CorruptCheckpoint(ValueError):
    """Serialized parameter blob failed validation (tensor_core.py:29-30)."""


# ---------------------------------------------------------------------------
# layer kinds (tensor_core.py:37-74)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Conv2d:
    in_ch: int
    out_ch: int
    kernel: int
    stride: int = 1
    padding: int = 0
    # Inception-V3 kinds (§8f row 4, not in the reference): an asymmetric
    # kernel kernel x kernel_w with padding (padding, padding_w); None = square
    kernel_w: int | None = None
    padding_w: int | None = None

    @property
    def kh(self) -> int:
        return self.kernel

    @property
    def kw(self) -> int:
        return self.kernel if self.kernel_w is None else self.kernel_w

    @property
    def ph(self) -> int:
        return self.padding

    @property
    def pw(self) -> int:
        return self.padding if self.padding_w is None else self.padding_w

    @property
    def square(self) -> bool:
        return self.kh == self.kw and self.ph == self.pw


@dataclass(frozen=True)
class MaxPool2d:
    kernel: int
    stride: int


@dataclass(frozen=True)
class Flatten:
    pass


@dataclass(frozen=True)
class FullyConnected:
    in_dim: int
    out_dim: int


@dataclass(frozen=True)
class ReLU:
    pass


@dataclass(frozen=True)
class SoftmaxCrossEntropy:
    pass


# -- ResNet-trunk kinds.  The reference has none of these
# (tensor_core.py:37-74 stops at SoftmaxCrossEntropy); their semantics are
# defined by oracle/stanza_oracle.py (bn_forward / gap_forward / residual) and
# their parity is unpinned.  They run only through the block engine.

@dataclass(frozen=True)
class BatchNorm2d:
    """Training-mode batch normalisation over (N, H, W) of each CONV worker's
    batch; gamma / beta [C] initialised to 1 / 0 without an RNG draw."""
    channels: int
    eps: float = 1e-5


@dataclass(frozen=True)
class GlobalAvgPool2d:
    """(C, H, W) -> (C, 1, 1)."""


@dataclass(frozen=True)
class Residual:
    """relu(body(x) + shortcut(x)); an empty shortcut is the identity.  Its
    parameter row is the body's tensors then the shortcut's."""
    body: tuple
    shortcut: tuple = ()


# -- Inception-V3 kinds (§8f row 4; semantics in oracle/stanza_oracle.py
# avgpool_* / "concat", parity unpinned like the ResNet kinds)

@dataclass(frozen=True)
class AvgPool2d:
    """Zero-padded average pool; every window is divided by kernel^2."""
    kernel: int
    stride: int
    padding: int = 0


@dataclass(frozen=True)
class Concat:
    """Branches applied to the same input, outputs concatenated along
    channels in branch order (an Inception module).  Its parameter row is
    every branch's tensors in order."""
    branches: tuple


LayerKind = Union[Conv2d, MaxPool2d, Flatten, FullyConnected, ReLU, SoftmaxCrossEntropy,
                  BatchNorm2d, GlobalAvgPool2d, Residual, AvgPool2d, Concat]


def has_params(layer) -> bool:
    if isinstance(layer, (Residual, Concat)):
        return bool(param_shapes(layer))
    return isinstance(layer, (Conv2d, FullyConnected, BatchNorm2d))


def param_shapes(layer) -> list[tuple[int, ...]]:
    """Weight then bias: conv [O,C,k,k]+[O], FC [in,out]+[out] (tensor_core.py:81-88);
    BatchNorm gamma+beta [C]; a residual block its sub-layers' in order."""
    if isinstance(layer, Conv2d):
        return [(layer.out_ch, layer.in_ch, layer.kh, layer.kw), (layer.out_ch,)]
    if isinstance(layer, FullyConnected):
        return [(layer.in_dim, layer.out_dim), (layer.out_dim,)]
    if isinstance(layer, BatchNorm2d):
        return [(layer.channels,), (layer.channels,)]
    if isinstance(layer, Residual):
        return [s for l in layer.body + layer.shortcut for s in param_shapes(l)]
    if isinstance(layer, Concat):
        return [s for br in layer.branches for l in br for s in param_shapes(l)]
    return []


def param_count(layer) -> int:
    return sum(int(np.prod(s)) for s in param_shapes(layer))


def fan_in(layer) -> int:
    if isinstance(layer, Conv2d):
        return layer.in_ch * layer.kh * layer.kw
    if isinstance(layer, FullyConnected):
        return layer.in_dim
    raise ValueError(f"{layer!r} has no parameters")


def out_shape(layer, in_shape: tuple[int, ...]) -> tuple[int, ...]:
    """Per-sample output shape; ShapeMismatch when the input cannot feed the
    layer (tensor_core.py:103-140)."""
    in_shape = tuple(in_shape)
    if isinstance(layer, Conv2d):
        if len(in_shape) != 3 or in_shape[0] != layer.in_ch:
            raise ShapeMismatch(f"Conv2d expects ({layer.in_ch}, H, W), got {in_shape}")
        oh = (in_shape[1] + 2 * layer.ph - layer.kh) // layer.stride + 1
        ow = (in_shape[2] + 2 * layer.pw - layer.kw) // layer.stride + 1
        if oh <= 0 or ow <= 0:
            raise ShapeMismatch(f"Conv2d kernel {layer.kh}x{layer.kw} too large for {in_shape}")
        return (layer.out_ch, oh, ow)
    if isinstance(layer, MaxPool2d):
        if len(in_shape) != 3:
            raise ShapeMismatch(f"MaxPool2d expects (C, H, W), got {in_shape}")
        oh = (in_shape[1] - layer.kernel) // layer.stride + 1
        ow = (in_shape[2] - layer.kernel) // layer.stride + 1
        if oh <= 0 or ow <= 0:
            raise ShapeMismatch(f"MaxPool2d kernel {layer.kernel} too large for {in_shape}")
        return (in_shape[0], oh, ow)
    if isinstance(layer, AvgPool2d):
        if len(in_shape) != 3:
            raise ShapeMismatch(f"AvgPool2d expects (C, H, W), got {in_shape}")
        oh = (in_shape[1] + 2 * layer.padding - layer.kernel) // layer.stride + 1
        ow = (in_shape[2] + 2 * layer.padding - layer.kernel) // layer.stride + 1
        if oh <= 0 or ow <= 0 or layer.padding * 2 > layer.kernel:
            raise ShapeMismatch(f"AvgPool2d kernel {layer.kernel} pad {layer.padding} does "
                                f"not fit {in_shape}")
        return (in_shape[0], oh, ow)
    if isinstance(layer, Concat):
        if not layer.branches or any(not br for br in layer.branches):
            raise ShapeMismatch("Concat needs non-empty branches")
        outs = []
        for br in layer.branches:
            shape = in_shape
            for l in br:
                shape = out_shape(l, shape)
            if len(shape) != 3:
                raise ShapeMismatch(f"Concat branch ends in {shape}, expected (C, H, W)")
            outs.append(shape)
        if len({o[1:] for o in outs}) != 1:
            raise ShapeMismatch(f"Concat branches disagree on H, W: {outs}")
        return (sum(o[0] for o in outs), outs[0][1], outs[0][2])
    if isinstance(layer, Flatten):
        return (int(np.prod(in_shape)),)
    if isinstance(layer, FullyConnected):
        if len(in_shape) != 1 or in_shape[0] != layer.in_dim:
            raise ShapeMismatch(f"FullyConnected expects ({layer.in_dim},), got {in_shape}")
        return (layer.out_dim,)
    if isinstance(layer, ReLU):
        return in_shape
    if isinstance(layer, SoftmaxCrossEntropy):
        if len(in_shape) != 1:
            raise ShapeMismatch(f"SoftmaxCrossEntropy expects logits (C,), got {in_shape}")
        return ()
    if isinstance(layer, BatchNorm2d):
        if len(in_shape) != 3 or in_shape[0] != layer.channels:
            raise ShapeMismatch(f"BatchNorm2d expects ({layer.channels}, H, W), got {in_shape}")
        return in_shape
    if isinstance(layer, GlobalAvgPool2d):
        if len(in_shape) != 3:
            raise ShapeMismatch(f"GlobalAvgPool2d expects (C, H, W), got {in_shape}")
        return (in_shape[0], 1, 1)
    if isinstance(layer, Residual):
        if not layer.body:
            raise ShapeMismatch("Residual needs a non-empty body")
        shape = in_shape
        for l in layer.body:
            shape = out_shape(l, shape)
        short = in_shape
        for l in layer.shortcut:
            short = out_shape(l, short)
        if shape != short:
            raise ShapeMismatch(f"Residual body gives {shape}, shortcut gives {short}")
        return shape
    raise TypeError(f"unknown layer kind {layer!r}")


def as_tuple(layer) -> tuple:
    """Plain-tuple form of a layer (the oracle's and the tests' vocabulary)."""
    if isinstance(layer, Conv2d):
        if not layer.square:
            return ("conv", layer.in_ch, layer.out_ch, (layer.kh, layer.kw), layer.stride,
                    (layer.ph, layer.pw))
        return ("conv", layer.in_ch, layer.out_ch, layer.kernel, layer.stride, layer.padding)
    if isinstance(layer, MaxPool2d):
        return ("maxpool", layer.kernel, layer.stride)
    if isinstance(layer, Flatten):
        return ("flatten",)
    if isinstance(layer, FullyConnected):
        return ("fc", layer.in_dim, layer.out_dim)
    if isinstance(layer, ReLU):
        return ("relu",)
    if isinstance(layer, SoftmaxCrossEntropy):
        return ("softmax_ce",)
    if isinstance(layer, BatchNorm2d):
        return ("bn", layer.channels, layer.eps)
    if isinstance(layer, GlobalAvgPool2d):
        return ("gap",)
    if isinstance(layer, Residual):
        return ("residual", tuple(as_tuple(l) for l in layer.body),
                tuple(as_tuple(l) for l in layer.shortcut))
    if isinstance(layer, AvgPool2d):
        return ("avgpool", layer.kernel, layer.stride, layer.padding)
    if isinstance(layer, Concat):
        return ("concat", tuple(tuple(as_tuple(l) for l in br) for br in layer.branches))
    raise TypeError(f"unknown layer kind {layer!r}")


# ---------------------------------------------------------------------------
# device plumbing
# ---------------------------------------------------------------------------

_WORKSPACE: dict = {}
WORKSPACE_BYTES = 256 << 20


def workspace(device, key: str | None = None) -> torch.Tensor:
    """Per-device split-K scratch (the ABI itself never allocates); ``key``
    names a separate one for work issued on another stream concurrently
    (the single-device FC weight gradients on the side stream)."""
    dev = torch.device(device)
    ws = _WORKSPACE.get((dev, key))
    if ws is None:
        ws = torch.empty(WORKSPACE_BYTES, dtype=torch.uint8, device=dev)
        _WORKSPACE[(dev, key)] = ws
    return ws


def ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def stream_of(device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _need_cuda(x: torch.Tensor, what: str) -> None:
    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise TypeError(f"{what}: expected a CUDA tensor (there is no CPU path)")
    if x.dtype != torch.float32 or not x.is_contiguous():
        raise TypeError(f"{what}: expected a contiguous float32 tensor")


def _check_batch(layer, x, rank):
    if x.dim() != rank:
        raise ShapeMismatch(f"{type(layer).__name__} expects {rank}-d batched input, "
                            f"got shape {tuple(x.shape)}")


# ---------------------------------------------------------------------------
# operator contract (tensor_core.py:153-301)
# ---------------------------------------------------------------------------

def forward(layer, params: Sequence[torch.Tensor], x: torch.Tensor, labels=None):
    """Run one layer over a batch on the GPU.  Returns (output, cache).

    For SoftmaxCrossEntropy the output is the per-sample loss vector and
    ``labels`` (integer class ids) is required; the logits gradient is
    produced in the same pass and kept in the cache.
    """
    _need_cuda(x, type(layer).__name__)
    dev = x.device
    st = stream_of(dev)
    ws = workspace(dev)
    if isinstance(layer, Conv2d):
        _check_batch(layer, x, 4)
        if x.shape[1] != layer.in_ch:
            raise ShapeMismatch(f"Conv2d expects {layer.in_ch} channels, got {x.shape[1]}")
        n, c, h, w = x.shape
        _, oh, ow = out_shape(layer, (c, h, w))
        y = torch.empty((n, layer.out_ch, oh, ow), device=dev, dtype=torch.float32)
        _lib.call("stz_conv2d_fwd", ptr(x), ptr(params[0]), ptr(params[1]), ptr(y), n, c, h, w,
                  layer.out_ch, layer.kernel, layer.stride, layer.padding, 0, ptr(ws),
                  ws.numel(), st)
        return y, x
    if isinstance(layer, MaxPool2d):
        _check_batch(layer, x, 4)
        n, c, h, w = x.shape
        _, oh, ow = out_shape(layer, (c, h, w))
        y = torch.empty((n, c, oh, ow), device=dev, dtype=torch.float32)
        arg = torch.empty((n, c, oh, ow), device=dev, dtype=torch.uint8)
        _lib.call("stz_maxpool2d_fwd", ptr(x), ptr(y), ptr(arg), n, c, h, w, layer.kernel,
                  layer.stride, st)
        return y, (arg, tuple(x.shape))
    if isinstance(layer, Flatten):
        if x.dim() < 2:
            raise ShapeMismatch(f"Flatten expects batched input, got shape {tuple(x.shape)}")
        return x.reshape(x.shape[0], -1), tuple(x.shape)
    if isinstance(layer, FullyConnected):
        _check_batch(layer, x, 2)
        if x.shape[1] != layer.in_dim:
            raise ShapeMismatch(f"FullyConnected expects dim {layer.in_dim}, got {x.shape[1]}")
        y = torch.empty((x.shape[0], layer.out_dim), device=dev, dtype=torch.float32)
        _lib.call("stz_fc_fwd", ptr(x), ptr(params[0]), ptr(params[1]), ptr(y), x.shape[0],
                  layer.in_dim, layer.out_dim, 0, ptr(ws), ws.numel(), st)
        return y, x
    if isinstance(layer, ReLU):
        y = torch.empty_like(x)
        _lib.call("stz_relu_fwd", ptr(x), ptr(y), x.numel(), st)
        return y, y
    if isinstance(layer, SoftmaxCrossEntropy):
        _check_batch(layer, x, 2)
        if labels is None:
            raise ValueError("SoftmaxCrossEntropy needs labels")
        lab = torch.as_tensor(labels).to(device=dev, dtype=torch.int32).contiguous()
        if lab.shape[0] != x.shape[0]:
            raise ShapeMismatch(f"{lab.shape[0]} labels for batch of {x.shape[0]}")
        losses = torch.empty(x.shape[0], device=dev, dtype=torch.float32)
        dz = torch.empty_like(x)
        _lib.call("stz_softmax_ce", ptr(x), ptr(lab), ptr(losses), ptr(dz), x.shape[0],
                  x.shape[1], st)
        return losses, dz
    raise TypeError(f"unknown layer kind {layer!r}")


def backward(layer, params: Sequence[torch.Tensor], cache, gy):
    """Backward for one layer.  Returns (grad_input, param_grad_list); param
    grads are sums over the batch.  gy is ignored for SoftmaxCrossEntropy."""
    if isinstance(layer, SoftmaxCrossEntropy):
        return cache, []
    _need_cuda(gy, type(layer).__name__)
    dev = gy.device
    st = stream_of(dev)
    ws = workspace(dev)
    if isinstance(layer, Conv2d):
        x = cache
        n, c, h, w = x.shape
        gx = torch.empty_like(x)
        gw = torch.empty_like(params[0])
        gb = torch.empty_like(params[1])
        args = (n, c, h, w, layer.out_ch, layer.kernel, layer.stride, layer.padding,
                ptr(ws), ws.numel(), st)
        _lib.call("stz_conv2d_bwd_data", ptr(gy), ptr(params[0]), ptr(gx), ptr(None), *args)
        _lib.call("stz_conv2d_bwd_filter", ptr(x), ptr(gy), ptr(gw), ptr(gb), *args)
        return gx, [gw, gb]
    if isinstance(layer, MaxPool2d):
        arg, shape = cache
        gx = torch.empty(shape, device=dev, dtype=torch.float32)
        _lib.call("stz_maxpool2d_bwd", ptr(gy), ptr(arg), ptr(gx), ptr(None), *shape,
                  layer.kernel, layer.stride, st)
        return gx, []
    if isinstance(layer, Flatten):
        return gy.reshape(cache), []
    if isinstance(layer, FullyConnected):
        x = cache
        m = x.shape[0]
        gx = torch.empty_like(x)
        gw = torch.empty_like(params[0])
        gb = torch.empty_like(params[1])
        _lib.call("stz_fc_bwd_data", ptr(gy), ptr(params[0]), ptr(gx), ptr(None), m,
                  layer.in_dim, layer.out_dim, ptr(ws), ws.numel(), st)
        _lib.call("stz_fc_bwd_weight", ptr(x), ptr(gy), ptr(gw), ptr(gb), m, layer.in_dim,
                  layer.out_dim, ptr(ws), ws.numel(), st)
        return gx, [gw, gb]
    if isinstance(layer, ReLU):
        gx = torch.empty_like(gy)
        _lib.call("stz_relu_bwd", ptr(gy), ptr(cache), ptr(gx), gy.numel(), st)
        return gx, []
    raise TypeError(f"unknown layer kind {layer!r}")


def block_forward(layers, params, x, labels=None):
    """Forward through a list of layers (tensor_core.py:304-311)."""
    caches = []
    for layer, p in zip(layers, params):
        x, cache = forward(layer, p, x, labels=labels)
        caches.append(cache)
    return x, caches


def block_backward(layers, params, caches, gy):
    """Backward through a block (tensor_core.py:314-325)."""
    grads = [[] for _ in layers]
    for i in range(len(layers) - 1, -1, -1):
        gy, g = backward(layers[i], params[i], caches[i], gy)
        grads[i] = g
    return gy, grads


# ---------------------------------------------------------------------------
# init and optimizer (tensor_core.py:332-388)
# ---------------------------------------------------------------------------

def seeded_init(layers, seed: int) -> list[list[np.ndarray]]:
    """Host-side fan-in uniform init, bit-identical to the reference: one
    PCG64(seed) stream, U[-s, s] with s = sqrt(1/fan_in), weight then bias,
    layer order (tensor_core.py:332-346).  Upload with ``to_device``."""
    gen = np.random.Generator(np.random.PCG64(seed))
    return [_init_layer(gen, layer) for layer in layers]


def _init_layer(gen, layer) -> list[np.ndarray]:
    if isinstance(layer, BatchNorm2d):      # §8f kinds: no draw for gamma / beta
        return [np.ones(layer.channels, FLOAT), np.zeros(layer.channels, FLOAT)]
    if isinstance(layer, Residual):
        return [t for l in layer.body + layer.shortcut for t in _init_layer(gen, l)]
    if isinstance(layer, Concat):
        return [t for br in layer.branches for l in br for t in _init_layer(gen, l)]
    bound = float(np.sqrt(1.0 / fan_in(layer))) if has_params(layer) else 0.0
    return [gen.uniform(-bound, bound, size=s).astype(FLOAT) for s in param_shapes(layer)]


def to_device(nested, device) -> list[list[torch.Tensor]]:
    return [[torch.from_numpy(np.ascontiguousarray(t)).to(device) for t in layer]
            for layer in nested]


@dataclass
class OptimizerState:
    """Momentum-SGD state for one parameter set (tensor_core.py:349-363)."""
    lr: float
    momentum: float = 0.9
    velocity: list = field(default_factory=list)

    def __post_init__(self):
        if not 0.0 <= self.momentum < 1.0:
            raise ValueError(f"momentum must be in [0, 1), got {self.momentum}")

    @classmethod
    def for_params(cls, params, lr: float, momentum: float = 0.9) -> "OptimizerState":
        return cls(lr=lr, momentum=momentum,
                   velocity=[[torch.zeros_like(t) for t in layer] for layer in params])


def inv_batch(n: int) -> float:
    """float32(1) / float32(n), exactly as tensor_core.py:376."""
    return float(FLOAT(1.0) / FLOAT(n))


def sgd_step(params, grads_sum, n: int, opt: OptimizerState):
    """One momentum-SGD step from gradient sums over n samples, in place on
    the device, reference fp32 op order (tensor_core.py:366-388)."""
    inv_n = inv_batch(n)
    for li, layer_params in enumerate(params):
        for ti, w in enumerate(layer_params):
            g = grads_sum[li][ti]
            if tuple(g.shape) != tuple(w.shape):
                raise ShapeMismatch(f"grad shape {tuple(g.shape)} vs param shape "
                                    f"{tuple(w.shape)}")
            v = opt.velocity[li][ti]
            _lib.call("stz_sgd_momentum", ptr(w), ptr(v), ptr(g.contiguous()), w.numel(),
                      float(opt.lr), float(opt.momentum), inv_n, stream_of(w.device))
    return params
