"""Fused execution of one block (CONV trunk or FC head) on one GPU.

A ``BlockEngine`` owns, for a fixed batch size:

* flat parameter / velocity / gradient buffers for its block (one tensor
  each; per-layer views in the reference layouts -- conv W [O,C,k,k], FC W
  [in,out] -- each view 16-byte aligned), so the gradient allreduce and the
  momentum step are single calls over one vector (no pack/unpack,
  reference tensor_core.py:501-524);
* preallocated activation, argmax and gradient buffers (no allocation per
  step, so a whole step can be captured in a CUDA graph);
* a fused plan over the C ABI: conv/FC + following ReLU fuse into the GEMM
  epilogue; a ReLU's backward fuses into the input-gradient kernel of the
  layer that consumed it (conv/FC dgrad or max-pool backward, skipping
  Flatten, which is a view); SoftmaxCE emits loss and dlogits in one pass;
  the first layer of the CONV block skips its input gradient, which the
  reference computes and discards (stanza_runtime.py:366-369).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .tensor_core import (Conv2d, Flatten, FullyConnected, MaxPool2d, ReLU,
                          ShapeMismatch, SoftmaxCrossEntropy, inv_batch, out_shape,
                          param_shapes, ptr, stream_of, workspace)

_ALIGN = 4  # floats: keeps every per-tensor view 16-byte aligned


def _aligned(n: int) -> int:
    return (n + _ALIGN - 1) // _ALIGN * _ALIGN


@dataclass
class _Op:
    kind: str                 # conv | fc | maxpool | relu | flatten | softmax_ce
    layer: object
    index: int                # layer index within the block
    in_shape: tuple           # per-sample
    out_shape: tuple          # per-sample
    fused_relu: bool = False  # conv/fc: epilogue applies the following ReLU
    mask_from: int = -1       # bwd: op index whose output masks this op's input grad
    relu_bwd_fused: bool = False  # relu: its backward is done by its consumer
    skip_dgrad: bool = False


class BlockEngine:
    """One block of layers bound to a device, a batch size and flat buffers."""

    def __init__(self, layers, in_shape, batch: int, device, params=None, velocities=None,
                 need_input_grad: bool = True, shared=None, input_grad_buffer=None):
        self.layers = tuple(layers)
        self.in_shape = tuple(in_shape)
        self.batch = int(batch)
        self.device = torch.device(device)
        self.need_input_grad = need_input_grad
        self._build_plan()
        self._layout_params()
        dev, f32 = self.device, torch.float32
        if shared is not None:                   # FC replicas on one GPU share (w, v)
            if shared.total != self.total:
                raise ShapeMismatch("shared engine has a different parameter layout")
            self.params_flat, self.vel_flat = shared.params_flat, shared.vel_flat
        else:
            self.params_flat = torch.zeros(self.total, dtype=f32, device=dev)
            self.vel_flat = torch.zeros(self.total, dtype=f32, device=dev)
        self.grad_flat = torch.zeros(self.total, dtype=f32, device=dev)
        self.params = self._views(self.params_flat)
        self.velocity = self._views(self.vel_flat)
        self.grads = self._views(self.grad_flat)
        if shared is None and params is not None:
            self.load(params, velocities)
        self._alloc_activations(input_grad_buffer)

    # -- plan ------------------------------------------------------------------

    def _build_plan(self):
        ops, shape = [], self.in_shape
        for i, layer in enumerate(self.layers):
            kind = {Conv2d: "conv", FullyConnected: "fc", MaxPool2d: "maxpool", ReLU: "relu",
                    Flatten: "flatten", SoftmaxCrossEntropy: "softmax_ce"}[type(layer)]
            nxt = out_shape(layer, shape)
            ops.append(_Op(kind, layer, i, shape, nxt))
            shape = nxt
        self.out_shape = shape
        for i, op in enumerate(ops):
            if op.kind == "relu" and i > 0 and ops[i - 1].kind in ("conv", "fc"):
                ops[i - 1].fused_relu = True
        # ReLU backward goes into the input-gradient kernel of its consumer
        for i, op in enumerate(ops):
            if op.kind != "relu":
                continue
            j = i + 1
            while j < len(ops) and ops[j].kind == "flatten":
                j += 1
            if j < len(ops) and ops[j].kind in ("conv", "fc", "maxpool"):
                ops[j].mask_from = i
                op.relu_bwd_fused = True
        if ops and not self.need_input_grad:
            ops[0].skip_dgrad = True
        self.ops = ops

    def _layout_params(self):
        self.slots, off = [], 0
        for layer in self.layers:
            row = []
            for shp in param_shapes(layer):
                n = int(np.prod(shp))
                row.append((off, shp, n))
                off += _aligned(n)
            self.slots.append(row)
        self.total = max(off, _ALIGN)
        self.param_count = sum(n for row in self.slots for _, _, n in row)

    def _views(self, flat):
        return [[flat[o:o + n].view(shp) for (o, shp, n) in row] for row in self.slots]

    def _alloc_activations(self, input_grad_buffer):
        dev, b, f32 = self.device, self.batch, torch.float32
        self.acts: list = [None] * len(self.ops)
        self.args: list = [None] * len(self.ops)
        self.gin: list = [None] * len(self.ops)   # gradient wrt each op's input
        self.losses = None
        self.dlogits = None
        for i, op in enumerate(self.ops):
            if op.kind == "relu" and i > 0 and self.ops[i - 1].fused_relu:
                continue                          # aliases its producer's output
            if op.kind == "flatten":
                continue                          # view of its input
            if op.kind == "softmax_ce":
                self.losses = torch.zeros(b, dtype=f32, device=dev)
                self.dlogits = torch.zeros((b, *op.in_shape), dtype=f32, device=dev)
                continue
            self.acts[i] = torch.zeros((b, *op.out_shape), dtype=f32, device=dev)
            if op.kind == "maxpool":
                self.args[i] = torch.zeros((b, *op.out_shape), dtype=torch.uint8, device=dev)
        for i, op in enumerate(self.ops):
            if op.kind in ("flatten", "softmax_ce"):
                continue
            if op.kind == "relu" and op.relu_bwd_fused:
                continue
            if i == 0:
                if not self.need_input_grad:
                    continue
                if input_grad_buffer is not None:
                    self.gin[0] = input_grad_buffer
                    continue
            self.gin[i] = torch.zeros((b, *op.in_shape), dtype=f32, device=dev)
        self.loss_sum = torch.zeros(1, dtype=torch.float64, device=dev)

    # -- parameters --------------------------------------------------------------

    def load(self, params, velocities=None):
        """Upload nested numpy (or tensor) params/velocities in reference layout."""
        for li, row in enumerate(self.slots):
            for ti, _ in enumerate(row):
                self.params[li][ti].copy_(torch.as_tensor(np.asarray(params[li][ti])))
                if velocities is not None:
                    self.velocity[li][ti].copy_(torch.as_tensor(np.asarray(velocities[li][ti])))

    def state_numpy(self):
        """(params, velocities) as nested fp32 numpy arrays, reference layout."""
        p = [[t.detach().cpu().numpy().copy() for t in row] for row in self.params]
        v = [[t.detach().cpu().numpy().copy() for t in row] for row in self.velocity]
        return p, v

    # -- execution ------------------------------------------------------------------

    def _act(self, i):
        """Output buffer of op i (resolving ReLU / Flatten aliases)."""
        op = self.ops[i]
        if op.kind == "flatten" or (op.kind == "relu" and self.acts[i] is None):
            src = self._act(i - 1) if i > 0 else self._x
            return src.reshape((self.batch, *op.out_shape))
        return self.acts[i]

    def _input(self, i):
        return self._x if i == 0 else self._act(i - 1)

    def forward(self, x: torch.Tensor, labels: torch.Tensor | None = None,
                loss_out: torch.Tensor | None = None):
        """Run the block on x [batch, *in_shape]; returns the block output
        (per-sample losses for a loss block).  The float64 loss sum goes to
        ``loss_sum``, or is ADDED into ``loss_out`` when given."""
        if tuple(x.shape) != (self.batch, *self.in_shape):
            raise ShapeMismatch(f"block expects {(self.batch, *self.in_shape)}, "
                                f"got {tuple(x.shape)}")
        self._x = x
        self._labels = labels
        st = stream_of(self.device)
        ws = workspace(self.device)
        b = self.batch
        for i, op in enumerate(self.ops):
            xin = self._input(i)
            if op.kind == "conv":
                l = op.layer
                c, h, w = op.in_shape
                _lib.call("stz_conv2d_fwd", ptr(xin), ptr(self.params[i][0]),
                          ptr(self.params[i][1]), ptr(self.acts[i]), b, c, h, w, l.out_ch,
                          l.kernel, l.stride, l.padding, int(op.fused_relu), ptr(ws),
                          ws.numel(), st)
            elif op.kind == "fc":
                l = op.layer
                _lib.call("stz_fc_fwd", ptr(xin), ptr(self.params[i][0]),
                          ptr(self.params[i][1]), ptr(self.acts[i]), b, l.in_dim, l.out_dim,
                          int(op.fused_relu), ptr(ws), ws.numel(), st)
            elif op.kind == "maxpool":
                c, h, w = op.in_shape
                _lib.call("stz_maxpool2d_fwd", ptr(xin), ptr(self.acts[i]), ptr(self.args[i]),
                          b, c, h, w, op.layer.kernel, op.layer.stride, st)
            elif op.kind == "relu":
                if self.acts[i] is not None:
                    _lib.call("stz_relu_fwd", ptr(xin), ptr(self.acts[i]), xin.numel(), st)
            elif op.kind == "softmax_ce":
                if labels is None:
                    raise ValueError("SoftmaxCrossEntropy needs labels")
                _lib.call("stz_softmax_ce", ptr(xin), ptr(labels), ptr(self.losses),
                          ptr(self.dlogits), b, op.in_shape[0], st)
                tgt, acc = (self.loss_sum, 0) if loss_out is None else (loss_out, 1)
                _lib.call("stz_sum_f32", ptr(self.losses), b, ptr(tgt), acc, st)
        return self.losses if self.losses is not None else self._act(len(self.ops) - 1)

    def backward(self, gy: torch.Tensor | None = None):
        """Backward through the block; parameter-gradient sums land in
        ``grad_flat``.  Returns the gradient wrt the block input (None when
        the block was built with need_input_grad=False)."""
        st = stream_of(self.device)
        ws = workspace(self.device)
        b = self.batch
        g = gy
        for i in range(len(self.ops) - 1, -1, -1):
            op = self.ops[i]
            xin = self._input(i)
            mask = self._act(op.mask_from) if op.mask_from >= 0 else None
            if op.kind == "softmax_ce":
                g = self.dlogits
            elif op.kind == "flatten":
                g = g.reshape((b, *op.in_shape))
            elif op.kind == "relu":
                if not op.relu_bwd_fused:
                    out = self.gin[i]
                    _lib.call("stz_relu_bwd", ptr(g), ptr(self._act(i)), ptr(out), g.numel(), st)
                    g = out
            elif op.kind == "maxpool":
                if op.skip_dgrad:
                    g = None
                    continue
                c, h, w = op.in_shape
                out = self.gin[i]
                _lib.call("stz_maxpool2d_bwd", ptr(g), ptr(self.args[i]), ptr(out), ptr(mask),
                          b, c, h, w, op.layer.kernel, op.layer.stride, st)
                g = out
            elif op.kind == "conv":
                l = op.layer
                c, h, w = op.in_shape
                dims = (b, c, h, w, l.out_ch, l.kernel, l.stride, l.padding, ptr(ws),
                        ws.numel(), st)
                _lib.call("stz_conv2d_bwd_filter", ptr(xin), ptr(g), ptr(self.grads[i][0]),
                          ptr(self.grads[i][1]), *dims)
                if op.skip_dgrad:
                    g = None
                    continue
                out = self.gin[i]
                _lib.call("stz_conv2d_bwd_data", ptr(g), ptr(self.params[i][0]), ptr(out),
                          ptr(mask), *dims)
                g = out
            elif op.kind == "fc":
                l = op.layer
                _lib.call("stz_fc_bwd_weight", ptr(xin), ptr(g), ptr(self.grads[i][0]),
                          ptr(self.grads[i][1]), b, l.in_dim, l.out_dim, ptr(ws), ws.numel(),
                          st)
                if op.skip_dgrad:
                    g = None
                    continue
                out = self.gin[i]
                _lib.call("stz_fc_bwd_data", ptr(g), ptr(self.params[i][0]), ptr(out),
                          ptr(mask), b, l.in_dim, l.out_dim, ptr(ws), ws.numel(), st)
                g = out
        return g

    def sgd(self, n: int, lr: float, mu: float, grad: torch.Tensor | None = None):
        """Momentum step over the whole flat block (tensor_core.py:366-388)."""
        g = self.grad_flat if grad is None else grad
        _lib.call("stz_sgd_momentum", ptr(self.params_flat), ptr(self.vel_flat), ptr(g),
                  self.total, float(lr), float(mu), inv_batch(n), stream_of(self.device))

    def add_grads_from(self, other: "BlockEngine"):
        """grad_flat += other.grad_flat (replica gradient sum on one device)."""
        _lib.call("stz_vec_add", ptr(self.grad_flat), ptr(other.grad_flat), self.total,
                  stream_of(self.device))
