"""Fused execution of one block (CONV trunk or FC head) on one GPU.

A ``BlockEngine`` owns, for a fixed batch size:

* fp32 master parameter / velocity / gradient buffers for its block, one
  flat tensor each with per-layer views in the reference layouts (conv W
  [O,C,k,k], FC W [in,out]; every view 16-byte aligned), so the gradient
  allreduce and the momentum step are single calls over one vector (no
  pack/unpack, reference tensor_core.py:501-524);
* split-plane copies of the weights in GEMM-ready layouts (conv forward
  [O][kh][kw][C8], conv input-gradient [C][kh][kw][O8], FC [in][out8]),
  refreshed after every update;
* split-plane activation / gradient buffers (three bf16 planes whose sum is
  the fp32 value exactly; conv tensors NHWC with channels padded to 8, flat
  tensors [rows][D8]), preallocated for the batch so a step never allocates;
* a fused plan over the C ABI (``stzx_*``): conv/FC + following ReLU in the
  GEMM epilogue; a ReLU's backward folded into the input-gradient kernel of
  the layer that consumed it (conv/FC dgrad, max-pool backward); a max-pool
  followed by Flatten writes the CHW-flat (reference flatten order) tensor
  directly; SoftmaxCE emits loss and dlogits in one pass; the first layer of
  the CONV block skips its input gradient (stanza_runtime.py:366-369 discards
  it).

The ResNet-trunk kinds of SURVEY.md §8f row 4 (not in the reference):
BatchNorm2d (statistics per ``group`` of samples = one CONV worker's batch,
following ReLU fused into its apply pass), GlobalAvgPool2d (a following
Flatten is a view), and Residual, run by two child engines (body, shortcut)
whose parameter / velocity / gradient views live inside this engine's flat
vectors; the residual add + ReLU is fused into the body's last BatchNorm.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .tensor_core import (AvgPool2d, BatchNorm2d, Concat, Conv2d, Flatten, FullyConnected,
                          GlobalAvgPool2d, MaxPool2d, ReLU, Residual, ShapeMismatch,
                          SoftmaxCrossEntropy, inv_batch, out_shape, param_shapes, ptr, stream_of,
                          workspace)

_ALIGN = 4  # floats: keeps every fp32 per-tensor view 16-byte aligned


def _aligned(n: int) -> int:
    return (n + _ALIGN - 1) // _ALIGN * _ALIGN


def rup8(n: int) -> int:
    return (n + 7) // 8 * 8


class Split:
    """A split-plane tensor: storage [3, *dims] bf16, plane stride ``ps``.
    layout "nhwc": dims (N, H, W, C8), logical channels C;
    layout "rows": dims (N, D8), logical width D."""

    def __init__(self, storage: torch.Tensor, layout: str, logical: int, row0: int = 0,
                 rows: int | None = None):
        self.storage = storage
        self.layout = layout
        self.logical = logical                       # C (nhwc) or D (rows)
        self.ps = storage[0].numel()
        self.row0 = row0                             # row offset of a slice view
        self.rows = storage.shape[1] if rows is None else rows

    @staticmethod
    def alloc(layout, dims, logical, device):
        return Split(torch.zeros((3, *dims), dtype=torch.bfloat16, device=device), layout,
                     logical)

    @property
    def row_elems(self) -> int:
        return int(np.prod(self.storage.shape[2:]))

    @property
    def width(self) -> int:
        return self.storage.shape[-1]

    def ptr(self) -> int:
        return self.storage.data_ptr() + self.row0 * self.row_elems * 2

    def rows_view(self, lo: int, hi: int) -> "Split":
        s = Split(self.storage, self.layout, self.logical, self.row0 + lo, hi - lo)
        return s

    def plane_rows(self, p: int) -> torch.Tensor:
        """Plane p restricted to this view's rows (a contiguous tensor view)."""
        return self.storage[p, self.row0:self.row0 + self.rows]

    def to_float(self) -> torch.Tensor:
        """Debug read-back: exact fp32 values of this view."""
        planes = [self.plane_rows(p).float() for p in range(3)]
        return (planes[0] + planes[1]) + planes[2]


@dataclass
class _Op:
    kind: str                 # conv | fc | maxpool | relu | flatten | softmax_ce | bn | gap |
    #                           residual | avgpool | concat
    layer: object
    index: int
    in_shape: tuple           # per-sample logical shape
    out_shape: tuple
    fused_relu: bool = False  # conv/fc: epilogue applies the following ReLU
    mask_from: int = -1       # bwd: op whose output (a ReLU output) masks the input grad
    relu_bwd_fused: bool = False
    skip_dgrad: bool = False
    flat_out: bool = False    # maxpool: writes the CHW-flat tensor for a following Flatten
    s2d: tuple | None = None  # first strided conv as space-to-depth: (ks, Cs8, Hs, Ws)
    bias_by_bn: bool = False  # conv: the following BatchNorm's backward sums its bias gradient
    c8_in: int = 0            # conv: input channel stride when not rup8(in_ch) (first layer)


class BlockEngine:
    """One block of layers bound to a device, a batch size and its buffers."""

    def __init__(self, layers, in_shape, batch: int, device, params=None, velocities=None,
                 need_input_grad: bool = True, shared=None, input_grad_buffer=None,
                 allocate: bool = True, group: int | None = None, flats=None, tag: str = ""):
        self.layers = tuple(layers)
        self.in_shape = tuple(in_shape)
        self.batch = int(batch)
        self.device = torch.device(device)
        self.need_input_grad = need_input_grad
        # BatchNorm statistics group (samples): one CONV worker's batch
        self.group = self.batch if group is None else int(group)
        if self.batch % self.group:
            raise ShapeMismatch(f"batch {self.batch} is not a multiple of the group {self.group}")
        self.tag = tag
        self.ws_key = None        # split-K scratch: see tensor_core.workspace
        # (n, lr, mu) while the runtime lets the FC weight gradients apply the
        # momentum step in their epilogue (one FC worker); layers so updated
        self.sgd_in_wgrad = None
        self._sgd_done: set = set()
        # set by the runtime: conv bias column sums run on this stream,
        # concurrently with the rest of the backward (joined before the update)
        self.bias_stream = None
        self._bias_events: dict = {}
        # set by the runtime: (stream, n, lr, mu) -- each conv layer's momentum
        # step + weight repack runs on that stream as soon as its input and
        # weight gradients are issued (joined before the next forward)
        self.update_side = None
        # set by the runtime: conv weight gradients run on this stream, beside
        # the input-gradient chain on the current stream
        self.wgrad_stream = None
        self._wgrad_events: dict = {}
        self._build_plan()
        self._layout_params()
        self.children: dict = {}
        if not allocate:
            return
        dev, f32 = self.device, torch.float32
        if flats is not None:                    # a residual block's child: views of the parent
            base, (pf, vf, gf) = flats
            self.params_flat, self.vel_flat = pf[base:base + self.total], vf[base:base + self.total]
            self.grad_flat = gf[base:base + self.total]
            self.wplanes = self._alloc_weight_planes()
        elif shared is not None:                   # FC replicas on one GPU share (w, v, planes)
            if shared.total != self.total:
                raise ShapeMismatch("shared engine has a different parameter layout")
            self.params_flat, self.vel_flat = shared.params_flat, shared.vel_flat
            self.wplanes = shared.wplanes
        else:
            self.params_flat = torch.zeros(self.total, dtype=f32, device=dev)
            self.vel_flat = torch.zeros(self.total, dtype=f32, device=dev)
            self.wplanes = self._alloc_weight_planes()
        if flats is None:
            self.grad_flat = torch.zeros(self.total, dtype=f32, device=dev)
        self.params = self._views(self.params_flat)
        self.velocity = self._views(self.vel_flat)
        self.grads = self._views(self.grad_flat)
        self._make_children()
        if shared is None and params is not None:
            self.load(params, velocities)
        self._alloc_activations(input_grad_buffer)

    # -- plan ----------------------------------------------------------------------

    def _build_plan(self):
        ops, shape = [], self.in_shape
        for i, layer in enumerate(self.layers):
            kind = {Conv2d: "conv", FullyConnected: "fc", MaxPool2d: "maxpool", ReLU: "relu",
                    Flatten: "flatten", SoftmaxCrossEntropy: "softmax_ce", BatchNorm2d: "bn",
                    GlobalAvgPool2d: "gap", Residual: "residual", AvgPool2d: "avgpool",
                    Concat: "concat"}[type(layer)]
            nxt = out_shape(layer, shape)
            ops.append(_Op(kind, layer, i, shape, nxt))
            shape = nxt
        self.out_shape = shape
        for i, op in enumerate(ops):
            if op.kind == "relu" and i > 0 and ops[i - 1].kind in ("conv", "fc", "bn"):
                ops[i - 1].fused_relu = True
            if op.kind == "flatten" and i > 0 and ops[i - 1].kind in ("maxpool", "gap"):
                ops[i - 1].flat_out = True      # gap: (C,1,1) NHWC is the flat row already
        for i, op in enumerate(ops):
            if op.kind == "bn" and i > 0 and ops[i - 1].kind == "conv":
                ops[i - 1].bias_by_bn = True     # gx of that BatchNorm is the conv's output grad
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
            # a strided first conv on few channels (AlexNet conv1) runs as a
            # stride-1 conv over space-to-depth blocks: TMA-eligible channels
            l0 = ops[0].layer
            if ops[0].kind == "conv" and l0.stride > 1 and rup8(l0.in_ch) < 32 \
                    and l0.in_ch * l0.stride ** 2 <= 256 and l0.square:
                ks = -(-l0.kernel // l0.stride)
                cs8 = -(-(l0.in_ch * l0.stride ** 2) // 32) * 32
                _, oh, ow = ops[0].out_shape
                # (ResNet-50's stem padded to 64 channels would take the
                # shifted-window weight gradient, 0.39 -> 0.28 ms, but its
                # im2col forward then multiplies the padding: 0.23 -> 0.34 ms)
                ops[0].s2d = (ks, cs8, oh - 1 + ks, ow - 1 + ks)
            elif ops[0].kind == "conv" and l0.stride == 1 and rup8(l0.in_ch) < 32 \
                    and os.environ.get("STZ_FIRST_C32", "1") != "0":
                # a stride-1 first conv on few channels (VGG-16 conv1_1): its
                # input is packed 32 channels wide (zeros past in_ch), so the
                # forward and the weight gradient run on the TMA GEMM instead
                # of the cp.async fallback that needs no 32-channel k-blocks
                ops[0].c8_in = 32
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

    def _make_children(self):
        """Body / shortcut engines of each Residual op and branch engines of
        each Concat op, their parameters views of this engine's flat vectors
        at the op's row offset."""
        flats = (self.params_flat, self.vel_flat, self.grad_flat)
        for i, op in enumerate(self.ops):
            if op.kind == "concat":
                base = self.slots[i][0][0] if self.slots[i] else 0
                kids = []
                for bi, br in enumerate(op.layer.branches):
                    shp = op.in_shape
                    for l in br:
                        shp = out_shape(l, shp)
                    if shp[0] % 8:
                        raise ShapeMismatch(f"Concat branch {bi} gives {shp[0]} channels: "
                                            "branch widths must be multiples of 8")
                    eng = BlockEngine(br, op.in_shape, self.batch, self.device,
                                      need_input_grad=True, group=self.group, flats=(base, flats),
                                      tag=f"{self.tag}c{i}b{bi}.")
                    base += eng.total if eng.param_count else 0
                    if eng.ops[-1].kind == "relu":     # its backward: the concat's masked copy
                        eng.ops[-1].relu_bwd_fused = True
                    kids.append(eng)
                self.children[i] = tuple(kids)
                continue
            if op.kind != "residual":
                continue
            base = self.slots[i][0][0] if self.slots[i] else 0
            kids = []
            for part, name in ((op.layer.body, "b"), (op.layer.shortcut, "s")):
                if not part:
                    kids.append(None)
                    continue
                eng = BlockEngine(part, op.in_shape, self.batch, self.device,
                                  need_input_grad=True, group=self.group, flats=(base, flats),
                                  tag=f"{self.tag}r{i}{name}.")
                base += eng.total if eng.param_count else 0
                kids.append(eng)
            self.children[i] = tuple(kids)

    def set_workspace_key(self, key: str | None) -> None:
        """Use the split-K scratch named ``key`` (this engine and its children)."""
        self.ws_key = key
        for kids in self.children.values():
            for k in kids:
                if k is not None:
                    k.set_workspace_key(key)

    def has_bn(self) -> bool:
        """Whether the block normalises over its batch (BatchNorm, directly or
        inside a residual block): passes must cover whole sample groups."""
        def walk(layers):
            for l in layers:
                if isinstance(l, BatchNorm2d):
                    return True
                if isinstance(l, Residual) and walk(l.body + l.shortcut):
                    return True
                if isinstance(l, Concat) and any(walk(br) for br in l.branches):
                    return True
            return False
        return walk(self.layers)

    def _alloc_weight_planes(self):
        dev = self.device
        planes = {}
        for i, op in enumerate(self.ops):
            l = op.layer
            if op.kind == "conv":
                kk, c8, o8 = l.kh * l.kw, op.c8_in or rup8(l.in_ch), rup8(l.out_ch)
                if op.s2d is not None:
                    ks, cs8, _, _ = op.s2d
                    kk, c8 = ks * ks, cs8
                wf = torch.zeros((3, l.out_ch, kk * c8), dtype=torch.bfloat16, device=dev)
                wd = None if op.skip_dgrad else torch.zeros((3, l.in_ch, kk * o8),
                                                            dtype=torch.bfloat16, device=dev)
                planes[i] = (wf, wd)
            elif op.kind == "fc":
                planes[i] = (torch.zeros((3, l.in_dim, rup8(l.out_dim)), dtype=torch.bfloat16,
                                         device=dev), None)
        return planes

    # -- buffers -------------------------------------------------------------------

    def _split_for(self, shape, rows: int, flat_from_nhwc: bool = False):
        dev = self.device
        if len(shape) == 3:
            c, h, w = shape
            return Split.alloc("nhwc", (rows, h, w, rup8(c)), c, dev)
        d = shape[0]
        return Split.alloc("rows", (rows, rup8(d)), d, dev)

    def _alloc_activations(self, input_grad_buffer):
        b = self.batch
        dev = self.device
        n = len(self.ops)
        self.acts: list = [None] * n      # Split output of op i (aliases resolved in _act)
        self.args: list = [None] * n
        self.gin: list = [None] * n       # Split gradient wrt op i's input
        self.logits = None
        self.losses = None
        self.dlogits = None
        self.xin = None   # packed block input, allocated on first pack_input()
        self.xin32 = None  # its 32-channel-wide copy for a first conv with c8_in
        self._gout = None  # per-op output-gradient buffers of the last backward
        self.bnstats: dict = {}   # bn op -> float64 [groups][C8][2] (mean, rstd)
        for i, op in enumerate(self.ops):
            if op.kind == "relu" and i > 0 and self.ops[i - 1].fused_relu:
                continue
            if op.kind == "residual":             # the body's last BatchNorm writes it
                body, _ = self.children[i]
                self.acts[i] = body._act(len(body.ops) - 1)
                continue
            if op.kind == "bn":
                c = op.in_shape[0]
                self.bnstats[i] = torch.zeros((b // self.group, rup8(c), 2), dtype=torch.float64,
                                              device=dev)
            if op.kind == "flatten":
                src_flat = i > 0 and self.ops[i - 1].flat_out
                if not src_flat and len(op.in_shape) == 3:
                    self.acts[i] = self._split_for(op.out_shape, b)   # relayout target
                continue
            if op.kind == "softmax_ce":
                c = op.in_shape[0]
                self.losses = torch.zeros(b, dtype=torch.float32, device=dev)
                self.dlogits = Split.alloc("rows", (b, rup8(c)), c, dev)
                continue
            if op.kind == "fc" and i + 1 < n and self.ops[i + 1].kind == "softmax_ce":
                self.logits = torch.zeros((b, op.out_shape[0]), dtype=torch.float32, device=dev)
                continue
            shape = op.out_shape
            if op.kind in ("maxpool", "gap") and op.flat_out:
                shape = (int(np.prod(op.out_shape)),)
            self.acts[i] = self._split_for(shape, b)
            if op.kind == "maxpool":
                c, oh, ow = op.out_shape
                self.args[i] = torch.zeros((b, oh, ow, rup8(c)), dtype=torch.uint8, device=dev)
        for i, op in enumerate(self.ops):
            if op.kind in ("softmax_ce",):
                continue
            if op.kind == "relu" and op.relu_bwd_fused:
                continue
            if op.kind == "flatten":
                src_flat = i > 0 and self.ops[i - 1].flat_out
                if src_flat or len(op.in_shape) != 3:
                    continue
            if i == 0:
                if not self.need_input_grad:
                    continue
                if input_grad_buffer is not None:
                    self.gin[0] = input_grad_buffer
                    continue
            self.gin[i] = self._split_for(op.in_shape, b)
        self._concat_gy: dict = {}        # concat op -> per-branch output-gradient buffers
        for i, op in enumerate(self.ops):
            if op.kind == "concat":
                self._concat_gy[i] = [self._split_for(kid.out_shape, b)
                                      for kid in self.children[i]]
        self.loss_sum = torch.zeros(1, dtype=torch.float64, device=dev)

    # -- parameters ------------------------------------------------------------------

    def load(self, params, velocities=None):
        """Upload nested numpy (or tensor) params/velocities in reference layout."""
        for li, row in enumerate(self.slots):
            for ti, _ in enumerate(row):
                self.params[li][ti].copy_(torch.as_tensor(np.asarray(params[li][ti])))
                if velocities is not None:
                    self.velocity[li][ti].copy_(torch.as_tensor(np.asarray(velocities[li][ti])))
        self.pack_weights()

    def _conv_pack_jobs(self, skip=frozenset()) -> list:
        """(w, wf, wd, psf, psd, O, C, kh, kw, C8, O8) of every plain conv layer
        of this engine and its residual / concat children."""
        jobs = []
        for i, (a, b) in self.wplanes.items():
            op = self.ops[i]
            if i in skip or op.kind != "conv" or op.s2d is not None:
                continue
            l = op.layer
            jobs.append((self.params[i][0].data_ptr(), a.data_ptr(),
                         0 if b is None else b.data_ptr(), a[0].numel(),
                         0 if b is None else b[0].numel(), l.out_ch, l.in_ch, l.kh, l.kw,
                         op.c8_in or rup8(l.in_ch), rup8(l.out_ch)))
        for kids in self.children.values():
            for k in kids:
                if k is not None:
                    jobs += k._conv_pack_jobs()
        return jobs

    def pack_weights(self, skip=frozenset()):
        """Refresh the split-plane weight copies from the fp32 masters (except
        the layers in ``skip``, already repacked by the fused SGD): every conv
        layer of the block (children included) in one launch."""
        st = stream_of(self.device)
        key = tuple(sorted(skip))
        cache = getattr(self, "_pack_cache", None)
        if cache is None or cache[0] != key:
            jobs = self._conv_pack_jobs(skip)
            arr = (_lib.ConvPack * max(len(jobs), 1))(*[_lib.ConvPack(*j) for j in jobs])
            nbytes = sum(4.0 * j[5] * j[6] * j[7] * j[8]
                         + 6.0 * (j[3] + j[4]) for j in jobs)
            self._pack_cache = cache = (key, arr, len(jobs), nbytes)
        _, arr, njobs, nbytes = cache
        for lo in range(0, njobs, _lib.MAX_CONV_PACK):
            n = min(_lib.MAX_CONV_PACK, njobs - lo)
            sub = ctypes.cast(ctypes.byref(arr, lo * ctypes.sizeof(_lib.ConvPack)),
                              ctypes.POINTER(_lib.ConvPack))
            _lib.call("stzx_pack_conv_w_multi", sub, n, st, tag=f"{self.tag}pack_conv_w",
                      nbytes=nbytes)
        for i, (a, b) in self.wplanes.items():
            if i in skip:
                continue
            op = self.ops[i]
            l = op.layer
            w = self.params[i][0]
            if op.kind == "conv" and op.s2d is not None:
                _lib.call("stzx_pack_conv_w_s2d", ptr(w), ptr(a), a[0].numel(), l.out_ch,
                          l.in_ch, l.kernel, l.stride, op.s2d[1], st)
            elif op.kind == "fc":
                _lib.call("stzx_pack_rows", ptr(w), ptr(a), a[0].numel(), l.in_dim, l.out_dim,
                          rup8(l.out_dim), st)

    def state_numpy(self):
        """(params, velocities) as nested fp32 numpy arrays, reference layout."""
        p = [[t.detach().cpu().numpy().copy() for t in row] for row in self.params]
        v = [[t.detach().cpu().numpy().copy() for t in row] for row in self.velocity]
        return p, v

    # -- execution -------------------------------------------------------------------

    def op_flops(self, i: int, rows: int | None = None) -> float:
        """Algorithmic FLOPs of op i's forward contraction (2*M*N*K with the
        logical channel counts) over `rows` samples (default: the batch); its
        dgrad and wgrad have the same count."""
        op = self.ops[i]
        l = op.layer
        b = self.batch if rows is None else rows
        if op.kind == "conv":
            _, oh, ow = op.out_shape
            return 2.0 * b * oh * ow * l.out_ch * l.in_ch * l.kh * l.kw
        if op.kind == "fc":
            return 2.0 * b * l.in_dim * l.out_dim
        return 0.0

    def _rows(self, rows):
        """(r0, r1, view) for a pass over samples [r0, r1) of the batch (a
        micro-batch): view(split) restricts a full-batch Split to those rows."""
        r0, r1 = (0, self.batch) if rows is None else (int(rows[0]), int(rows[1]))
        if not 0 <= r0 < r1 <= self.batch:
            raise ShapeMismatch(f"rows {rows} outside the batch of {self.batch}")
        if (r0, r1) == (0, self.batch):
            return r0, r1, (lambda sp: sp)
        return r0, r1, (lambda sp: None if sp is None else sp.rows_view(r0, r1))

    def _act(self, i):
        """Output Split of op i, resolving ReLU / Flatten aliases."""
        if i < 0:
            return self._x
        op = self.ops[i]
        if self.acts[i] is not None:
            return self.acts[i]
        if op.kind in ("relu", "flatten"):
            return self._act(i - 1)
        return None

    def _check_groups(self, r0, r1):
        if r0 % self.group or (r1 - r0) % self.group:
            raise ShapeMismatch(f"BatchNorm needs whole sample groups of {self.group}; "
                                f"got rows [{r0}, {r1})")

    def _input(self, i):
        return self._x if i == 0 else self._act(i - 1)

    def pack_input(self, x: torch.Tensor, rows=None) -> Split:
        """fp32 batch in the reference layout -> the packed block input (only
        samples [r0, r1) when `rows` is given).  Returns the full-batch Split."""
        if tuple(x.shape) != (self.batch, *self.in_shape):
            raise ShapeMismatch(f"block expects {(self.batch, *self.in_shape)}, "
                                f"got {tuple(x.shape)}")
        r0, r1, view = self._rows(rows)
        b = r1 - r0
        st = stream_of(self.device)
        op0 = self.ops[0]
        if self.xin is None:
            if op0.s2d is not None:
                ks, cs8, hs, ws_ = op0.s2d
                l0 = op0.layer
                self.xin = Split.alloc("nhwc", (self.batch, hs, ws_, cs8),
                                       l0.in_ch * l0.stride ** 2, self.device)
            else:
                self.xin = self._split_for(self.in_shape, self.batch)
            if op0.c8_in:   # the forward's copy, 32 channels wide (the wgrad reads xin)
                c, h, w = self.in_shape
                self.xin32 = Split.alloc("nhwc", (self.batch, h, w, op0.c8_in), c, self.device)
        s = view(self.xin)
        xs = x[r0:r1]
        if op0.s2d is not None:
            ks, cs8, hs, ws_ = op0.s2d
            c, h, w = self.in_shape
            _lib.call("stzx_pack_s2d", ptr(xs), s.ptr(), s.ps, b, c, h, w,
                      op0.layer.stride, op0.layer.padding, hs, ws_, cs8, st,
                      tag=f"{self.tag}pack_s2d", nbytes=4.0 * b * c * h * w + 6.0 * b * s.row_elems)
        elif s.layout == "nhwc":
            c, h, w = self.in_shape
            _lib.call("stzx_pack_nchw", ptr(xs), s.ptr(), s.ps, b, c, h, w, s.width, st,
                      tag=f"{self.tag}pack_nchw", nbytes=4.0 * b * c * h * w + 6.0 * b * s.row_elems)
            if op0.c8_in:
                s32 = view(self.xin32)
                _lib.call("stzx_pack_nchw", ptr(xs), s32.ptr(), s32.ps, b, c, h, w, s32.width,
                          st, tag=f"{self.tag}pack_nchw32",
                          nbytes=4.0 * b * c * h * w + 6.0 * b * s32.row_elems)
        else:
            _lib.call("stzx_pack_rows", ptr(xs), s.ptr(), s.ps, b, self.in_shape[0],
                      s.width, st)
        return self.xin

    def forward(self, x, labels: torch.Tensor | None = None,
                loss_out: torch.Tensor | None = None, rows=None, sum_loss: bool = True,
                residual: "Split | None" = None):
        """Run the block.  ``x`` is a fp32 batch in the reference layout or an
        already-packed Split (e.g. the CONV block's output rows), always
        full-batch shaped; ``rows = (r0, r1)`` runs only samples [r0, r1) (a
        micro-batch; ``labels`` is full-batch too).  Returns the output Split
        of those rows (per-sample fp32 losses for a loss block).  The float64
        loss sum goes to ``loss_sum`` or is ADDED into ``loss_out``.
        ``residual`` (a residual block's body): full-batch Split added to the
        last op's (a BatchNorm's) output before a ReLU."""
        r0, r1, V = self._rows(rows)
        if isinstance(x, torch.Tensor):
            x = self.pack_input(x, rows)
        self._x = x
        st = stream_of(self.device)
        ws = workspace(self.device, self.ws_key)
        b = r1 - r0
        for i, op in enumerate(self.ops):
            xin = V(self._input(i))
            if i == 0 and op.c8_in:
                if self._x is not self.xin:
                    raise ShapeMismatch("a block whose first conv reads a 32-wide input copy "
                                        "takes fp32 batches (pack_input)")
                xin = V(self.xin32)
            l = op.layer
            if op.kind == "conv":
                c, h, w = op.in_shape
                y = V(self.acts[i])
                wf, _ = self.wplanes[i]
                if op.s2d is not None:             # stride-1 conv over s2d blocks
                    ks, cs8, hs, ws_ = op.s2d
                    _lib.call("stzx_conv_fwd_s2d", xin.ptr(), xin.ps, ptr(wf), wf[0].numel(),
                              ptr(self.params[i][1]), y.ptr(), y.ps, b,
                              l.in_ch * l.stride * l.stride, cs8, hs, ws_, l.out_ch, y.width, ks,
                              int(op.fused_relu), ptr(ws), ws.numel(), st,
                              flops=self.op_flops(i, b), tag=f"{self.tag}conv{i}_fwd")
                else:
                    _lib.call("stzx_conv2_fwd", xin.ptr(), xin.ps, ptr(wf), wf[0].numel(),
                              ptr(self.params[i][1]), y.ptr(), y.ps, b, xin.width, h, w,
                              l.out_ch, y.width, l.kh, l.kw, l.stride, l.ph, l.pw,
                              int(op.fused_relu), ptr(ws), ws.numel(), st,
                              flops=self.op_flops(i, b), tag=f"{self.tag}conv{i}_fwd")
            elif op.kind == "fc":
                wp, _ = self.wplanes[i]
                if self.acts[i] is not None:
                    y = V(self.acts[i])
                    _lib.call("stzx_fc_fwd", xin.ptr(), xin.ps, ptr(wp), wp[0].numel(),
                              ptr(self.params[i][1]), y.ptr(), y.ps, None, b, l.in_dim,
                              xin.width, l.out_dim, y.width, int(op.fused_relu), ptr(ws),
                              ws.numel(), st, flops=self.op_flops(i, b), tag=f"{self.tag}fc{i}_fwd")
                else:
                    _lib.call("stzx_fc_fwd", xin.ptr(), xin.ps, ptr(wp), wp[0].numel(),
                              ptr(self.params[i][1]), None, 0, ptr(self.logits[r0:r1]), b,
                              l.in_dim, xin.width, l.out_dim, rup8(l.out_dim), int(op.fused_relu),
                              ptr(ws), ws.numel(), st, flops=self.op_flops(i, b),
                              tag=f"{self.tag}fc{i}_fwd")
            elif op.kind == "maxpool":
                c, h, w = op.in_shape
                y = V(self.acts[i])
                _lib.call("stzx_maxpool_fwd", xin.ptr(), xin.ps, y.ptr(), y.ps,
                          ptr(self.args[i][r0:r1]), b, c, xin.width, h, w, l.kernel, l.stride,
                          y.width if op.flat_out else 0, st, tag=f"{self.tag}pool{i}_fwd",
                          nbytes=6.0 * b * xin.row_elems + 7.0 * b * self.args[i][0].numel())
            elif op.kind == "relu":
                if self.acts[i] is not None:
                    y = V(self.acts[i])
                    _lib.call("stzx_relu_fwd", xin.ptr(), xin.ps, y.ptr(), y.ps,
                              b * xin.row_elems, st)
            elif op.kind == "flatten":
                if self.acts[i] is not None:               # NHWC -> CHW-flat relayout
                    c, h, w = op.in_shape
                    y = V(self.acts[i])
                    _lib.call("stzx_nhwc_to_flat", xin.ptr(), xin.ps, y.ptr(), y.ps, b, c, h, w,
                              xin.width, y.width, st)
            elif op.kind == "bn":
                self._check_groups(r0, r1)
                c, h, w = op.in_shape
                y = V(self.acts[i])
                last = i == len(self.ops) - 1 and residual is not None
                res = V(residual) if last else None
                _lib.call("stzx_bn_fwd", xin.ptr(), xin.ps, ptr(self.params[i][0]),
                          ptr(self.params[i][1]), None if res is None else res.ptr(),
                          0 if res is None else res.ps, y.ptr(), y.ps,
                          ptr(self.bnstats[i][r0 // self.group:]), b, h * w, c, y.width,
                          self.group, float(l.eps), int(op.fused_relu or last), ptr(ws),
                          ws.numel(), st, tag=f"{self.tag}bn{i}_fwd",
                          nbytes=6.0 * (3 + (res is not None)) * b * xin.row_elems)
            elif op.kind == "gap":
                c, h, w = op.in_shape
                y = V(self.acts[i])
                _lib.call("stzx_gap_fwd", xin.ptr(), xin.ps, y.ptr(), y.ps, b, h * w, xin.width, st,
                          tag=f"{self.tag}gap{i}_fwd", nbytes=6.0 * b * (xin.row_elems + y.width))
            elif op.kind == "avgpool":
                c, h, w = op.in_shape
                y = V(self.acts[i])
                _lib.call("stzx_avgpool_fwd", xin.ptr(), xin.ps, y.ptr(), y.ps, b, xin.width, h, w,
                          l.kernel, l.stride, l.padding, st, tag=f"{self.tag}avgpool{i}_fwd",
                          nbytes=6.0 * b * (xin.row_elems + y.row_elems))
            elif op.kind == "concat":
                # every branch on the same input; each branch's output is copied
                # into its channel slice of the concatenated tensor
                x_full = self._input(i)
                y = V(self.acts[i])
                _, oh, ow = op.out_shape
                c0 = 0
                for kid in self.children[i]:
                    kid.forward(x_full, rows=rows)
                    out = V(kid._act(len(kid.ops) - 1))
                    cb = kid.out_shape[0]
                    _lib.call("stzx_copy_channels", out.ptr(), out.ps, out.width, 0, y.ptr(), y.ps,
                              y.width, c0, b * oh * ow, cb, None, 0, 0, st,
                              tag=f"{self.tag}concat{i}_fwd", nbytes=12.0 * b * oh * ow * cb)
                    c0 += cb
            elif op.kind == "residual":
                body, short = self.children[i]
                x_full = self._input(i)
                s_full = x_full
                if short is not None:
                    short.forward(x_full, rows=rows)
                    s_full = short._act(len(short.ops) - 1)
                body.forward(x_full, rows=rows, residual=s_full)
            elif op.kind == "softmax_ce":
                if labels is None:
                    raise ValueError("SoftmaxCrossEntropy needs labels")
                c = op.in_shape[0]
                dl = V(self.dlogits)
                _lib.call("stzx_softmax_ce", ptr(self.logits[r0:r1]), ptr(labels[r0:r1]),
                          ptr(self.losses[r0:r1]), dl.ptr(), dl.ps, b, c, dl.width, st)
                if sum_loss:
                    self.sum_loss(loss_out, rows)
        if self.losses is not None:
            return self.losses[r0:r1]
        return V(self._act(len(self.ops) - 1))

    def backward(self, gy: Split | None = None, rows=None, accumulate: bool = False,
                 phase: str = "all", gy_mask: Split | None = None):
        """Backward through the block; parameter-gradient sums land in
        ``grad_flat`` (ADDED to it with ``accumulate``: micro-batches of one
        iteration).  ``gy`` is full-batch shaped; ``rows = (r0, r1)`` runs
        samples [r0, r1) of the last forward over them.  ``phase``:

        * "all"   -- weight and input gradients, layer by layer;
        * "dgrad" -- only the input-gradient chain (pool / ReLU / conv and FC
          dgrad): what a peer waits for.  Each layer's output gradient stays
          in its own full-batch buffer;
        * "wgrad" -- only the weight / bias gradients, from the buffers a
          "dgrad" pass left (over ``rows``; the FC worker runs it over the
          whole batch after the boundary gradients have left).

        ``gy_mask`` (a residual block's body / shortcut): ``gy`` is the
        gradient of relu(last output + other branch); the last op (a
        BatchNorm) applies that ReLU's mask (plane 0 of ``gy_mask`` > 0).

        Returns the input-gradient Split of ``rows`` (None when the block has
        no input gradient, or for phase "wgrad")."""
        if phase not in ("all", "dgrad", "wgrad"):
            raise ValueError(f"unknown backward phase {phase!r}")
        r0, r1, V = self._rows(rows)
        st = stream_of(self.device)
        ws = workspace(self.device, self.ws_key)
        b = r1 - r0
        acc = int(bool(accumulate))
        do_w, do_d = phase in ("all", "wgrad"), phase in ("all", "dgrad")
        if phase == "wgrad":
            if self._gout is None:
                raise RuntimeError("backward(phase='wgrad') needs a preceding 'dgrad' pass")
            for i, op in enumerate(self.ops):
                if op.kind in ("conv", "fc"):
                    self._wgrad(i, V(self._input(i)), V(self._gout[i]), b, acc, ws, st)
                elif op.kind in ("residual", "concat"):
                    for k in self.children[i]:
                        if k is not None:
                            k.backward(rows=rows, accumulate=accumulate, phase="wgrad")
            return None
        gout = [None] * len(self.ops)   # full-batch output-gradient buffer per op
        g_full = gy
        for i in range(len(self.ops) - 1, -1, -1):
            op = self.ops[i]
            l = op.layer
            xin = V(self._input(i))
            g = V(g_full)
            gout[i] = g_full
            # the ReLU output feeding this op IS its input (possibly flattened):
            # > 0 exactly where the ReLU passed its gradient
            mptr = xin.ptr() if op.mask_from >= 0 else None
            if op.kind == "softmax_ce":
                g_full = self.dlogits
            elif op.kind == "flatten":
                if self.acts[i] is not None:              # CHW-flat -> NHWC relayout back
                    c, h, w = op.in_shape
                    out = V(self.gin[i])
                    _lib.call("stzx_flat_to_nhwc", g.ptr(), g.ps, out.ptr(), out.ps, b, c, h, w,
                              out.width, g.width, st)
                    g_full = self.gin[i]
            elif op.kind == "relu":
                if not op.relu_bwd_fused:
                    out = V(self.gin[i])
                    src = V(self._act(i))
                    _lib.call("stzx_relu_bwd", g.ptr(), g.ps, src.ptr(), out.ptr(), out.ps,
                              b * g.row_elems, st)
                    g_full = self.gin[i]
            elif op.kind == "bn":
                # dgamma / dbeta come out of the same reduction as the input
                # gradient, so they are produced in the "dgrad" pass
                self._check_groups(r0, r1)
                c, h, w = op.in_shape
                out = None if op.skip_dgrad else V(self.gin[i])
                m = V(gy_mask) if (gy_mask is not None and i == len(self.ops) - 1) else None
                gbias = ptr(self.grads[i - 1][1]) if (
                    out is not None and i > 0 and self.ops[i - 1].bias_by_bn) else None
                _lib.call("stzx_bn_bwd", g.ptr(), g.ps, None if m is None else m.ptr(),
                          xin.ptr(), xin.ps,
                          ptr(self.bnstats[i][r0 // self.group:]), ptr(self.params[i][0]),
                          ptr(self.grads[i][0]), ptr(self.grads[i][1]), gbias, acc,
                          None if out is None else out.ptr(), 0 if out is None else out.ps,
                          b, h * w, c, xin.width, self.group, ptr(ws), ws.numel(), st,
                          tag=f"{self.tag}bn{i}_bwd",
                          nbytes=(12.0 + 18.0 * (out is not None) + 4.0 * (m is not None))
                          * b * xin.row_elems)
                g_full = None if out is None else self.gin[i]
            elif op.kind == "gap":
                c, h, w = op.in_shape
                out = V(self.gin[i])
                _lib.call("stzx_gap_bwd", g.ptr(), g.ps, out.ptr(), out.ps, b, h * w, out.width,
                          st, tag=f"{self.tag}gap{i}_bwd", nbytes=6.0 * b * (out.row_elems + g.width))
                g_full = self.gin[i]
            elif op.kind == "avgpool":
                c, h, w = op.in_shape
                out = V(self.gin[i])
                _lib.call("stzx_avgpool_bwd", g.ptr(), g.ps, out.ptr(), out.ps, b, out.width, h, w,
                          l.kernel, l.stride, l.padding, st, tag=f"{self.tag}avgpool{i}_bwd",
                          nbytes=6.0 * b * (out.row_elems + g.row_elems))
                g_full = self.gin[i]
            elif op.kind == "concat":
                # each branch's channel slice of the gradient into its own
                # buffer, the branch backward, then the fp32 left fold of the
                # branches' input gradients in branch order
                _, oh, ow = op.out_shape
                c0, gxs = 0, []
                y_full = V(self.acts[i])
                for kid, gyb in zip(self.children[i], self._concat_gy[i]):
                    cb = kid.out_shape[0]
                    gv = V(gyb)
                    # a branch closing with a ReLU gets its mask applied here
                    # (the concat output slice is that ReLU's output)
                    masked = kid.ops[-1].kind == "relu" and kid.ops[-1].relu_bwd_fused
                    _lib.call("stzx_copy_channels", g.ptr(), g.ps, g.width, c0, gv.ptr(), gv.ps,
                              gv.width, 0, b * oh * ow, cb, y_full.ptr() if masked else None,
                              y_full.width if masked else 0, c0 if masked else 0, st,
                              tag=f"{self.tag}concat{i}_bwd",
                              nbytes=(12.0 + 2.0 * masked) * b * oh * ow * cb)
                    gxs.append(kid.backward(gyb, rows=rows, accumulate=accumulate, phase=phase))
                    c0 += cb
                out = V(self.gin[i])
                pos = 0
                while pos < len(gxs):        # fp32 left fold in branch order, <= 4 per pass
                    take = min(4 if pos == 0 else 3, len(gxs) - pos)
                    srcs = ([] if pos == 0 else [out]) + gxs[pos:pos + take]
                    pos += take
                    if len(srcs) == 1:       # a single branch: its input gradient as is
                        _lib.call("stzx_copy_channels", srcs[0].ptr(), srcs[0].ps,
                                  srcs[0].width, 0, out.ptr(), out.ps, out.width, 0,
                                  b * out.row_elems // out.width, out.width, None, 0, 0, st)
                        break
                    xs = _lib.ptr_array([sp.ptr() for sp in srcs])
                    pss = (ctypes.c_size_t * len(srcs))(*[sp.ps for sp in srcs])
                    _lib.call("stzx_add_n", xs, pss, len(srcs), out.ptr(), out.ps,
                              b * out.row_elems, st, tag=f"{self.tag}concat{i}_add",
                              nbytes=6.0 * (len(srcs) + 1) * b * out.row_elems)
                g_full = self.gin[i]
            elif op.kind == "residual":
                # the block's final ReLU mask (its output z > 0) is applied by
                # the consumers of the incoming gradient: the body's and the
                # projection shortcut's last BatchNorm, or the add itself for
                # an identity shortcut
                body, short = self.children[i]
                z_full = self.acts[i]
                gb = body.backward(g_full, rows=rows, accumulate=accumulate, phase=phase,
                                   gy_mask=z_full)
                mask_b = None
                if short is not None:
                    gs = short.backward(g_full, rows=rows, accumulate=accumulate, phase=phase,
                                        gy_mask=z_full)
                else:
                    gs, mask_b = g, V(z_full)
                out = V(self.gin[i])
                _lib.call("stzx_add", gb.ptr(), gb.ps, gs.ptr(), gs.ps,
                          None if mask_b is None else mask_b.ptr(), out.ptr(), out.ps,
                          b * out.row_elems, st, tag=f"{self.tag}res{i}_add",
                          nbytes=(18.0 + 2.0 * (mask_b is not None)) * b * out.row_elems)
                g_full = self.gin[i]
            elif op.kind == "maxpool":
                if op.skip_dgrad:
                    g_full = None
                    continue
                c, h, w = op.in_shape
                out = V(self.gin[i])
                _lib.call("stzx_maxpool_bwd", g.ptr(), g.ps, ptr(self.args[i][r0:r1]), out.ptr(),
                          out.ps, mptr, b, c, out.width, h, w, l.kernel, l.stride,
                          g.width if op.flat_out else 0, st, tag=f"{self.tag}pool{i}_bwd",
                          nbytes=7.0 * b * self.args[i][0].numel()
                          + (6.0 + 2.0 * (mptr is not None)) * b * out.row_elems)
                g_full = self.gin[i]
            elif op.kind in ("conv", "fc"):
                if do_w and self.wgrad_stream is not None and op.kind == "conv" \
                        and not self.children:
                    self._wgrad_side(i, xin, g, b, acc)
                elif do_w:
                    self._wgrad(i, xin, g, b, acc, ws, st)
                if op.skip_dgrad or (op.kind == "conv" and op.s2d is not None):
                    g_full = None
                    continue
                out = V(self.gin[i])
                if op.kind == "conv":
                    c, h, w = op.in_shape
                    _, wd = self.wplanes[i]
                    _lib.call("stzx_conv2_dgrad", g.ptr(), g.ps, ptr(wd), wd[0].numel(),
                              out.ptr(), out.ps, mptr, b, c, out.width, h, w, g.width, l.kh, l.kw,
                              l.stride, l.ph, l.pw, ptr(ws), ws.numel(), st,
                              flops=self.op_flops(i, b), tag=f"{self.tag}conv{i}_dgrad")
                else:
                    wp, _ = self.wplanes[i]
                    _lib.call("stzx_fc_dgrad", g.ptr(), g.ps, ptr(wp), wp[0].numel(), out.ptr(),
                              out.ps, mptr, b, l.in_dim, out.width, g.width, ptr(ws),
                              ws.numel(), st, flops=self.op_flops(i, b), tag=f"{self.tag}fc{i}_dgrad")
                if (self.update_side is not None and do_w and op.kind == "conv"
                        and not self.children and not accumulate):
                    self._update_layer_side(i)
                g_full = self.gin[i]
        self._gout = gout
        return V(g_full)

    def sum_loss(self, loss_out: torch.Tensor | None = None, rows=None):
        """Float64 sum of the per-sample losses of ``rows`` (last forward) into
        ``loss_sum``, or ADDED into ``loss_out``."""
        r0, r1, _ = self._rows(rows)
        tgt, acc = (self.loss_sum, 0) if loss_out is None else (loss_out, 1)
        _lib.call("stz_sum_f32", ptr(self.losses[r0:r1]), r1 - r0, ptr(tgt), acc,
                  stream_of(self.device))

    def _wgrad(self, i, xin, g, b, acc, ws, st):
        """Weight and bias gradient sums of conv / FC op i from its input rows
        ``xin`` and output-gradient rows ``g`` (``acc``: add into grad_flat)."""
        op = self.ops[i]
        l = op.layer
        side_bias = (op.kind == "conv" and not op.bias_by_bn and self.bias_stream is not None)
        if side_bias:
            self._colsum_side(i, g, b, acc)
        if op.kind == "conv" and op.s2d is not None:
            ks, cs8, hs, ws_ = op.s2d
            _lib.call("stzx_conv_wgrad_s2d", xin.ptr(), xin.ps, g.ptr(), g.ps,
                      ptr(self.grads[i][0]),
                      None if (op.bias_by_bn or side_bias) else ptr(self.grads[i][1]),
                      acc, b, l.in_ch, cs8,
                      hs, ws_, l.out_ch, g.width, l.kernel, l.stride, ptr(ws), ws.numel(), st,
                      flops=self.op_flops(i, b), tag=f"{self.tag}conv{i}_wgrad")
        elif op.kind == "conv":
            c, h, w = op.in_shape
            # summed by the BN backward, or on the bias stream
            gb = None if (op.bias_by_bn or side_bias) else ptr(self.grads[i][1])
            _lib.call("stzx_conv2_wgrad", xin.ptr(), xin.ps, g.ptr(), g.ps,
                      ptr(self.grads[i][0]), gb, acc, b, c, xin.width, h,
                      w, l.out_ch, g.width, l.kh, l.kw, l.stride, l.ph, l.pw, ptr(ws),
                      ws.numel(), st, flops=self.op_flops(i, b), tag=f"{self.tag}conv{i}_wgrad")
        elif self.sgd_in_wgrad is not None and i in self.fused_pack_ranges()[2]:
            # one FC worker owns this layer: the momentum step runs in the
            # weight-gradient epilogue (gW never stored)
            n, lr, mu = self.sgd_in_wgrad
            wf = self.wplanes[i][0]
            _lib.call("stzx_fc_wgrad_sgd", xin.ptr(), xin.ps, g.ptr(), g.ps,
                      ptr(self.params[i][0]), ptr(self.velocity[i][0]), wf.data_ptr(),
                      wf[0].numel(), ptr(self.params[i][1]), ptr(self.velocity[i][1]),
                      ptr(self.grads[i][0]), ptr(self.grads[i][1]), acc, b, l.in_dim,
                      xin.width, l.out_dim, g.width, float(lr), float(mu), inv_batch(n),
                      ptr(ws), ws.numel(), st, flops=self.op_flops(i, b),
                      tag=f"{self.tag}fc{i}_wgrad",
                      nbytes=22.0 * l.in_dim * l.out_dim)
            self._sgd_done.add(i)
        else:
            _lib.call("stzx_fc_wgrad", xin.ptr(), xin.ps, g.ptr(), g.ps,
                      ptr(self.grads[i][0]), ptr(self.grads[i][1]), acc, b, l.in_dim,
                      xin.width, l.out_dim, g.width, ptr(ws), ws.numel(), st,
                      flops=self.op_flops(i, b), tag=f"{self.tag}fc{i}_wgrad")

    def _colsum_side(self, i, g, b, acc):
        """Conv op i's bias gradient (column sums of its output gradient
        ``g``, b samples) on ``self.bias_stream``, ordered after the work
        that produced g; its own split-K scratch."""
        main = torch.cuda.current_stream(self.device)
        ev = torch.cuda.Event()
        ev.record(main)
        self.bias_stream.wait_event(ev)
        _, oh, ow = self.ops[i].out_shape
        with torch.cuda.stream(self.bias_stream):
            ws = workspace(self.device, "bias_side")
            _lib.call("stzx_colsum", g.ptr(), g.ps, b * oh * ow, self.ops[i].layer.out_ch,
                      g.width, ptr(self.grads[i][1]), acc, ptr(ws), ws.numel(),
                      stream_of(self.device), tag=f"{self.tag}conv{i}_bias",
                      nbytes=6.0 * b * oh * ow * g.width)
            done = torch.cuda.Event()
            done.record(self.bias_stream)
            self._bias_events[i] = done

    def _wgrad_side(self, i, xin, g, b, acc):
        """Conv op i's weight (and bias) gradient on ``self.wgrad_stream``,
        ordered after the work that produced its output gradient; its own
        split-K scratch."""
        main = torch.cuda.current_stream(self.device)
        ev = torch.cuda.Event()
        ev.record(main)
        self.wgrad_stream.wait_event(ev)
        with torch.cuda.stream(self.wgrad_stream):
            ws = workspace(self.device, "wgrad_side")
            self._wgrad(i, xin, g, b, acc, ws, stream_of(self.device))
            done = torch.cuda.Event()
            done.record(self.wgrad_stream)
            self._wgrad_events[i] = done

    def _update_layer_side(self, i):
        """Conv op i's momentum step (its W and b slice of the flat block) and
        split-plane repack on the update stream, after the input- and
        weight-gradient work issued so far (and its bias sums)."""
        stream, n, lr, mu = self.update_side
        main = torch.cuda.current_stream(self.device)
        ev = torch.cuda.Event()
        ev.record(main)
        stream.wait_event(ev)
        if i in self._bias_events:
            stream.wait_event(self._bias_events.pop(i))
        if i in self._wgrad_events:
            stream.wait_event(self._wgrad_events.pop(i))
        (off, _, _), (boff, _, bcnt) = self.slots[i]
        cnt = boff + bcnt - off
        l = self.ops[i].layer
        wf, wd = self.wplanes[i]
        with torch.cuda.stream(stream):
            st = stream_of(self.device)
            _lib.call("stz_sgd_momentum_pack", ptr(self.params_flat[off:]),
                      ptr(self.vel_flat[off:]), ptr(self.grad_flat[off:]), cnt, float(lr),
                      float(mu), inv_batch(n), _lib.range_array([]), 0, st,
                      tag=f"{self.tag}conv{i}_sgd", nbytes=20.0 * cnt)
            _lib.call("stzx_pack_conv2_w", ptr(self.params[i][0]), ptr(wf), wf[0].numel(),
                      ptr(wd), 0 if wd is None else wd[0].numel(), l.out_ch, l.in_ch, l.kh,
                      l.kw, self.ops[i].c8_in or rup8(l.in_ch), rup8(l.out_ch), st)
        self._sgd_done.add(i)

    def fused_pack_ranges(self):
        """(ctypes stz_plane_range array, count, layer indices): the FC weights,
        whose split-plane copy [in][out8] is row-major, are repacked inside
        the SGD kernel (stz_sgd_momentum_pack / stz_allreduce_sgd); the conv
        weight copies are permuted and keep their own pack kernels."""
        if getattr(self, "_pack_ranges", None) is None:
            rs, idx = [], []
            for i, (a, _) in sorted(self.wplanes.items()):
                op = self.ops[i]
                if op.kind != "fc" or 2 * len(rs) + 3 > 16:   # ranges + gaps <= 16
                    continue
                off, _, cnt = self.slots[i][0]
                l = op.layer
                rs.append((off, cnt, a.data_ptr(), a[0].numel(), l.out_dim, rup8(l.out_dim)))
                idx.append(i)
            self._pack_ranges = (_lib.range_array(rs), len(rs), frozenset(idx))
        return self._pack_ranges

    def _skip_ranges(self, done):
        """Pack ranges for an update after the layers in ``done`` were
        updated already (in their weight-gradient epilogue, or on the update
        stream): each such layer's parameter slice is skipped (planes NULL,
        D = 0; consecutive skipped layers merge, alignment gaps included); the
        other FC layers keep their fused repack."""
        fused = self.fused_pack_ranges()[2]
        rs, prev_done = [], False
        for i, row in enumerate(self.slots):
            if not row:
                continue
            if i in done:
                lo, hi = row[0][0], row[-1][0] + row[-1][2]
                if prev_done:
                    lo = rs.pop()[0]
                rs.append((lo, hi - lo, None, 0, 0, 0))
            elif i in fused:
                l = self.ops[i].layer
                a = self.wplanes[i][0]
                off, _, cnt = row[0]
                rs.append((off, cnt, a.data_ptr(), a[0].numel(), l.out_dim, rup8(l.out_dim)))
            prev_done = i in done
        return _lib.range_array(rs), len(rs)

    def fused_param_count(self) -> int:
        """Parameters whose split-plane copy the fused SGD rewrites (FC W)."""
        _, _, idx = self.fused_pack_ranges()
        return sum(self.slots[i][0][2] for i in idx)

    def sgd(self, n: int, lr: float, mu: float, grad: torch.Tensor | None = None):
        """Momentum step over the whole flat block (tensor_core.py:366-388)
        fused with the refresh of the FC split-plane weight copies; the conv
        copies are repacked after it."""
        g = self.grad_flat if grad is None else grad
        ranges, nr, fused = self.fused_pack_ranges()
        if self._sgd_done:
            done, self._sgd_done = self._sgd_done, set()
            if all(i in done for i, row in enumerate(self.slots) if row):
                return                      # every parameter was already updated
            ranges, nr = self._skip_ranges(done)
            fused = frozenset(fused | done)
        _lib.call("stz_sgd_momentum_pack", ptr(self.params_flat), ptr(self.vel_flat), ptr(g),
                  self.total, float(lr), float(mu), inv_batch(n), ranges, nr,
                  stream_of(self.device), tag=f"{self.tag}sgd_pack",
                  nbytes=20.0 * self.total + 6.0 * self.fused_param_count())
        self.pack_weights(skip=fused)

    def add_grads_from(self, other: "BlockEngine"):
        """grad_flat += other.grad_flat (replica gradient sum on one device)."""
        _lib.call("stz_vec_add", ptr(self.grad_flat), ptr(other.grad_flat), self.total,
                  stream_of(self.device))
