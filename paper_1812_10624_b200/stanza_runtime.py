"""Layer-separated training on B200s -- drop-in for the reference runtime.

``StanzaCluster(spec, *, n_conv, n_fc, batch_fn, lr, momentum=0.9, ...)``
and ``.train(iterations) -> StanzaResult(losses, state, transport)`` keep the
signature and semantics of /root/reference/pkg/src/stanza/stanza_runtime.py
:96-375.  One BSP iteration (:352-375):

  conv_compute  CONV trunk forward on each worker's batch (it, i)
  activations   many-to-one gather of [K, A] activations + labels into the
                FC worker's input rows, in ascending CONV index
  fc_compute    FC head forward + SoftmaxCE + backward on the gathered batch
  boundary      one-to-many scatter of each worker's [K, A] boundary grads
  (conv bwd)    CONV trunk backward from the boundary gradient
  exchange      allreduce(sum) of CONV grads over the CONV group and, iff
                n_fc > 1, of FC grads over the FC group
  update        momentum SGD with n = n_conv * K on every replica

Two deployments:

* single device (``comm=None``): every role on one GPU.  CONV replicas are
  bit-identical by construction (reference test_stanza_runtime.py:70-83), so
  the trunk runs once over the n_conv*K concatenated samples; each FC worker
  runs its own head pass over its contiguous row slice (zero-copy gather and
  scatter) and the FC replica gradients are summed on device.  With
  n_conv = n_fc = 1 this is the co-located 1-GPU configuration.
* one process per GPU (``comm=RoleComm``): rank i < n_conv is CONV worker
  i, rank n_conv + j is FC worker j; the exchanges are NCCL point-to-point
  ops and sub-group allreduces (comm.py).
"""

from __future__ import annotations

import random
from collections import Counter
from dataclasses import dataclass, field

import numpy as np
import torch

from .checkpointing import TrainState, state_to_bytes
from .engine import BlockEngine
from .model_partition import ConfigError, ModelSpec, Partition, mlp_split, split
from .roles import group_rows, plan_groups
from .tensor_core import ShapeMismatch, seeded_init


def dist_backend() -> str | None:
    import torch.distributed as dist
    return dist.get_backend() if dist.is_available() and dist.is_initialized() else None


class MissingSource(TimeoutError):
    """An expected upstream node never delivered its payload."""


class Tag:
    """Message classes of the per-iteration contract (reference transport.Tag)."""
    ACTIVATIONS = "activations"
    CONTROL = "control"
    BOUNDARY_GRADS = "boundary_grads"
    ALLREDUCE_CHUNK = "allreduce_chunk"
    CHECKPOINT = "checkpoint"


@dataclass
class PhaseRecord:
    label: str
    payload_bytes: int = 0
    elapsed_ms: float | None = None


@dataclass
class PhaseLedger:
    """Device-side stand-in for the reference's TrafficLedger: the phase
    sequence of every iteration, payload bytes per message class (what the
    reference's ledger tests pin, test_stanza_runtime.py:158-179) and, when
    phase timing is on, CUDA-event milliseconds per phase."""
    phases: list = field(default_factory=list)
    tag_payload_bytes: Counter = field(default_factory=Counter)
    tag_messages: Counter = field(default_factory=Counter)

    def record(self, label: str, nbytes: int = 0) -> PhaseRecord:
        rec = PhaseRecord(label, nbytes)
        self.phases.append(rec)
        return rec


@dataclass
class StanzaResult:
    losses: list
    state: TrainState | None
    transport: PhaseLedger


PHASES = ("conv_compute", "activations", "fc_compute", "boundary", "exchange", "update")


class StanzaCluster:
    """A layer-separated deployment on B200 GPUs.

    batch_fn(iteration, conv_index) -> (inputs [K, ...] float32, labels [K])
    exactly as in the reference; iteration indices are absolute so resumed
    runs replay the same data.  ``device`` selects the GPU (single-device
    mode); ``comm`` switches to one-process-per-GPU mode.
    """

    def __init__(self, spec: ModelSpec, *, n_conv: int, n_fc: int, batch_fn, lr: float,
                 momentum: float = 0.9, conv_time: float = 0.0, fc_unit_time: float = 0.0,
                 net=None, seed: int = 0, boundary: int | None = None,
                 state: TrainState | None = None, device=None, comm=None,
                 time_phases: bool = False, micro_batches: int | None = None,
                 segment_graphs: bool = True, exchange: str | None = None):
        if lr <= 0.0:
            raise ConfigError(f"learning rate must be positive, got {lr}")
        if not 0.0 <= momentum < 1.0:
            raise ValueError(f"momentum must be in [0, 1), got {momentum}")
        self.spec = spec
        self.layers = spec.require_layers()
        self.partition: Partition = (mlp_split(spec, boundary) if boundary is not None
                                     else split(spec))
        self.batch_fn = batch_fn
        self.lr, self.momentum = float(lr), float(momentum)
        self.conv_time, self.fc_unit_time = float(conv_time), float(fc_unit_time)
        self.seed = seed
        self.n_conv, self.n_fc = n_conv, n_fc
        self.conv_to_fc = plan_groups(n_conv, n_fc)
        self.max_group = max(self.conv_to_fc.count(j) for j in range(n_fc))
        self.comm = comm
        self.time_phases = time_phases
        self.k = spec.batch_k
        # micro-batch pipelining of CONV fwd -> gather -> FC -> scatter -> CONV bwd
        # (one process per GPU only).  Gradient sums are
        # unchanged up to fp32 summation order.
        from .engine import BlockEngine as _BE
        has_bn = (not spec.is_profile) and _BE(self.partition.conv_block, spec.input_shape, 1,
                                                "cpu", allocate=False).has_bn()
        if has_bn and micro_batches is not None and micro_batches > 1:
            raise ConfigError("BatchNorm normalises over each CONV worker's whole batch: "
                              "micro_batches must be 1")
        if micro_batches is None and has_bn:
            micro_batches = 1
        if micro_batches is None:
            # measured (AlexNet K=128, images/s): 1:1 29.3k / 30.1k / 26.6k and
            # 3:1 77.3k / 85.8k / 78.0k at 1 / 2 / 4 micro-batches
            micro_batches = 2 if (comm is not None and spec.batch_k % 2 == 0
                                  and spec.batch_k >= 32) else 1
        if micro_batches < 1 or spec.batch_k % micro_batches:
            raise ConfigError(f"micro_batches={micro_batches} must divide batch_k="
                              f"{spec.batch_k}")
        if comm is None:
            micro_batches = 1
        self.micro = int(micro_batches)
        # one process per GPU: each compute segment of the pipelined step is
        # captured as a CUDA graph the second time it runs (NCCL stays eager)
        self.segment_graphs = bool(segment_graphs) and comm is not None
        # gradient exchange + update of one process per GPU: "peer" = the fused
        # NVLink peer-memory kernels (stz_allreduce_sgd), "nccl" = NCCL
        # all_reduce followed by the SGD kernel (and the only choice on gloo)
        if exchange is None:
            exchange = "peer" if comm is not None and dist_backend() == "nccl" else "nccl"
        if exchange not in ("peer", "nccl"):
            raise ConfigError(f"exchange must be 'peer' or 'nccl', got {exchange!r}")
        self.exchange = exchange if comm is not None else "local"
        self._peer = None
        self._seg_graphs: dict = {}
        self._steps_done = 0
        cut = self.partition.split_index

        ref = seeded_init(self.layers, seed)
        if state is None:
            full0 = ref
            vel0 = [[np.zeros_like(t) for t in layer] for layer in ref]
            self.iteration = 0
        else:
            for what, nested in (("snapshot parameters", state.params),
                                 ("snapshot velocities", state.velocities)):
                flat_r = [t for layer in ref for t in layer]
                flat_c = [t for layer in nested for t in layer]
                if len(flat_r) != len(flat_c) or any(
                        tuple(a.shape) != tuple(np.shape(b)) for a, b in zip(flat_r, flat_c)):
                    raise ShapeMismatch(f"{what}: structure does not match the model")
            full0, vel0 = state.params, state.velocities
            self.iteration = state.iteration

        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(device)
        self.conv_ids = [("conv", i) for i in range(n_conv)]
        self.fc_ids = [("fc", j) for j in range(n_fc)]
        self.transport = PhaseLedger()
        self.replica_snapshots: dict = {}
        self._fc_replica = None          # (params_flat, vel_flat) on the holder's GPU
        self._replica_holder = None
        self._replica_iteration = None

        conv_block, fc_block = self.partition.conv_block, self.partition.fc_block
        in_shape = tuple(spec.input_shape)
        self.boundary_shape = tuple(self._shape_at(cut))
        a = int(np.prod(self.boundary_shape))
        self.boundary_activations = a
        dev = self.device
        k = self.k
        self.conv = None
        self.fcs: list[BlockEngine] = []

        from .engine import Split, rup8
        a8 = rup8(a)
        if comm is None:
            nk = n_conv * k
            self.x = torch.zeros((nk, *in_shape), dtype=torch.float32, device=dev)
            self.labels = torch.zeros(nk, dtype=torch.int32, device=dev)
            self.gboundary = Split.alloc("rows", (nk, a8), a, dev)
            self.conv = BlockEngine(conv_block, in_shape, nk, dev, full0[:cut], vel0[:cut],
                                    need_input_grad=False, group=k)
            for j in range(n_fc):
                lo, hi = group_rows(self.conv_to_fc, j)
                eng = BlockEngine(fc_block, (a,), (hi - lo) * k, dev,
                                  full0[cut:], vel0[cut:], need_input_grad=True,
                                  shared=self.fcs[0] if self.fcs else None,
                                  input_grad_buffer=self.gboundary.rows_view(lo * k, hi * k))
                eng.rows = (lo * k, hi * k)
                self.fcs.append(eng)
        else:
            if comm.n_conv != n_conv or comm.n_fc != n_fc:
                raise ConfigError("communicator roles do not match (n_conv, n_fc)")
            if comm.is_conv:
                self.x = torch.zeros((k, *in_shape), dtype=torch.float32, device=dev)
                self.labels = torch.zeros(k, dtype=torch.int32, device=dev)
                self.gboundary = Split.alloc("rows", (k, a8), a, dev)
                self.conv = BlockEngine(conv_block, in_shape, k, dev, full0[:cut], vel0[:cut],
                                        need_input_grad=False, group=k)
            else:
                self.x = None
                self.gboundary = None
                g = len(comm.members(comm.index))
                self.fc_in = Split.alloc("rows", (g * k, a8), a, dev)
                self.labels = torch.zeros(g * k, dtype=torch.int32, device=dev)
                eng = BlockEngine(fc_block, (a,), g * k, dev, full0[cut:], vel0[cut:],
                                  need_input_grad=True)
                eng.rows = (0, g * k)
                self.fcs.append(eng)
            if self.exchange == "peer":   # collective: every rank maps its role group
                self._peer = comm.peer_exchange(self.conv if comm.is_conv else self.fcs[0])
        self._loss_slots = None

    # -- helpers -------------------------------------------------------------------------

    def _shape_at(self, cut):
        from .tensor_core import out_shape
        shape = tuple(self.spec.input_shape)
        for layer in self.layers[:cut]:
            shape = out_shape(layer, shape)
        return shape

    def group_members(self, fc_index: int) -> list[int]:
        return [i for i, j in enumerate(self.conv_to_fc) if j == fc_index]

    @property
    def conv_params(self):
        """CONV replica parameters (device views, reference layout)."""
        return self.conv.params if self.conv is not None else None

    @property
    def fc_params(self):
        return self.fcs[0].params if self.fcs else None

    def local_conv_indices(self) -> list[int]:
        if self.comm is None:
            return list(range(self.n_conv))
        return [self.comm.index] if self.comm.is_conv else []

    # -- one iteration on device-resident inputs ------------------------------------

    def load_batch(self, it: int) -> None:
        """Fetch this process's CONV batches from batch_fn and upload them."""
        idx = self.local_conv_indices()
        if not idx:
            return
        xs, ys = [], []
        for i in idx:
            x, y = self.batch_fn(it, i)
            if x.shape[0] != self.k:
                raise ShapeMismatch(f"CONV batch has {x.shape[0]} samples, "
                                    f"expected batch_k={self.k}")
            xs.append(np.asarray(x, dtype=np.float32))
            ys.append(np.asarray(y))
        x = torch.from_numpy(np.ascontiguousarray(np.concatenate(xs)))
        y = torch.from_numpy(np.concatenate(ys).astype(np.int32))
        self.x.copy_(x.pin_memory(), non_blocking=True)
        self.labels.copy_(y.pin_memory(), non_blocking=True)

    def step(self, loss_slot: torch.Tensor | None = None, x: torch.Tensor | None = None,
             labels: torch.Tensor | None = None) -> None:
        """One layer-separated iteration on the batch in ``self.x`` /
        ``self.labels`` (or on device-resident ``x`` / ``labels`` of the same
        shapes, e.g. a pre-staged pool).  Adds the iteration's summed
        per-sample loss into loss_slot (float64, on this process's FC
        workers).  Single-device mode runs the reference's BSP phase order
        below; one process per GPU runs _step_pipelined."""
        x_in = self.x if x is None else x
        lab_all = self.labels if labels is None else labels
        if self.comm is not None:
            return self._step_pipelined(loss_slot, x_in, lab_all)
        k = self.k
        n = self.n_conv * k
        led = self.transport
        a_bytes = self.boundary_activations * k * 4
        ev = self._events() if self.time_phases else None
        mark = (lambda label: ev.append((label, self._event()))) if ev is not None else \
            (lambda label: None)
        mark("conv_compute")
        led.record("conv_compute")
        acts = self.conv.forward(x_in)

        mark("activations")
        led.record("activations", self.n_conv * (a_bytes + k * 4))
        led.tag_payload_bytes[Tag.ACTIVATIONS] += self.n_conv * a_bytes
        led.tag_payload_bytes[Tag.CONTROL] += self.n_conv * k * 4
        led.tag_messages[Tag.ACTIVATIONS] += self.n_conv
        led.tag_messages[Tag.CONTROL] += self.n_conv

        mark("fc_compute")
        led.record("fc_compute")
        for j, eng in enumerate(self.fcs):
            lo, hi = eng.rows
            eng.forward(acts.rows_view(lo, hi), lab_all[lo:hi], loss_out=loss_slot)
            eng.backward()

        # the FC block's exchange + update depend only on the FC gradients: they
        # run on a side stream, concurrently with the CONV backward (the
        # momentum kernel is HBM-bound and co-resides with the GEMMs, which
        # are bound by the L2 -> SM feed); joined before the step ends
        overlap = ev is None
        main = torch.cuda.current_stream(self.device)
        if overlap:
            side = self._side_stream()
            side.wait_stream(main)
            with torch.cuda.stream(side):
                for eng in self.fcs[1:]:
                    self.fcs[0].add_grads_from(eng)
                self.fcs[0].sgd(n, self.lr, self.momentum)

        mark("boundary")
        led.record("boundary", self.n_conv * a_bytes)
        led.tag_payload_bytes[Tag.BOUNDARY_GRADS] += self.n_conv * a_bytes
        led.tag_messages[Tag.BOUNDARY_GRADS] += self.n_conv
        self.conv.backward(self.gboundary)

        mark("exchange")
        ring = lambda p, m: 0 if m == 1 else int(2 * (m - 1) * p * 4)  # noqa: E731
        ar_bytes = ring(self.partition.conv_params, self.n_conv) + \
            (ring(self.partition.fc_params, self.n_fc) if self.n_fc > 1 else 0)
        led.record("exchange", ar_bytes)
        led.tag_payload_bytes[Tag.ALLREDUCE_CHUNK] += ar_bytes
        if not overlap:
            for eng in self.fcs[1:]:
                self.fcs[0].add_grads_from(eng)

        mark("update")
        led.record("update")
        self.conv.sgd(n, self.lr, self.momentum)
        if overlap:
            main.wait_stream(side)
        else:
            self.fcs[0].sgd(n, self.lr, self.momentum)
        mark("end")
        if ev is not None:
            self._pending_events.append(ev)

    def _side_stream(self) -> "torch.cuda.Stream":
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(self.device)
        return self._side

    def _segment(self, key, fn) -> None:
        """Run a compute segment of the pipelined step: eagerly during the
        first step (kernel attributes, workspaces), then captured into a CUDA
        graph the first time its ``key`` -- every pointer its kernels bake in
        -- is seen, and replayed from then on."""
        if not self.segment_graphs or self.time_phases or self._steps_done == 0:
            fn()
            return
        g = self._seg_graphs.get(key)
        if g is None:
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream(self.device)
            s.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.stream(s):
                with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
                    fn()
            torch.cuda.current_stream(self.device).wait_stream(s)
            self._seg_graphs[key] = g
        g.replay()

    def _step_pipelined(self, loss_slot, x_in, lab_all) -> None:
        """One iteration in the one-process-per-GPU deployment, pipelined over
        ``self.micro`` micro-batches of kb = K / micro samples per CONV worker.

        CONV worker: forward each micro-batch and post its activations at
        once (the FC worker starts while the next micro-batch is computed);
        as each micro-batch's boundary gradient arrives, its input-gradient
        chain (overlapping the FC worker's next micro-batch); then every
        weight gradient once over the whole batch.
        FC worker: per micro-batch, receive the group's rows (its input is
        laid out [micro-batch][member][kb], so each micro-batch is
        contiguous), run the FC forward and only the input-gradient chain,
        and post each member's boundary rows back; the FC weight gradients
        follow over the whole batch, overlapping the CONV backward.  With
        micro = 1 this is the BSP step with the FC weight gradients moved off
        the critical path.  Exchange and update are the BSP step's; the sums
        are unchanged up to fp32 summation order."""
        comm = self.comm
        comm.warm(self.device)
        m, k = self.micro, self.k
        kb = k // m
        n = self.n_conv * k
        led = self.transport
        a_bytes = self.boundary_activations * k * 4
        ev = self._events() if self.time_phases else None
        mark = (lambda label: ev.append((label, self._event()))) if ev is not None else \
            (lambda label: None)
        led.record("conv_compute")
        led.record("activations", self.n_conv * (a_bytes + k * 4))
        led.tag_payload_bytes[Tag.ACTIVATIONS] += self.n_conv * a_bytes
        led.tag_payload_bytes[Tag.CONTROL] += self.n_conv * k * 4
        led.tag_messages[Tag.ACTIVATIONS] += self.n_conv * m
        led.tag_messages[Tag.CONTROL] += self.n_conv * m
        led.record("fc_compute")
        led.record("boundary", self.n_conv * a_bytes)
        led.tag_payload_bytes[Tag.BOUNDARY_GRADS] += self.n_conv * a_bytes
        led.tag_messages[Tag.BOUNDARY_GRADS] += self.n_conv * m

        if comm.is_conv:
            mark("conv_compute")
            sends = []
            for j in range(m):
                rows = (j * kb, (j + 1) * kb)
                self._segment(("conv_fwd", j, x_in.data_ptr()),
                              lambda rows=rows: self.conv.forward(x_in, rows=rows))
                acts = self.conv._act(len(self.conv.ops) - 1).rows_view(*rows)
                sends += comm.post_activations(
                    [acts.plane_rows(p) for p in range(3)] + [lab_all[rows[0]:rows[1]]], None)
            mark("activations")
            recvs = []
            for j in range(m):
                gb = self.gboundary.rows_view(j * kb, (j + 1) * kb)
                recvs += comm.post_boundary(None, [gb.plane_rows(p) for p in range(3)])
            mark("fc_compute")
            per = len(recvs) // m
            for j in range(m):
                # the input-gradient chain of micro-batch j as soon as its
                # boundary rows land (overlaps the FC worker's next one) ...
                for w in recvs[j * per:(j + 1) * per]:
                    w.wait()
                if j == 0:
                    mark("boundary")
                self._segment(("conv_dgrad", j), lambda j=j: self.conv.backward(
                    self.gboundary, rows=(j * kb, (j + 1) * kb), phase="dgrad"))
            # ... then every weight / bias gradient once, over the whole batch
            self._segment(("conv_wgrad",), lambda: self.conv.backward(phase="wgrad"))
            for w in sends:
                w.wait()
        else:
            eng = self.fcs[0]
            g = len(comm.members(comm.index))
            loss_to = loss_slot
            if loss_to is None:           # micro-batch sums accumulate into loss_sum
                eng.loss_sum.zero_()
                loss_to = eng.loss_sum
            mark("conv_compute")
            mark("activations")
            sends = []
            for j in range(m):
                base = j * g * kb
                recv = []
                for pos in range(g):
                    rv = self.fc_in.rows_view(base + pos * kb, base + (pos + 1) * kb)
                    recv.append([rv.plane_rows(p) for p in range(3)] +
                                [self.labels[base + pos * kb:base + (pos + 1) * kb]])
                for w in comm.post_activations(None, recv):
                    w.wait()
                if j == 0:
                    mark("fc_compute")
                rows = (base, base + g * kb)

                def fc_mb(rows=rows):
                    eng.forward(self.fc_in, self.labels, rows=rows, sum_loss=False)
                    eng.backward(rows=rows, phase="dgrad")
                self._segment(("fc_mb", j), fc_mb)
                eng.sum_loss(loss_to, rows)
                gx = eng.gin[0].rows_view(*rows)
                sends += comm.post_boundary(
                    [[gx.rows_view(pos * kb, (pos + 1) * kb).plane_rows(p) for p in range(3)]
                     for pos in range(g)], None)
            mark("boundary")
            self._segment(("fc_wgrad",), lambda: eng.backward(phase="wgrad"))  # overlaps CONV bwd
            for w in sends:
                w.wait()

        mark("exchange")
        ring = lambda p, mm: 0 if mm == 1 else int(2 * (mm - 1) * p * 4)  # noqa: E731
        ar_bytes = ring(self.partition.conv_params, self.n_conv) + \
            (ring(self.partition.fc_params, self.n_fc) if self.n_fc > 1 else 0)
        led.record("exchange", ar_bytes)
        led.tag_payload_bytes[Tag.ALLREDUCE_CHUNK] += ar_bytes
        if self._peer is not None:
            # exchange + update fused over NVLink peer memory (one segment)
            self._segment(("peer_exchange_sgd",),
                          lambda: self._peer.run(n, self.lr, self.momentum))
            mark("update")
            led.record("update")
        else:
            comm.allreduce_grads(self.conv.grad_flat if comm.is_conv else self.fcs[0].grad_flat)
            mark("update")
            led.record("update")
            if self.conv is not None:
                self._segment(("conv_sgd",), lambda: self.conv.sgd(n, self.lr, self.momentum))
            if self.fcs:
                self._segment(("fc_sgd",), lambda: self.fcs[0].sgd(n, self.lr, self.momentum))
        mark("end")
        if ev is not None:
            self._pending_events.append(ev)
        self._steps_done += 1

    def capture(self, x: torch.Tensor | None = None, labels: torch.Tensor | None = None,
                loss_slot: torch.Tensor | None = None) -> "torch.cuda.CUDAGraph":
        """Capture one whole iteration (every kernel of conv fwd, FC step,
        conv bwd, update) as a CUDA graph on device-resident inputs; replay()
        runs it with no host launch overhead.  Single-device mode only (the
        NCCL exchanges of the one-process-per-GPU mode stay eager).  Call
        once eagerly first so every kernel attribute / tensor map is set."""
        if self.comm is not None:
            raise RuntimeError("graph capture covers the single-device deployment")
        slot = loss_slot
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                if slot is not None:
                    slot.zero_()
                self.step(slot, x=x, labels=labels)
        torch.cuda.current_stream(self.device).wait_stream(s)
        # the ledger recorded the captured step once; it describes a replay
        return g

    # -- public API ------------------------------------------------------------------

    def autotune_tiles(self, x: torch.Tensor | None = None,
                       labels: torch.Tensor | None = None) -> dict:
        """Measure the GEMM tile shapes of this cluster's step on this GPU
        (`_lib.autotune_tiles`) and install the winners for every later step
        and capture.  Runs one full iteration (like step(); its loss is not
        recorded), on every rank when the cluster spans processes.  The
        parameters and velocities this process holds are restored afterwards
        (and their split-plane weight copies repacked), so training continues
        from the same state as without it."""
        from . import _lib
        engines = [e for e in [self.conv, *self.fcs] if e is not None]
        saved = [(e.params_flat.clone(), e.vel_flat.clone()) for e in engines]
        table = _lib.autotune_tiles(lambda: self.step(None, x=x, labels=labels))
        for e, (pf, vf) in zip(engines, saved):
            e.params_flat.copy_(pf)
            e.vel_flat.copy_(vf)
            e.pack_weights()
        torch.cuda.synchronize(self.device)
        return table

    def train(self, iterations: int) -> StanzaResult:
        """Run `iterations` more iterations; may be called repeatedly."""
        slots = torch.zeros(max(iterations, 1), dtype=torch.float64, device=self.device)
        self._pending_events = []
        for s in range(iterations):
            self.load_batch(self.iteration)
            self.step(slots[s:s + 1] if self.fcs else None)
            self.iteration += 1
        if self.comm is not None:
            self.comm.sum_scalar(slots)     # FC ranks hold the loss sums
        n = self.n_conv * self.k
        losses = [float(v) / n for v in slots[:iterations].cpu().tolist()]
        self._resolve_phase_times()
        return StanzaResult(losses=losses, state=self.state(), transport=self.transport)

    def state(self) -> TrainState | None:
        """Full state stitched from the first CONV and the first FC replica.
        Collective in one-process-per-GPU mode: FC worker 0 ships its block to
        rank 0, which returns the TrainState (other ranks return None)."""
        if self.comm is None:
            cp, cv = self.conv.state_numpy()
            fp, fv = self.fcs[0].state_numpy()
            return TrainState(self.iteration, cp + fp, cv + fv)
        import torch.distributed as dist
        fc0 = self.comm.n_conv
        rank = self.comm.rank
        if rank == fc0:
            dist.send(self.fcs[0].params_flat, 0)
            dist.send(self.fcs[0].vel_flat, 0)
        if rank != 0:
            return None
        cut = self.partition.split_index
        proto = BlockEngine(self.partition.fc_block, (self.boundary_activations,), 1,
                            self.device, allocate=False)
        pf = torch.empty(proto.total, dtype=torch.float32, device=self.device)
        vf = torch.empty_like(pf)
        dist.recv(pf, fc0)
        dist.recv(vf, fc0)
        fp = [[t.cpu().numpy().copy() for t in row] for row in proto._views(pf)]
        fv = [[t.cpu().numpy().copy() for t in row] for row in proto._views(vf)]
        cp, cv = self.conv.state_numpy()
        assert len(cp) == cut
        return TrainState(self.iteration, cp + fp, cv + fv)

    def checkpoint(self) -> TrainState:
        """Snapshot the run (stanza_runtime.py:182-211).  FC worker 0's block
        state (w, v) is also replicated to a seeded-random CONV worker so the
        heavyweight FC parameters exist on two GPUs: a device-to-device copy
        over NVLink into a buffer on the holder's GPU (one process per GPU)
        or a device copy (single device).  The holder keeps the replica
        resident in HBM for restore_fc_replica() and its STZC blob in
        replica_snapshots, byte-identical to the reference's
        (checkpointing.py:44-50).  Collective in one-process-per-GPU mode;
        returns the TrainState on rank 0 (None elsewhere), like state()."""
        holder = random.Random((self.seed << 32) ^ self.iteration).randrange(self.n_conv)
        self._replicate_fc(holder)
        st = self.state()
        blob = self._replica_blob()
        if blob is not None:
            self.replica_snapshots[self.conv_ids[holder]] = blob
        nbytes = 2 * 4 * self.partition.fc_params + 16 * len(self.layers)
        self.transport.record("checkpoint", nbytes)
        self.transport.tag_payload_bytes[Tag.CHECKPOINT] += nbytes
        self.transport.tag_messages[Tag.CHECKPOINT] += 1
        return st

    def _fc_proto(self) -> BlockEngine:
        return BlockEngine(self.partition.fc_block, (self.boundary_activations,), 1,
                           self.device, allocate=False)

    def _replicate_fc(self, holder: int) -> None:
        self._replica_holder, self._replica_iteration = holder, self.iteration
        if self.comm is None:
            eng = self.fcs[0]
            self._fc_replica = (eng.params_flat.clone(), eng.vel_flat.clone())
            return
        import torch.distributed as dist
        comm = self.comm
        fc0 = comm.n_conv
        ops = []
        if comm.rank == fc0:
            ops = [dist.P2POp(dist.isend, t, holder, group=comm.act_group)
                   for t in (self.fcs[0].params_flat, self.fcs[0].vel_flat)]
        elif comm.rank == holder:
            total = self._fc_proto().total
            if self._fc_replica is None or self._fc_replica[0].numel() != total:
                self._fc_replica = (torch.empty(total, dtype=torch.float32, device=self.device),
                                    torch.empty(total, dtype=torch.float32, device=self.device))
            ops = [dist.P2POp(dist.irecv, t, fc0, group=comm.act_group)
                   for t in self._fc_replica]
        for w in (dist.batch_isend_irecv(ops) if ops else []):
            w.wait()

    def _holds_replica(self) -> bool:
        if self._fc_replica is None:
            return False
        return self.comm is None or self.comm.rank == self._replica_holder

    def _replica_blob(self) -> bytes | None:
        """STZC blob of the resident replica (on its holder), else None."""
        if not self._holds_replica():
            return None
        proto = self._fc_proto()
        pf, vf = self._fc_replica
        fp = [[t.cpu().numpy().copy() for t in row] for row in proto._views(pf)]
        fv = [[t.cpu().numpy().copy() for t in row] for row in proto._views(vf)]
        return state_to_bytes(TrainState(self._replica_iteration, fp, fv))

    def restore_fc_replica(self) -> int:
        """Reload every FC replica's (w, v) from the checkpoint replica held on
        the CONV worker's GPU (the paper's FC-worker recovery):
        the holder sends it over NVLink to each FC worker, which repacks its
        split-plane weight copies.  Collective in one-process-per-GPU mode.
        Returns the iteration the replica was taken at."""
        if self._replica_holder is None:
            raise RuntimeError("no FC replica: call checkpoint() first")
        if self.comm is None:
            pf, vf = self._fc_replica
            self.fcs[0].params_flat.copy_(pf)
            self.fcs[0].vel_flat.copy_(vf)
            self.fcs[0].pack_weights()
            return self._replica_iteration
        import torch.distributed as dist
        comm = self.comm
        ops = []
        if comm.rank == self._replica_holder:
            for r in comm.fc_ranks:
                ops += [dist.P2POp(dist.isend, t, r, group=comm.act_group)
                        for t in self._fc_replica]
        elif not comm.is_conv:
            eng = self.fcs[0]
            ops = [dist.P2POp(dist.irecv, t, self._replica_holder, group=comm.act_group)
                   for t in (eng.params_flat, eng.vel_flat)]
        for w in (dist.batch_isend_irecv(ops) if ops else []):
            w.wait()
        if not comm.is_conv:
            self.fcs[0].pack_weights()
        return self._replica_iteration

    # -- phase timing ----------------------------------------------------------------

    def _events(self):
        return []

    def _event(self):
        e = torch.cuda.Event(enable_timing=True)
        e.record(torch.cuda.current_stream(self.device))
        return e

    def _resolve_phase_times(self):
        if not self.time_phases or not getattr(self, "_pending_events", None):
            return
        torch.cuda.synchronize(self.device)
        recs = [p for p in self.transport.phases if p.label in PHASES]
        i = len(recs) - 6 * len(self._pending_events)
        for ev in self._pending_events:
            for (label, e0), (_, e1) in zip(ev[:-1], ev[1:]):
                recs[i].elapsed_ms = e0.elapsed_time(e1)
                i += 1
        self._pending_events = []
