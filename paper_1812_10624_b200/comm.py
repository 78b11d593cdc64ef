"""Role communicator: one process per GPU, CONV and FC groups over NCCL.

Replaces the reference's simulated network for the three per-iteration
exchanges of the layer-separated step (stanza_runtime.py:228-338):

* activations: many-to-one, CONV i -> FC conv_to_fc[i]; the FC worker
  receives each member's [K, A] block straight into rows [pos*K, (pos+1)*K)
  of its input buffer (zero-copy concat, :64-85, :266-267), labels likewise;
* boundary gradients: one-to-many, the mirror image (:278-307, :274-275);
* gradient exchange: allreduce(sum) of the flat block-gradient vector on the
  CONV sub-group and, iff n_fc > 1, on the FC sub-group (:309-338).  The two
  groups are disjoint process sets, so their allreduces overlap naturally.

All of it is expressed with torch.distributed point-to-point ops and
sub-group collectives, so the same code runs over NCCL on B200s and over
gloo on CPU tensors (the multi-process CPU tests).

Two data paths:

* ``PeerLink`` + ``PeerExchange`` (exchange="peer", the default between
  GPUs of one node): the gather / scatter and the gradient exchange are
  kernels that load and store peer memory mapped through CUDA IPC, ordered
  by device-side flags (csrc/stz_peer.cuh).  torch.distributed only carries
  the one-time handle exchange, so the process group can be NCCL or gloo --
  gloo lets several ranks share one GPU (the multi-process parity tests on
  a 1-GPU box).
* NCCL point-to-point ops and sub-group allreduces (exchange="nccl"), which
  also run over gloo on CPU tensors (the multi-process CPU tests).  Micro-
  batch pipelining posts the two P2P directions
  asynchronously: a CONV worker sends every micro-batch's activations before
  it receives any boundary gradient, while its FC worker alternates receive
  / compute / send.  Each direction therefore runs on its own communicator
  (own NCCL stream), so neither queue can block the other.
"""

from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist

from .roles import plan_groups


def _nccl() -> bool:
    """Whether the default process group moves CUDA tensors over NCCL (a
    "nccl" or mixed "cpu:gloo,cuda:nccl" backend)."""
    return "nccl" in str(dist.get_backend())


class RoleComm:
    """Rank r < n_conv is CONV worker r; rank n_conv + j is FC worker j."""

    def __init__(self, n_conv: int, n_fc: int, group=None):
        if not dist.is_initialized():
            raise RuntimeError("torch.distributed must be initialized (one process per GPU)")
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if self.world != n_conv + n_fc:
            raise ValueError(f"world size {self.world} != n_conv + n_fc = {n_conv + n_fc}")
        self.n_conv, self.n_fc = n_conv, n_fc
        self.conv_to_fc = plan_groups(n_conv, n_fc)
        self.conv_ranks = list(range(n_conv))
        self.fc_ranks = list(range(n_conv, n_conv + n_fc))
        # every rank must create every group, members or not
        self.conv_group = dist.new_group(self.conv_ranks) if n_conv > 1 else None
        self.fc_group = dist.new_group(self.fc_ranks) if n_fc > 1 else None
        self.is_conv = self.rank < n_conv
        self.index = self.rank if self.is_conv else self.rank - n_conv
        # one communicator per P2P direction for the pipelined step
        everyone = list(range(self.world))
        self.act_group = dist.new_group(everyone)
        self.grad_group = dist.new_group(everyone)
        self._warm = False

    def warm(self, device) -> None:
        """Create the NCCL communicators of the P2P groups eagerly (a P2P op
        must not be the first call on an NCCL group unless every rank joins)."""
        if self._warm:
            return
        dev = torch.device(device) if _nccl() else torch.device("cpu")
        t = torch.zeros(1, device=dev)
        for g in (self.act_group, self.grad_group):
            dist.all_reduce(t, group=g)
        self._warm = True

    # -- topology -------------------------------------------------------------------

    def members(self, fc_index: int) -> list[int]:
        """CONV indices served by FC worker fc_index, ascending (concat order)."""
        return [i for i, j in enumerate(self.conv_to_fc) if j == fc_index]

    def fc_rank_of(self, conv_index: int) -> int:
        return self.n_conv + self.conv_to_fc[conv_index]

    def fc_index_of(self, conv_index: int) -> int:
        return self.conv_to_fc[conv_index]

    # -- exchanges --------------------------------------------------------------------

    def gather_activations(self, send: list | None, recv: list | None, k: int = 0) -> None:
        """CONV side: ``send`` = tensors of its [K, ...] block (the three
        split planes and the labels).  FC side: ``recv[pos]`` = matching
        tensors (row slices of its input buffers) for member ``pos``, which
        are received in place -- ascending CONV order, zero-copy concat."""
        ops = []
        if self.is_conv:
            dst = self.fc_rank_of(self.index)
            ops += [dist.P2POp(dist.isend, t, dst) for t in send]
        else:
            for pos, i in enumerate(self.members(self.index)):
                ops += [dist.P2POp(dist.irecv, t, i) for t in recv[pos]]
        for req in dist.batch_isend_irecv(ops):
            req.wait()

    def scatter_boundary(self, send: list | None, recv: list | None, k: int = 0) -> None:
        """FC side: ``send[pos]`` = row slices of its boundary gradient for
        member ``pos``; CONV side: ``recv`` = its [K, ...] gradient tensors."""
        ops = []
        if self.is_conv:
            src = self.fc_rank_of(self.index)
            ops += [dist.P2POp(dist.irecv, t, src) for t in recv]
        else:
            for pos, i in enumerate(self.members(self.index)):
                ops += [dist.P2POp(dist.isend, t, i) for t in send[pos]]
        for req in dist.batch_isend_irecv(ops):
            req.wait()

    # -- asynchronous exchanges (micro-batch pipelining) ----------------------------

    def post_activations(self, send: list | None, recv: list | None) -> list:
        """Like gather_activations for ONE micro-batch, but posted on the
        activation communicator and returned un-waited (wait() on the FC side
        before the tensors are read; on the CONV side before the buffers are
        overwritten)."""
        ops = []
        if self.is_conv:
            dst = self.fc_rank_of(self.index)
            ops += [dist.P2POp(dist.isend, t, dst, group=self.act_group) for t in send]
        else:
            for pos, i in enumerate(self.members(self.index)):
                ops += [dist.P2POp(dist.irecv, t, i, group=self.act_group) for t in recv[pos]]
        return dist.batch_isend_irecv(ops)

    def post_boundary(self, send: list | None, recv: list | None) -> list:
        """scatter_boundary for ONE micro-batch on the gradient communicator,
        returned un-waited."""
        ops = []
        if self.is_conv:
            src = self.fc_rank_of(self.index)
            ops += [dist.P2POp(dist.irecv, t, src, group=self.grad_group) for t in recv]
        else:
            for pos, i in enumerate(self.members(self.index)):
                ops += [dist.P2POp(dist.isend, t, i, group=self.grad_group) for t in send[pos]]
        return dist.batch_isend_irecv(ops)

    def allreduce_grads(self, flat: torch.Tensor) -> None:
        """Sum the flat gradient vector over this rank's role group."""
        group = self.conv_group if self.is_conv else self.fc_group
        if group is not None:
            dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)

    def sum_scalar(self, t: torch.Tensor) -> None:
        if t.is_cuda and not _nccl():
            c = t.cpu()
            dist.all_reduce(c, op=dist.ReduceOp.SUM)
            t.copy_(c)
            return
        dist.all_reduce(t, op=dist.ReduceOp.SUM)

    def p2p(self, sends=(), recvs=()) -> None:
        """Blocking point-to-point transfers of whole tensors on the
        activation communicator: ``sends`` = [(tensor, dst_rank)], ``recvs``
        = [(tensor, src_rank)].  Device tensors are staged through host
        memory when the process group is not NCCL (gloo)."""
        staged = not _nccl()
        ops, back = [], []
        for t, r in sends:
            ops.append(dist.P2POp(dist.isend, t.cpu() if staged and t.is_cuda else t, r,
                                  group=self.act_group))
        for t, r in recvs:
            buf = torch.empty(t.shape, dtype=t.dtype) if staged and t.is_cuda else t
            if buf is not t:
                back.append((t, buf))
            ops.append(dist.P2POp(dist.irecv, buf, r, group=self.act_group))
        for w in (dist.batch_isend_irecv(ops) if ops else []):
            w.wait()
        for t, buf in back:
            t.copy_(buf)

    def barrier(self) -> None:
        dist.barrier()

    def group_of_role(self):
        """(process group, member ranks) of this rank's role group; group is
        None when the role group has one member."""
        if self.is_conv:
            return self.conv_group, self.conv_ranks
        return self.fc_group, self.fc_ranks

    def peer_exchange(self, engine) -> "PeerExchange":
        """Map this role group's gradient / reduced-gradient / flag buffers
        into every member (CUDA IPC over NVLink) for the fused exchange +
        update (stz_allreduce_sgd)."""
        group, ranks = self.group_of_role()
        return PeerExchange(engine, group, ranks.index(self.rank), len(ranks))


class _IpcMap:
    """CUDA-IPC handles of local tensors and the mapping of peers' handles
    (each peer allocation opened once)."""

    def __init__(self):
        self._opened: dict[bytes, int] = {}

    @staticmethod
    def handle(t: torch.Tensor):
        from . import _lib
        h = ctypes.create_string_buffer(_lib.IPC_HANDLE_BYTES)
        off = ctypes.c_size_t(0)
        _lib.call("stz_ipc_handle", ctypes.c_void_p(t.data_ptr()), h, ctypes.byref(off))
        return bytes(h.raw), int(off.value)

    def open(self, handle: bytes, off: int) -> int:
        from . import _lib
        base = self._opened.get(handle)
        if base is None:
            out = ctypes.c_void_p(0)
            _lib.call("stz_ipc_open", ctypes.create_string_buffer(handle, len(handle)),
                      ctypes.byref(out))
            base = self._opened[handle] = int(out.value)
        return base + off

    def close(self) -> None:
        from . import _lib
        for base in self._opened.values():
            _lib.call("stz_ipc_close", ctypes.c_void_p(base))
        self._opened.clear()


class PeerLink:
    """The CONV <-> FC link of the layer-separated step over peer memory
    (reference _activations_phase / collect_group_activations /
    _boundary_phase, stanza_runtime.py:64-85, :228-307; kernels
    stz_link_* in csrc/stz_peer.cuh).

    Per micro-batch j (kb = K / m rows per CONV worker):

    * CONV worker i -> its FC worker: ``put_acts`` stores its kb boundary
      rows as fp32 into the FC worker's staging rows [(j*g + pos)*kb, ...)
      and its labels into the FC worker's label rows, then sets slot
      pos*m + j; the FC worker's ``get_acts(j)`` waits for the g slots of
      micro-batch j and splits the g*kb staged rows into its input rows --
      the FC input is laid out [micro][member][kb], members ascending (the
      reference's concat order, :266-267);
    * FC worker -> each member: ``put_grads(j)`` stores member pos's kb
      boundary-gradient rows into that member's staging rows [j*kb, ...)
      and sets its slot j; the CONV worker's ``get_grads(j)`` waits and
      splits them into its boundary-gradient rows.

    Collective constructor (every rank of the world, handle exchange over
    torch.distributed, any backend)."""

    def __init__(self, comm: "RoleComm", device, k: int, micro: int, a: int,
                 dst=None, labels=None):
        from . import _lib
        self.comm, self.k, self.m, self.a = comm, k, micro, a
        self.kb = k // micro
        dev = torch.device(device)
        self.device = dev
        self.flags = torch.zeros(_lib.LINK_FLAG_WORDS, dtype=torch.int32, device=dev)
        self.dst = dst                 # Split receiving the split rows (FC input / CONV gboundary)
        self.labels = labels           # FC: int32 [g*K] label rows
        if comm.is_conv:
            self.g = len(comm.members(comm.fc_index_of(comm.index)))
            self.pos = comm.members(comm.fc_index_of(comm.index)).index(comm.index)
            self.stage = torch.zeros(k * a, dtype=torch.float32, device=dev)
        else:
            self.g = len(comm.members(comm.index))
            self.stage = torch.zeros(self.g * k * a, dtype=torch.float32, device=dev)
        if self.g * micro > _lib.LINK_SLOTS:
            raise ValueError(f"{self.g} members x {micro} micro-batches exceed "
                             f"{_lib.LINK_SLOTS} link slots")
        torch.cuda.synchronize(dev)       # flags are zero before any peer can write them
        self._ipc = _IpcMap()
        mine = [self._ipc.handle(self.flags), self._ipc.handle(self.stage),
                self._ipc.handle(labels) if labels is not None else None]
        objs = [None] * comm.world
        dist.all_gather_object(objs, mine)
        self.fail_word = None
        if comm.is_conv:
            fc = comm.fc_rank_of(comm.index)
            fl, st, lb = objs[fc]
            self._peer_flags = self._ipc.open(*fl)
            self._peer_stage = self._ipc.open(*st)
            self._peer_labels = self._ipc.open(*lb)
        else:
            self._members = []
            for i in comm.members(comm.index):
                fl, st, _ = objs[i]
                self._members.append((self._ipc.open(*fl), self._ipc.open(*st)))
        dist.barrier()

    def _stream(self):
        from .tensor_core import stream_of
        return stream_of(self.device)

    def begin(self) -> None:
        from . import _lib
        _lib.call("stz_link_begin", self.flags.data_ptr(), self._stream())

    def put_acts(self, j: int, rows, labels: torch.Tensor) -> None:
        """CONV side: ``rows`` = the Split view of micro-batch j's boundary
        activations (kb rows), ``labels`` its kb int32 labels."""
        from . import _lib
        kb, a = self.kb, self.a
        row0 = (j * self.g + self.pos) * kb
        _lib.call("stz_link_put", rows.ptr(), rows.ps, kb, a, rows.width,
                  self._peer_stage + row0 * a * 4, labels.data_ptr(),
                  self._peer_labels + row0 * 4, self.flags.data_ptr(),
                  self._peer_flags + 4 * (self.pos * self.m + j), self._stream(),
                  nbytes=kb * a * 10.0 + kb * 8.0, tag="link_put_acts")

    def get_acts(self, j: int) -> None:
        """FC side: wait for every member's micro-batch j, then split its
        g*kb staged rows into the input rows [j*g*kb, (j+1)*g*kb)."""
        from . import _lib
        gk = self.g * self.kb
        out = self.dst.rows_view(j * gk, (j + 1) * gk)
        _lib.call("stz_link_get", self.stage.data_ptr() + j * gk * self.a * 4, gk, self.a,
                  out.ptr(), out.ps, out.width, self.flags.data_ptr(), j, self.g, self.m,
                  self._stream(), nbytes=gk * self.a * 10.0, tag="link_get_acts")

    def put_grads(self, j: int, rows) -> None:
        """FC side: ``rows`` = the Split view of micro-batch j's g*kb boundary
        gradient rows ([member][kb]); member pos gets its kb rows."""
        from . import _lib
        kb, a = self.kb, self.a
        for pos, (fl, st) in enumerate(self._members):
            v = rows.rows_view(pos * kb, (pos + 1) * kb)
            _lib.call("stz_link_put", v.ptr(), v.ps, kb, a, v.width, st + j * kb * a * 4,
                      None, None, self.flags.data_ptr(), fl + 4 * j, self._stream(),
                      nbytes=kb * a * 10.0, tag="link_put_grads")

    def get_grads(self, j: int) -> None:
        """CONV side: wait for micro-batch j's boundary gradient, then split
        it into rows [j*kb, (j+1)*kb) of the boundary-gradient buffer."""
        from . import _lib
        kb = self.kb
        out = self.dst.rows_view(j * kb, (j + 1) * kb)
        _lib.call("stz_link_get", self.stage.data_ptr() + j * kb * self.a * 4, kb, self.a,
                  out.ptr(), out.ps, out.width, self.flags.data_ptr(), j, 1, 1,
                  self._stream(), nbytes=kb * self.a * 10.0, tag="link_get_grads")

    def probe(self, src_rows, labels=None, reps: int = 20) -> dict:
        """Time the step's own exchange pattern alone (collective, after
        training): ``reps`` back-to-back round trips of micro-batch 0 --
        CONV: begin, put_acts(0), get_grads(0); FC: begin, get_acts(0),
        put_grads(0) -- on the real buffers, no compute in between.
        ``src_rows``: the Split rows this rank sends (CONV: its kb boundary
        rows; FC: its g*kb boundary-gradient rows).  Returns the mean
        milliseconds per round trip (max over ranks) and the bytes one
        round trip moves into + out of this rank's FC worker."""
        torch.cuda.synchronize(self.device)
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            self.begin()
            if self.comm.is_conv:
                self.put_acts(0, src_rows, labels)
                self.get_grads(0)
            else:
                self.get_acts(0)
                self.put_grads(0, src_rows)
        e1.record()
        torch.cuda.synchronize(self.device)
        t = torch.tensor([e0.elapsed_time(e1) / reps], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return {"round_trip_ms": float(t.item()),
                "bytes_per_direction": self.g * self.kb * self.a * 4}

    def ceiling(self, nbytes: int = 256 << 20, reps: int = 5) -> float | None:
        """Single-peer link ceiling of the put kernel (collective): CONV
        worker 0 stores ``nbytes`` of fp32 into a buffer mapped from its FC
        worker, timed on the sender (the kernel's closing system fence waits
        for the stores to land).  GB/s on rank 0, None elsewhere."""
        from . import _lib
        from .engine import Split
        d = 8192
        rows = max(1, nbytes // (4 * d))
        fc0 = self.comm.fc_rank_of(0)
        me = self.comm.rank
        dst = torch.empty(rows * d if me == fc0 else 1, dtype=torch.float32, device=self.device)
        h = [self._ipc.handle(dst)] if me == fc0 else [None]
        objs = [None] * self.comm.world
        dist.all_gather_object(objs, h[0])
        gbs = torch.zeros(1, dtype=torch.float64)
        if me == 0:
            src = Split.alloc("rows", (rows, d), d, self.device)
            remote = self._ipc.open(*objs[fc0])
            slot = torch.zeros(1, dtype=torch.int32, device=self.device)   # local dummy slot

            def put():
                _lib.call("stz_link_put", src.ptr(), src.ps, rows, d, d, remote, None, None,
                          self.flags.data_ptr(), slot.data_ptr(), self._stream())
            put()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                put()
            e1.record()
            torch.cuda.synchronize(self.device)
            gbs[0] = rows * d * 4 / (e0.elapsed_time(e1) / reps / 1e3) / 1e9
        dist.barrier()
        return float(gbs.item()) if me == 0 else None

    def failure(self) -> str | None:
        """Description of a timed-out wait (reads the status word: syncs)."""
        from . import _lib
        st = int(self.flags[_lib.LINK_STATUS].item())
        if st == 0:
            return None
        slot = st & 0xFFFF
        epoch = int(self.flags[_lib.LINK_EPOCH].item())
        if self.comm.is_conv:
            src = f"fc{self.comm.fc_index_of(self.comm.index)}"
            return f"no boundary gradients from {src} (micro-batch {slot}, step {epoch})"
        pos, j = divmod(slot, self.m)
        i = self.comm.members(self.comm.index)[pos]
        return f"no activations from conv{i} (micro-batch {j}, step {epoch})"

    def close(self) -> None:
        self._ipc.close()


class PeerExchange:
    """Gradient exchange + momentum SGD of one role group over NVLink peer
    memory, without NCCL on the data path (stanza_runtime.py:309-350;
    kernels in csrc/stz_peer.cuh).

    Each member owns its engine's flat gradient vector, a reduced-gradient
    vector of the same length and a flag block.  Their CUDA-IPC handles are
    exchanged once over the role group (host plumbing); every member then
    holds device pointers to every other member's buffers, and one call to
    stz_allreduce_sgd per iteration does barrier -> reduce-push (member r sums
    chunk r of all gradients in group-rank order and stores it into every
    member's reduced vector) -> barrier -> SGD + split-plane repack from the
    local reduced vector.  Every replica ends bit-identical."""

    def __init__(self, engine, group, me: int, nranks: int):
        from . import _lib
        self.engine = engine
        self.me, self.nranks = me, nranks
        dev = engine.device
        self.flags = torch.zeros(_lib.PEER_FLAG_WORDS, dtype=torch.int32, device=dev)
        self.red = torch.zeros(engine.total, dtype=torch.float32, device=dev) if nranks > 1 \
            else engine.grad_flat
        self._ipc = _IpcMap()
        grads, reds, flags = [0] * nranks, [0] * nranks, [0] * nranks
        grads[me], reds[me], flags[me] = (engine.grad_flat.data_ptr(), self.red.data_ptr(),
                                          self.flags.data_ptr())
        if nranks > 1:
            torch.cuda.synchronize(dev)       # flags are zero before any peer can write them
            mine = [self._ipc.handle(t) for t in (engine.grad_flat, self.red, self.flags)]
            objs = [None] * nranks
            dist.all_gather_object(objs, mine, group=group)
            for j, theirs in enumerate(objs):
                if j == me:
                    continue
                grads[j], reds[j], flags[j] = (self._ipc.open(h, off) for h, off in theirs)
            dist.barrier(group=group)
        self._grads = _lib.ptr_array(grads)
        self._reds = _lib.ptr_array(reds)
        self._flags = _lib.ptr_array(flags)

    def run(self, n: int, lr: float, mu: float) -> None:
        """This member's exchange + update of one iteration (collective: every
        member of the group calls it once per iteration, in the same order)."""
        from . import _lib
        from .tensor_core import inv_batch, ptr, stream_of
        eng = self.engine
        ranges, nr, fused = eng.fused_pack_ranges()
        _lib.call("stz_allreduce_sgd", self._grads, self._reds, self._flags, self.nranks,
                  self.me, ptr(eng.params_flat), ptr(eng.vel_flat), eng.total, float(lr),
                  float(mu), inv_batch(n), ranges, nr, stream_of(eng.device),
                  tag=f"{eng.tag}exchange_sgd",
                  nbytes=20.0 * eng.total + 6.0 * eng.fused_param_count())
        eng.pack_weights(skip=fused)

    def failure(self) -> str | None:
        """Description of a timed-out barrier (reads the status word: syncs)."""
        from . import _lib
        st = int(self.flags[_lib.PEER_FLAG_STATUS].item())
        if st == 0:
            return None
        return f"group member {st & 0xFFFF} never reached the gradient exchange"

    def close(self) -> None:
        self._ipc.close()

