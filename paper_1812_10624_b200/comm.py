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

Micro-batch pipelining posts the two P2P directions
asynchronously: a CONV worker sends every micro-batch's activations before
it receives any boundary gradient, while its FC worker alternates receive /
compute / send.  Each direction therefore runs on its own communicator (own
NCCL stream), so neither queue can block the other.
"""

from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist

from .roles import plan_groups


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
        dev = torch.device(device) if dist.get_backend() == "nccl" else torch.device("cpu")
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
        dist.all_reduce(t, op=dist.ReduceOp.SUM)

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
        self._opened: dict[bytes, int] = {}
        grads, reds, flags = [0] * nranks, [0] * nranks, [0] * nranks
        grads[me], reds[me], flags[me] = (engine.grad_flat.data_ptr(), self.red.data_ptr(),
                                          self.flags.data_ptr())
        if nranks > 1:
            torch.cuda.synchronize(dev)       # flags are zero before any peer can write them
            mine = [self._handle(t) for t in (engine.grad_flat, self.red, self.flags)]
            objs = [None] * nranks
            dist.all_gather_object(objs, mine, group=group)
            for j, theirs in enumerate(objs):
                if j == me:
                    continue
                grads[j], reds[j], flags[j] = (self._open(h, off) for h, off in theirs)
            dist.barrier(group=group)
        self._grads = _lib.ptr_array(grads)
        self._reds = _lib.ptr_array(reds)
        self._flags = _lib.ptr_array(flags)

    @staticmethod
    def _handle(t: torch.Tensor):
        from . import _lib
        h = ctypes.create_string_buffer(_lib.IPC_HANDLE_BYTES)
        off = ctypes.c_size_t(0)
        _lib.call("stz_ipc_handle", ctypes.c_void_p(t.data_ptr()), h, ctypes.byref(off))
        return bytes(h.raw), int(off.value)

    def _open(self, handle: bytes, off: int) -> int:
        """Peer allocation base (opened once per allocation) + offset."""
        from . import _lib
        base = self._opened.get(handle)
        if base is None:
            out = ctypes.c_void_p(0)
            _lib.call("stz_ipc_open", ctypes.create_string_buffer(handle, len(handle)),
                      ctypes.byref(out))
            base = self._opened[handle] = int(out.value)
        return base + off

    def run(self, n: int, lr: float, mu: float) -> None:
        """This member's exchange + update of one iteration (collective: every
        member of the group calls it once per iteration, in the same order)."""
        from . import _lib
        from .tensor_core import inv_batch, ptr, stream_of
        eng = self.engine
        ranges, nr, fused = eng.fused_pack_ranges()
        _lib.call("stz_allreduce_sgd", self._grads, self._reds, self._flags, self.nranks,
                  self.me, ptr(eng.params_flat), ptr(eng.vel_flat), eng.total, float(lr),
                  float(mu), inv_batch(n), ranges, nr, stream_of(eng.device))
        eng.pack_weights(skip=fused)

    def close(self) -> None:
        from . import _lib
        for base in self._opened.values():
            _lib.call("stz_ipc_close", ctypes.c_void_p(base))
        self._opened.clear()

