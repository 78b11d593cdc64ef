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
