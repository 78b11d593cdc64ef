"""The one-process-per-GPU exchange (comm.RoleComm) on CPU tensors over
gloo: gather into FC input rows in ascending CONV order, scatter of boundary
rows, role-group allreduce -- world sizes 2 (1:1), 3 (2:1), 4 (2:2, 3:1) and 8
(7:1, 6:2: the 8-GPU splits, fan-in 7 and two FC groups of 3)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, n_conv, n_fc, port, q, gap_view=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1812_10624_b200.comm import RoleComm
        comm = RoleComm(n_conv, n_fc)
        k, a = 3, 5
        out = {}
        if comm.is_conv:
            i = comm.index
            acts = torch.full((k, a), float(i + 1)) + torch.arange(k * a).reshape(k, a) / 100
            labels = torch.full((k,), i, dtype=torch.int32)
            if gap_view:   # a global-pool boundary: NHWC [K,1,1,C8] rows, same bytes as [K,C8]
                acts = acts.reshape(k, 1, 1, a)
            comm.gather_activations([acts, labels], None)
            gy = torch.zeros(k, a)
            comm.scatter_boundary(None, [gy])
            out["gy"] = gy
            g = torch.full((7,), float(i + 1))
            comm.allreduce_grads(g)
            out["g"] = g
        else:
            members = comm.members(comm.index)
            fc_in = torch.zeros(len(members) * k, a)
            fc_lab = torch.zeros(len(members) * k, dtype=torch.int32)
            comm.gather_activations(None, [[fc_in[p * k:(p + 1) * k], fc_lab[p * k:(p + 1) * k]]
                                           for p in range(len(members))])
            out["fc_in"], out["fc_lab"], out["members"] = fc_in, fc_lab, members
            neg = -fc_in
            comm.scatter_boundary([[neg[p * k:(p + 1) * k]] for p in range(len(members))], None)
            g = torch.full((4,), 10.0 * (comm.index + 1))
            comm.allreduce_grads(g)
            out["g"] = g
        q.put((rank, {key: (v.tolist() if torch.is_tensor(v) else v) for key, v in out.items()}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_conv,n_fc,gap_view", [(1, 1, False), (2, 1, False), (2, 2, False),
                                                 (3, 1, False), (2, 1, True), (7, 1, False),
                                                 (6, 2, False)])
def test_role_exchange(n_conv, n_fc, gap_view):
    """gap_view: the CONV side sends its boundary as the [K,1,1,C] tensor a
    ResNet trunk's global pool leaves into [K,C] rows."""
    world = n_conv + n_fc
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, n_conv, n_fc, port, q, gap_view))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    k, a = 3, 5
    base = torch.arange(k * a).reshape(k, a) / 100
    from paper_1812_10624_b200.roles import plan_groups
    conv_to_fc = plan_groups(n_conv, n_fc)
    for r in range(n_conv, world):
        j = r - n_conv
        members = [i for i, f in enumerate(conv_to_fc) if f == j]
        fc_in = torch.tensor(res[r]["fc_in"])
        for pos, i in enumerate(members):
            assert torch.allclose(fc_in[pos * k:(pos + 1) * k], base + (i + 1))
            assert res[r]["fc_lab"][pos * k:(pos + 1) * k] == [i] * k
        expect_fc = sum(10.0 * (jj + 1) for jj in range(n_fc))
        assert res[r]["g"] == [expect_fc] * 4
    for i in range(n_conv):
        assert torch.allclose(torch.tensor(res[i]["gy"]), -(base + (i + 1)))
        assert res[i]["g"] == [float(sum(range(1, n_conv + 1)))] * 7



def _pipelined_worker(rank, world, n_conv, n_fc, m, port, q):
    """The posting order of StanzaCluster._step_pipelined: a CONV worker
    posts every micro-batch's activations, then every boundary receive; its
    FC worker alternates receive -> compute -> send per micro-batch."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1812_10624_b200.comm import RoleComm
        comm = RoleComm(n_conv, n_fc)
        comm.warm("cpu")
        k, a = 4 * m, 3
        kb = k // m
        out = {}
        if comm.is_conv:
            i = comm.index
            acts = 100.0 * (i + 1) + torch.arange(k * a, dtype=torch.float32).reshape(k, a)
            labels = torch.arange(k, dtype=torch.int32) + 1000 * i
            gy = torch.zeros(k, a)
            sends, recvs = [], []
            for j in range(m):
                sends += comm.post_activations([acts[j * kb:(j + 1) * kb],
                                                labels[j * kb:(j + 1) * kb]], None)
            for j in range(m):
                recvs += comm.post_boundary(None, [gy[j * kb:(j + 1) * kb]])
            for w in recvs + sends:
                w.wait()
            out["gy"] = gy
        else:
            members = comm.members(comm.index)
            g = len(members)
            fc_in = torch.zeros(g * k, a)
            fc_lab = torch.zeros(g * k, dtype=torch.int32)
            sends = []
            for j in range(m):
                base = j * g * kb
                for w in comm.post_activations(None, [
                        [fc_in[base + p * kb:base + (p + 1) * kb],
                         fc_lab[base + p * kb:base + (p + 1) * kb]] for p in range(g)]):
                    w.wait()
                gx = -fc_in[base:base + g * kb]          # the FC block's "input gradient"
                sends += comm.post_boundary([[gx[p * kb:(p + 1) * kb].clone()]
                                             for p in range(g)], None)
            for w in sends:
                w.wait()
            out["fc_in"], out["fc_lab"], out["members"] = fc_in, fc_lab, members
        q.put((rank, {key: (v.tolist() if torch.is_tensor(v) else v) for key, v in out.items()}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_conv,n_fc,m", [(1, 1, 2), (2, 1, 4), (2, 2, 3), (7, 1, 2),
                                           (6, 2, 2)])
def test_pipelined_exchange(n_conv, n_fc, m):
    world = n_conv + n_fc
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pipelined_worker, args=(r, world, n_conv, n_fc, m, port, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    k, a = 4 * m, 3
    kb = k // m
    from paper_1812_10624_b200.roles import plan_groups
    conv_to_fc = plan_groups(n_conv, n_fc)

    def acts_of(i):
        return 100.0 * (i + 1) + torch.arange(k * a, dtype=torch.float32).reshape(k, a)

    for r in range(n_conv, world):
        members = [i for i, f in enumerate(conv_to_fc) if f == r - n_conv]
        g = len(members)
        fc_in = torch.tensor(res[r]["fc_in"])
        lab = res[r]["fc_lab"]
        for j in range(m):                      # layout [micro-batch][member][kb]
            for pos, i in enumerate(members):
                lo = j * g * kb + pos * kb
                assert torch.equal(fc_in[lo:lo + kb], acts_of(i)[j * kb:(j + 1) * kb])
                assert lab[lo:lo + kb] == list(range(j * kb + 1000 * i, (j + 1) * kb + 1000 * i))
    for i in range(n_conv):
        assert torch.equal(torch.tensor(res[i]["gy"]), -acts_of(i))
