"""Benchmark of the B200 layer-separated training step (Stanza, arXiv 1812.10624).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--model alexnet_exec]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...
    python bench.py --impl reference ...      # the CPU reference arm

One step = one BSP layer-separated iteration (reference
stanza_runtime.py:352-375) over the configured workload: CONV trunk forward
on every CONV worker's K images, activation gather, FC head forward /
SoftmaxCE / backward, boundary-gradient scatter, CONV trunk backward,
CONV-group (and FC-group) gradient allreduce, momentum SGD -- nothing
skipped.  Roles per GPU count (roles.GPU_ROLES): 1 GPU co-locates CONV and
FC (1:1 on one device), 2 -> 1:1, 4 -> 3:1, 8 -> 7:1; K images per CONV
worker are fixed, so scaling is weak.  Rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import datetime
import json
import os
import statistics
import subprocess
import sys
import time
from contextlib import contextmanager

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "images/sec at 1/2/4/8 B200 (CONV:FC split); FC tensor-pipe %; NVLink GB/s"
UNIT = "images/sec"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--model", default="alexnet_exec")
    ap.add_argument("--batch-k", type=int, default=None)
    ap.add_argument("--fc-workers", type=int, default=None)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--pool", type=int, default=4, help="device-resident input batches")
    ap.add_argument("--eager", action="store_true", help="no CUDA graph (N=1 uses graphs)")
    ap.add_argument("--no-segment-graphs", action="store_true",
                    help="N>1: run every compute segment eagerly (debugging)")
    ap.add_argument("--exchange", default=None, choices=["peer", "nccl"],
                    help="N>1 gradient exchange + update: fused NVLink peer-memory kernels "
                         "(default) or NCCL all_reduce + SGD")
    ap.add_argument("--micro", type=int, default=None,
                    help="micro-batches per iteration for N>1 (default: 4 when K allows)")
    ap.add_argument("--no-autotune", action="store_true",
                    help="keep the cost model's GEMM tile shapes (no measured override)")
    ap.add_argument("--band", type=int, default=None, choices=[0, 1, 2],
                    help="shifted-window conv kernels: 0 off, 1 unpadded convs (default), "
                         "2 padded convs too")
    ap.add_argument("--no-nvlink-probe", action="store_true",
                    help="N>1: skip the untimed CONV<->FC transfer probe after the step")
    return ap.parse_args()


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


# ---------------------------------------------------------------------------
# CPU side: oracle port (the reference algorithm restated; test infra)
# ---------------------------------------------------------------------------

def blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        return max([d.get("num_threads", 1) for d in threadpool_info()] or [1])
    except Exception:  # pragma: no cover
        return 1


def host_info() -> dict:
    import platform
    import numpy as np
    cpu = ""
    try:
        with open("/proc/cpuinfo") as fh:
            cpu = next((l.split(":", 1)[1].strip() for l in fh if l.startswith("model name")), "")
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu": cpu or platform.processor(),
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS"),
            "blas_threads": blas_threads(), "numpy": np.__version__}


_REF_K = {"alexnet_exec": 128, "vgg16_exec": 64, "resnet50_exec": 32, "inception_v3_exec": 32}


def reference_sample(model: str, n_conv: int, n_fc: int, k: int) -> dict:
    """One bounded sample of the reference iteration on the host (the oracle
    port, pinned bit-exact to the reference's StanzaCluster), timed per part
    as BASELINE.md §2b item 3 prescribes:

    * t_img: the CONV trunk forward + backward on ONE image (the reference
      runs every CONV worker's trunk sequentially, stanza_runtime.py:218,
      :366, so a worker's K images cost K * t_img);
    * t_fc: one FC worker's step at its full M = (group size) * K rows --
      forward, SoftmaxCE, backward (stanza_runtime.py:255-276);
    * t_upd: the FC-group gradient sum (n_fc > 1) and the momentum SGD of
      every replica (stanza_runtime.py:309-350).

    The reference iteration is n_conv*K*t_img + n_fc*t_fc + t_upd
    (extrapolated from the measured parts; the FC workers run sequentially
    in the reference's _fc_step loop)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import stanza_oracle as orc
    table = {"alexnet_exec": orc.alexnet_layers, "vgg16_exec": orc.vgg16_layers,
             "resnet50_exec": orc.resnet_layers}
    if model in table:
        layers, shape = table[model]()
    else:   # the oracle runs any spec in its tuple grammar (e.g. the Inception kinds)
        from paper_1812_10624_b200.model_partition import builtin_model
        from paper_1812_10624_b200.tensor_core import as_tuple
        spec = builtin_model(model)
        layers, shape = [as_tuple(l) for l in spec.layers], tuple(spec.input_shape)
    cut = orc.split_index(layers)
    front, back = layers[:cut], layers[cut:]
    params = orc.seeded_init(layers, 3)
    conv_p, fc_p = params[:cut], params[cut:]
    mk = orc.batch_fn(shape, 1, 7, classes=1000)
    x, _ = mk(0, 0)
    t0 = time.perf_counter()
    a, cache = orc.block_forward(front, conv_p, x)
    orc.block_backward(front, conv_p, cache, np.ones_like(a))   # incl. layer-0 dgrad, as the reference
    t_img = time.perf_counter() - t0
    m = max(orc.plan_groups(n_conv, n_fc).count(j) for j in range(n_fc)) * k
    gen = np.random.Generator(np.random.PCG64(11))
    xs = gen.standard_normal((m, a.shape[1])).astype(np.float32)
    ys = gen.integers(0, 1000, size=m)
    t0 = time.perf_counter()
    out, fcache = orc.block_forward(back, fc_p, xs, labels=ys)
    _, fgrads = orc.block_backward(back, fc_p, fcache, None)
    t_fc = time.perf_counter() - t0
    conv_g = [[np.zeros_like(t) for t in row] for row in conv_p]
    t0 = time.perf_counter()
    if n_fc > 1:
        orc.allreduce_sum([orc._flat(fgrads)] * n_fc, 0)
    for _ in range(n_fc):
        orc.sgd_update(fc_p, fgrads, [[np.zeros_like(t) for t in r] for r in fc_p], n_conv * k,
                       0.01, 0.9)
    for _ in range(n_conv):
        orc.sgd_update(conv_p, conv_g, [[np.zeros_like(t) for t in r] for r in conv_p],
                       n_conv * k, 0.01, 0.9)
    t_upd = time.perf_counter() - t0
    t_iter = n_conv * k * t_img + n_fc * t_fc + t_upd
    return {"t_img": t_img, "t_fc": t_fc, "t_upd": t_upd, "t_iter": t_iter, "m": m}


def reference_baseline(model, n_conv, n_fc, k, steps, budget=150.0) -> dict:
    samples, t_start = [], time.perf_counter()
    for _ in range(max(steps, 1)):
        samples.append(reference_sample(model, n_conv, n_fc, k))
        if time.perf_counter() - t_start > budget:
            break
    t_iter = statistics.median(s["t_iter"] for s in samples)
    parts = {key: statistics.median(s[key] for s in samples) for key in ("t_img", "t_fc", "t_upd")}
    return {"value": n_conv * k / t_iter, "t_iter": t_iter, "samples": len(samples),
            "m": samples[0]["m"], **parts}


def reference_arm(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    from paper_1812_10624_b200.roles import gpu_roles
    n_conv, n_fc = gpu_roles(args.gpus, args.fc_workers)
    k = args.batch_k or _REF_K.get(args.model, 128)
    for _ in range(min(args.warmup, 1)):
        reference_sample(args.model, n_conv, n_fc, k)
    ref = reference_baseline(args.model, n_conv, n_fc, k, args.steps)
    info = host_info()
    line = {
        "impl": "reference", "metric": METRIC, "value": ref["value"], "unit": UNIT,
        "n_gpus": args.gpus, "steps": ref["samples"], "warmup": min(args.warmup, 1),
        "ms_per_step": ref["t_iter"] * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64-accumulate/f32-storage",
        "data": "synthetic",
        "config": workload_config(args, n_conv, n_fc, k),
        "cpu_baseline": {"value": ref["value"], "unit": UNIT, "cores": info["blas_threads"],
                         "kind": "port", "host": info, "sample": _sample_text(ref, n_conv, n_fc,
                                                                              k)},
        "e2e": {"value": ref["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _sample_text(ref, n_conv, n_fc, k):
    return (f"oracle/stanza_oracle.py (the reference algorithm, pinned bit-exact to its "
            f"StanzaCluster) per part, median of {ref['samples']} samples: CONV trunk "
            f"fwd+bwd {ref['t_img']:.3f} s/image, FC step at M={ref['m']} {ref['t_fc']:.3f} s, "
            f"exchange+SGD of every replica {ref['t_upd']:.3f} s; iteration = {n_conv}*{k}*t_img "
            f"+ {n_fc}*t_fc + t_upd = {ref['t_iter']:.1f} s (extrapolated: the reference runs "
            f"CONV workers and FC workers sequentially, stanza_runtime.py:218,:255-276,:366)")


def workload_config(args, n_conv, n_fc, k):
    side = {"inception_v3_exec": 299}.get(args.model, 224)
    return {"workload": f"{args.model} {side}x{side} synthetic, K={k} images per CONV worker, "
                        f"{n_conv} CONV : {n_fc} FC" + (" co-located on 1 GPU"
                                                         if args.gpus == 1 else ""),
            "model": args.model, "batch_per_conv_worker": k, "n_conv": n_conv, "n_fc": n_fc,
            "global_batch": n_conv * k, "parallelism": f"layer-separated {n_conv}:{n_fc}",
            "l2": "inputs larger than L2: pool of device-resident batches rotated"}


# ---------------------------------------------------------------------------
# GPU side
# ---------------------------------------------------------------------------

class ClockSampler:
    """nvidia-smi sampling (recipe clocks line).  Started before the warm-up
    so it is already emitting when the timed region begins; the summary keeps
    the samples whose timestamps fall inside the timed window (mark_start /
    mark_end), falling back to every sample taken under load (and saying so)
    when the window is shorter than the sampling period."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.t0 = self.t1 = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_gpu{index}.csv")

    def start(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=self.fh, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        if self.proc is not None:
            import atexit
            atexit.register(self.stop)   # never leave nvidia-smi running
        return self

    def mark_start(self):
        self.t0 = datetime.datetime.now()

    def mark_end(self):
        self.t1 = datetime.datetime.now()

    def stop(self):
        if self.proc is not None and self.proc.poll() is None:
            self.proc.terminate()
            self.proc.wait(timeout=5)
            self.fh.close()

    def summary(self):
        if self.proc is None or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f")
                rows.append((ts, float(parts[1]), float(parts[2]), parts[5:9]))
            except ValueError:
                continue
        window = "timed"
        sel = [r for r in rows if self.t0 and self.t1 and self.t0 <= r[0] <= self.t1]
        if not sel:   # timed region shorter than the sampling period: all samples under load
            sel, window = rows, "load"
        reasons = set()
        for r in sel:
            for name, flag in zip(names, r[3]):
                if flag.lower() == "active":
                    reasons.add(name)
        sm = [r[1] for r in sel]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": sel[-1][2] if sel else None, "reasons": sorted(reasons),
                "samples": len(sm), "window": window}


class CallTimer:
    """PROFILE_HOOK for paper_1812_10624_b200._lib: CUDA events around each
    ABI call on the launching (current) stream."""

    def __init__(self, torch):
        self.torch = torch
        self.records = []

    @contextmanager
    def __call__(self, name, args, flops=0.0, tag=None, nbytes=0.0):
        t = self.torch
        e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
        e0.record()
        yield
        e1.record()
        self.records.append(((tag or name, float(flops), float(nbytes)), e0, e1))

    def table(self):
        self.torch.cuda.synchronize()
        agg = {}
        for key, e0, e1 in self.records:
            ms = e0.elapsed_time(e1)
            tot, cnt = agg.get(key, (0.0, 0))
            agg[key] = (tot + ms, cnt + 1)
        return agg


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            p = json.load(fh)
        return p["bf16_tflops"], p["hbm_gbs"], "measured (MEASURED_PEAKS.json)"
    except (OSError, KeyError, ValueError):
        return 1590.0, 6650.0, "fallback (B200_PROFILING.md)"


def committed_traffic(kernel_key: str):
    path = os.path.join(ROOT, "profiles", "dram_traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(kernel_key)
    except (OSError, ValueError):
        return None


def nvlink_probe(torch, dist, cl, reps: int = 20) -> dict:
    """CONV<->FC traffic of the step through the step's own link calls,
    timed OUTSIDE the timed region (inside the step the transfers overlap
    compute, so no phase clock is a transfer time).  ``reps`` back-to-back
    round trips of micro-batch 0 on the real buffers (PeerLink.probe:
    CONV put_acts -> FC get_acts -> FC put_grads -> CONV get_grads, 4 B per
    element on the link, one message per member per direction), max over
    ranks; ``link_GBps`` = one 256 MiB put CONV 0 -> its FC worker (the
    same kernel, PeerLink.ceiling), the single-peer ceiling the fractions
    are taken against."""
    link = cl._link
    if link is None:
        return None
    kb = link.kb
    if cl.conv is not None:
        src = cl.conv._act(len(cl.conv.ops) - 1).rows_view(0, kb)
        labels = cl.labels[:kb] if cl.labels is not None else None
    else:
        src = cl.fcs[0].gin[0].rows_view(0, link.g * kb)
        labels = None
    rt = link.probe(src, labels, reps=reps)
    ceil = link.ceiling()
    objs = [None] * dist.get_world_size()
    dist.all_gather_object(objs, ceil)
    ceil = next(c for c in objs if c is not None)
    per_dir = rt["bytes_per_direction"]
    gbs = 2 * per_dir / (rt["round_trip_ms"] / 1e3) / 1e9
    return {
        "round_trip_ms": rt["round_trip_ms"], "bytes_per_direction": per_dir,
        "fan_in": link.g, "micro_batch_rows": kb,
        "exchange_GBps": gbs, "link_GBps": ceil, "frac_of_link": gbs / ceil if ceil else None,
        "nvlink5_GBps": 900.0, "frac_of_nvlink5": gbs / 900.0,
        "note": ("one micro-batch's gather (every member's kb x A rows, fp32 on the link, "
                 "into the FC worker) + scatter (back), through the step's PeerLink calls "
                 f"on the step's buffers, {reps} back-to-back round trips, max over ranks; "
                 "exchange_GBps = bytes into + out of the busiest FC worker / round-trip "
                 "time (includes the flag handshakes and the receivers' split kernels); "
                 "link_GBps = one 256 MiB put of the same kernel, CONV 0 -> its FC worker"),
    }


def main():
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)

    import torch
    import torch.distributed as dist

    from paper_1812_10624_b200 import _lib
    from paper_1812_10624_b200.model_partition import builtin_model
    from paper_1812_10624_b200.roles import gpu_roles
    from paper_1812_10624_b200.stanza_runtime import StanzaCluster

    rank, world, local = env_rank()
    if world != args.gpus and world == 1 and args.gpus > 1:
        raise SystemExit("--gpus N>1 must be launched with torch.distributed.run")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    lib = _lib.load()
    if args.band is not None:
        lib.stz_set_band(args.band)
    n_conv, n_fc = gpu_roles(args.gpus, args.fc_workers)
    k = args.batch_k or _REF_K.get(args.model, 4)
    spec = builtin_model(args.model, k)

    comm = None
    if world > 1:
        dist.init_process_group("cpu:gloo,cuda:nccl", device_id=dev)
        from paper_1812_10624_b200.comm import RoleComm
        comm = RoleComm(n_conv, n_fc)

    host_pool = []

    def batch_fn(it, i):   # a loader handing out pinned host batches (train(), e2e)
        return host_pool[it % len(host_pool)]

    cl = StanzaCluster(spec, n_conv=n_conv, n_fc=n_fc, batch_fn=batch_fn, lr=0.01,
                       momentum=0.9, seed=3, device=dev, comm=comm,
                       micro_batches=args.micro, exchange=args.exchange,
                       segment_graphs=not args.no_segment_graphs)
    is_conv_rank = cl.conv is not None
    classes = spec.layers[-2].out_dim
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    pool_x, pool_y = [], []
    if cl.x is not None:
        for _ in range(args.pool):
            pool_x.append(torch.randn(cl.x.shape, generator=gen, device=dev))
            pool_y.append(torch.randint(0, classes, cl.labels.shape, generator=gen,
                                        device=dev, dtype=torch.int32))
    slots = torch.zeros(max(args.steps, args.warmup, 1), dtype=torch.float64, device=dev)

    def one(i, slot=None):
        if pool_x:
            j = i % args.pool
            cl.step(slot, x=pool_x[j], labels=pool_y[j])
        else:
            cl.step(slot)

    def sync_all():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()

    clocks = ClockSampler(local).start()   # running before the timed region begins

    # warm-up (W >= 3 enforced); the measured GEMM tile shapes
    # (_lib.autotune_tiles) are chosen on the first, eager, warm-up step,
    # before any CUDA graph is captured
    warm = max(args.warmup, 3)
    tiles = {}
    for i in range(warm):
        sl = slots[i % slots.numel():i % slots.numel() + 1]
        if i == 0 and not args.no_autotune:
            tiles = _lib.autotune_tiles(lambda: one(0, sl))
        else:
            one(i, sl)
    sync_all()

    # one CUDA graph per pooled batch: the whole step (single device, or every
    # rank's part of it over the peer-memory link); exchange="nccl" keeps its
    # NCCL calls on the host and replays compute segments instead
    graphs = None
    if not args.eager and cl.graph_capable():
        graph_slots = torch.zeros((args.pool, 1), dtype=torch.float64, device=dev)
        graphs = [cl.capture(pool_x[j] if pool_x else None, pool_y[j] if pool_y else None,
                             graph_slots[j]) for j in range(args.pool)]
        sync_all()
        for j in range(args.pool):
            graphs[j].replay()
        sync_all()

        def one(i, slot=None):  # noqa: F811 -- the graph replay replaces the eager step
            graphs[i % args.pool].replay()
    elif world > 1:   # segment graphs are captured on first sight: visit every batch untimed
        for i in range(args.pool):
            one(warm + i, slots[0:1])
        sync_all()

    # ---- timed region: device-resident inputs ------------------------------------
    n0 = lib.stz_launch_count()
    if pool_x:
        cl.step(slots[0:1], x=pool_x[0], labels=pool_y[0])
    else:
        cl.step(slots[0:1])
    sync_all()
    per_step_launches = lib.stz_launch_count() - n0
    launches0 = lib.stz_launch_count()
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sync_all()
    clocks.mark_start()
    e0.record(stream)
    for i in range(args.steps):
        one(i, slots[i:i + 1])
    e1.record(stream)
    torch.cuda.synchronize(dev)
    clocks.mark_end()
    launches = lib.stz_launch_count() - launches0
    if graphs is not None:   # replays launch the captured kernels without host calls
        launches = per_step_launches * args.steps
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
    ms = float(t.item())
    images = n_conv * k
    value = images / (ms / 1e3)

    # ---- e2e: StanzaCluster.train() fed from pinned host batches ----------------
    # the public entry point: each iteration's batch comes from batch_fn (here a
    # loader returning pinned host tensors), is copied host -> device on train()'s
    # side stream while the previous step runs, every step is a graph replay, and
    # every step's loss is copied back to host memory
    for j in range(len(pool_x)):
        host_pool.append((pool_x[j].cpu().pin_memory(), pool_y[j].cpu().pin_memory()))
    cl.iteration = 0
    cl.train(2)                     # captures the feed buffers' graphs, untimed
    sync_all()
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    res = cl.train(args.steps)
    e3.record(stream)
    torch.cuda.synchronize(dev)
    e2e_ms = torch.tensor([e2.elapsed_time(e3) / args.steps], dtype=torch.float64, device=dev)
    h2d = (cl.x.numel() * 4 + cl.labels.numel() * 4) if pool_x else 0
    io = torch.tensor([float(h2d), float(8 if cl.fcs else 0)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
        dist.all_reduce(io, op=dist.ReduceOp.SUM)
    e2e_ms = float(e2e_ms.item())
    finite = all(l == l for l in res.losses)

    # ---- per-call kernel timing (separate, untimed eager pass) -------------------
    timer = CallTimer(torch)
    _lib.PROFILE_HOOK = timer
    cl.time_phases = True
    if pool_x:
        cl.step(None, x=pool_x[0], labels=pool_y[0])
    else:
        cl.step(None)
    _lib.PROFILE_HOOK = None
    cl._resolve_phase_times()
    cl.time_phases = False
    calls = timer.table()
    phase_ms = cl.device_phase_ms[-1] if cl.device_phase_ms else {}

    bf16_peak, hbm_peak, peak_src = peaks()
    # dominant kernel = the ABI call with the largest total time among the
    # ones that carry algorithmic work (GEMM FLOPs or HBM bytes); the link
    # gets (which include the wait for the peer) are not kernels of the step's work
    top_key, top = None, (0.0, 0)
    for key, (tot, cnt) in calls.items():
        if (key[1] > 0 or key[2] > 0) and tot > top[0] and not key[0].startswith("link_get"):
            top_key, top = key, (tot, cnt)
    fl = top_key[1] if top_key else 0.0
    nb = top_key[2] if top_key else 0.0
    avg_ms = top[0] / max(top[1], 1)
    achieved = fl / (avg_ms / 1e3) / 1e12 if avg_ms > 0 and fl > 0 else 0.0
    hbm_bound = fl == 0.0 and nb > 0.0      # a memory-bound kernel (BatchNorm, pool, ...)
    achieved_gbs = nb / (avg_ms / 1e3) / 1e9 if avg_ms > 0 and nb > 0 else 0.0
    kernel_key = f"{args.model}:{top_key[0]}" if top_key else None
    step_ms_sum = sum(tot for tot, _ in calls.values())
    fc_fl = sum(kk[1] * c for kk, (_, c) in calls.items() if kk[0].startswith("fc"))
    fc_ms = sum(tot for kk, (tot, _) in calls.items() if kk[0].startswith("fc") and kk[1] > 0)
    per_call = {}
    for kk, (tot, c) in sorted(calls.items(), key=lambda kv: -kv[1][0]):
        mean = tot / max(c, 1)
        gbs = kk[2] / (mean / 1e3) / 1e9 if kk[2] and tot else None
        name = kk[0]
        while name in per_call:          # same tag, different shape (e.g. two SGD blocks)
            name += "'"
        per_call[name] = {"ms": mean, "n": c, "total_ms": tot,
                           "tflops": (kk[1] / (mean / 1e3) / 1e12) if kk[1] and tot else None,
                           "GBps": gbs, "hbm_frac": gbs / hbm_peak if gbs else None}
    fc_tflops = fc_fl / (fc_ms / 1e3) / 1e12 if fc_ms > 0 else None
    # FC GEMMs against their own roofline: max(BF16x6 tensor time, HBM time
    # of the weight planes + activations); at M = 128-896 rows the weight
    # read dominates ("per-FC-GEMM bound = max(flops/peak,
    # bytes/HBM)")
    fc_roof = None
    if cl.fcs:
        eng = cl.fcs[0]
        rows_b, tot_ms, tot_bound = {}, 0.0, 0.0
        for kk, (tot, cnt) in calls.items():
            tag, fl = kk[0], kk[1]
            if not tag.startswith("fc") or fl <= 0 or "_" not in tag:
                continue
            li = int(tag[2:].split("_")[0])
            lay = eng.ops[li].layer
            m_rows = fl / (2.0 * lay.in_dim * lay.out_dim)
            w = lay.in_dim * lay.out_dim
            act = 6.0 * m_rows * (lay.in_dim + lay.out_dim)
            nbytes = act + (4.0 * w if tag.endswith("wgrad") else 6.0 * w)
            t_tc = fl / (bf16_peak / 6 * 1e12) * 1e3
            t_hbm = nbytes / (hbm_peak * 1e9) * 1e3
            mean = tot / max(cnt, 1)
            bound = max(t_tc, t_hbm)
            rows_b[tag] = {"ms": mean, "bound_ms": bound, "bound": "hbm" if t_hbm > t_tc else "tensor",
                           "frac": bound / mean if mean else None, "rows": m_rows,
                           "GBps": nbytes / (mean / 1e3) / 1e9 if mean else None}
            tot_ms += mean * cnt
            tot_bound += bound * cnt
        fc_roof = {"frac": tot_bound / tot_ms if tot_ms else None, "calls": rows_b,
                   "note": "bound = max(algorithmic FLOPs / (bf16 peak / 6), bytes / HBM peak); "
                           "bytes = weight planes (6 B/param; fp32 gradient write 4 B/param for "
                           "wgrad) + split-plane activations"}
    roofline = {
        "bound": "hbm", "kernel": kernel_key, "achieved": achieved_gbs, "peak": hbm_peak,
        "unit": "GB/s", "frac": achieved_gbs / hbm_peak if hbm_peak else None,
        "traffic": committed_traffic(kernel_key), "peak_source": peak_src,
        "note": ("achieved = algorithmic HBM bytes of that ABI call (split planes, 6 B per "
                 "element per pass) / its mean CUDA-event duration"),
        "share_of_step": top[0] / step_ms_sum if step_ms_sum else None,
        "calls": per_call,
    } if hbm_bound else {
        "bound": "tensor", "kernel": kernel_key, "achieved": achieved, "peak": bf16_peak,
        "unit": "TFLOP/s", "frac": achieved / bf16_peak if bf16_peak else None,
        "traffic": committed_traffic(kernel_key),
        "peak_source": peak_src,
        "note": ("achieved = algorithmic fp32 GEMM FLOPs (2*M*N*K of the conv/FC "
                 "contraction) / mean CUDA-event duration of that ABI call; the BF16x6 "
                 "split issues 6 bf16 MMAs per algorithmic MAC, so the tensor-pipe "
                 "occupancy is 6*frac and the scheme's own ceiling is frac = 1/6"),
        "tensor_pipe_frac": 6 * achieved / bf16_peak if bf16_peak else None,
        "share_of_step": top[0] / step_ms_sum if step_ms_sum else None,
        "calls": per_call,
    }

    probe = None
    if world > 1 and not args.no_nvlink_probe:
        probe = nvlink_probe(torch, dist, cl)

    clocks.stop()
    extras = {"rank": rank, "role": "conv" if is_conv_rank else "fc", "phase_ms": phase_ms,
              "roofline": roofline, "fc_tflops": fc_tflops, "launches": launches,
              "fc_roofline": fc_roof}
    if world > 1:
        objs = [None] * world
        dist.all_gather_object(objs, extras)
    else:
        objs = [extras]
    if rank == 0:
        conv_ex = next(o for o in objs if o["role"] == "conv")
        fc_ex = next((o for o in objs if o["fc_tflops"] is not None), conv_ex)
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            ref = reference_baseline(args.model, n_conv, n_fc, k, 1)
            info = host_info()
            cpu = {"value": ref["value"], "unit": UNIT, "cores": info["blas_threads"],
                   "kind": "port", "host": info, "sample": _sample_text(ref, n_conv, n_fc, k)}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": warm, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (N(0,1) images, uniform labels, "
                                    "device-resident pool, random-init weights)",
            "config": dict(workload_config(args, n_conv, n_fc, k), micro_batches=cl.micro,
                           exchange=cl.exchange),
            "roofline": conv_ex["roofline"],
            "cpu_baseline": cpu,
            "e2e": {"value": images / (e2e_ms / 1e3), "unit": UNIT,
                    "h2d_bytes_per_step": int(io[0].item()),
                    "d2h_bytes_per_step": int(io[1].item()),
                    "ms_per_step": e2e_ms, "losses_finite": finite,
                    "api": ("StanzaCluster.train(steps): batch_fn hands out pinned host "
                            "batches; train() copies each step's batch host -> device on a "
                            "side stream into the other of two persistent buffers while the "
                            "previous step's CUDA graph runs, and copies every step's loss "
                            "back to host memory")},
            "gpu_launches": int(sum(o["launches"] for o in objs)),
            "cuda_graph": bool(graphs is not None),
            "tile_overrides": {f"{kk[1]}": list(v) for kk, v in tiles.items()},
            "clocks": clocks.summary(),
            "fc_tensor_pipe_frac": (6 * fc_ex["fc_tflops"] / bf16_peak)
            if fc_ex["fc_tflops"] else None,
            "fc_tflops_algorithmic": fc_ex["fc_tflops"],
            "fc_roofline": fc_ex.get("fc_roofline"),
            "nvlink": probe,
            "phase_ms": {o["role"] + str(o["rank"]): o["phase_ms"] for o in objs},
            "gemm": "tcgen05 BF16x6 (3-way bf16 split, 6 MMAs, split fp32 TMEM accumulators)",
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        cl.close()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
