"""Node-assignment planner fed by constants measured on the B200 (SURVEY.md
8f row 3).

The closed-form model and the planner restate the reference's
``perf_model.py`` (stanza_iter_time :87-102, stanza_throughput :105-109,
window :64-71, assign_nodes :147-172, the constants text format :237-275):
a layer-separated iteration costs

    T_c + g * T_f + (2 g K A + max(window(n_c) P_c, window(n_f) P_fc)) * 32 / B

with g = ceil(n_c / n_f).  What changes is where the constants come from:
``measure_constants`` times the CONV block and the FC block forward+backward
on the GPU through the same engine the training step runs (CUDA events,
median over repetitions, the analogue of harness.bench_constants,
harness.py:659-707), the link bandwidth is a measured GPU-to-GPU copy over
NVLink (the nominal NVLink-5 900 GB/s per direction when the process sees one
GPU) and ``fc_memory_bytes`` is the free HBM of the device, so
``assign_nodes`` chooses among the splits one 8xB200 box offers (1:1, 3:1,
7:1, 6:2, ...) from measured numbers.

``pipelined_iter_time`` is this build's own model of its pipelined step
(stanza_runtime._step_pipelined): the FC worker's g*T_f overlaps the CONV
workers' compute, and the activation/boundary transfers of all but one
micro-batch hide behind it.  It is reported beside the reference model, not
used for parity.

    python -m paper_1812_10624_b200.planner --model alexnet_exec --nodes 8 [--measure]
"""

from __future__ import annotations

import argparse
import statistics
import sys
from dataclasses import dataclass

from .model_partition import ConfigError, Partition, builtin_model, parse_kv_text, split


class Infeasible(ValueError):
    """No node assignment satisfies the constraints (perf_model.py:26-27)."""


BITS_PER_ELEMENT = 32
NVLINK5_BYTES_PER_S = 900e9      # per direction per GPU (nominal)


@dataclass(frozen=True)
class PerfConstants:
    """Per-iteration compute times (seconds) and the link speed (bits/s),
    perf_model.py:33-55."""
    bandwidth: float = 10e9
    conv_time: float = 0.0
    fc_unit_time: float = 0.0
    ps_compute_time: float = 0.0

    def __post_init__(self):
        if self.bandwidth <= 0:
            raise ConfigError(f"bandwidth must be positive, got {self.bandwidth}")
        for name in ("conv_time", "fc_unit_time", "ps_compute_time"):
            if getattr(self, name) < 0:
                raise ConfigError(f"{name} must be nonnegative")


def window(n: int) -> int:
    """Busiest-member payload multiple of an n-member allreduce
    (perf_model.py:64-71): log2 n rounds, one more with a surplus."""
    if n < 1:
        raise ValueError(f"group size must be positive, got {n}")
    if n == 1:
        return 0
    m = n.bit_length() - 1
    return m if n == (1 << m) else m + 1


def _ceil_div(a: int, b: int) -> int:
    return -(-a // b)


def _check_pair(n_conv: int, n_fc: int) -> None:
    if n_conv < 1 or n_fc < 1:
        raise ConfigError("need at least one CONV and one FC worker, got "
                          f"n_conv={n_conv} n_fc={n_fc}")
    if n_fc > n_conv:
        raise ConfigError(f"more FC workers ({n_fc}) than CONV workers "
                          f"({n_conv}) leaves some idle")


def _wire_bits(part: Partition, n_conv: int, n_fc: int):
    g = _ceil_div(n_conv, n_fc)
    ak_bits = part.boundary_activations * part.spec.batch_k * BITS_PER_ELEMENT
    exchange = max(window(n_conv) * part.conv_params,
                   window(n_fc) * part.fc_params) * BITS_PER_ELEMENT
    return g, 2 * g * ak_bits, exchange


def stanza_iter_time(part: Partition, n_conv: int, n_fc: int, c: PerfConstants) -> float:
    """Modelled seconds per BSP layer-separated iteration (perf_model.py:87-102)."""
    _check_pair(n_conv, n_fc)
    g, transfer, exchange = _wire_bits(part, n_conv, n_fc)
    return c.conv_time + g * c.fc_unit_time + (transfer + exchange) / c.bandwidth


def stanza_throughput(part: Partition, n_conv: int, n_fc: int, c: PerfConstants) -> float:
    """Samples per second, n_conv local batches per iteration (perf_model.py:105-109)."""
    return n_conv * part.spec.batch_k / stanza_iter_time(part, n_conv, n_fc, c)


def pipelined_iter_time(part: Partition, n_conv: int, n_fc: int, c: PerfConstants,
                        micro: int = 2) -> float:
    """This build's pipelined step: max(T_c, g T_f) + one micro-batch's
    transfers + the exchange (the reference model's terms, overlapped)."""
    _check_pair(n_conv, n_fc)
    g, transfer, exchange = _wire_bits(part, n_conv, n_fc)
    return max(c.conv_time, g * c.fc_unit_time) + (transfer / micro + exchange) / c.bandwidth


@dataclass(frozen=True)
class Assignment:
    n_conv: int
    n_fc: int
    throughput: float


def assign_nodes(part: Partition, total_nodes: int, c: PerfConstants,
                 fc_memory_bytes: float | None = None, model=None) -> Assignment:
    """Best (n_conv, n_fc) split of ``total_nodes`` by exhaustive search
    (perf_model.py:147-172): n_fc <= n_conv; an FC worker must hold
    ceil(n_conv/n_fc) * K * A * 4 activation bytes within fc_memory_bytes;
    ties go to the smaller FC group.  ``model`` (default stanza_iter_time)
    may be pipelined_iter_time."""
    best: Assignment | None = None
    for n_fc in range(1, total_nodes):
        n_conv = total_nodes - n_fc
        if n_fc > n_conv:
            break
        if fc_memory_bytes is not None:
            held = _ceil_div(n_conv, n_fc) * part.spec.batch_k * part.boundary_activations * 4
            if held > fc_memory_bytes:
                continue
        t = (model or stanza_iter_time)(part, n_conv, n_fc, c)
        thr = n_conv * part.spec.batch_k / t
        if best is None or thr > best.throughput:
            best = Assignment(n_conv=n_conv, n_fc=n_fc, throughput=thr)
    if best is None:
        raise Infeasible(f"no feasible (n_conv, n_fc) split of {total_nodes} "
                         "nodes under the given constraints")
    return best


def parse_constants_text(text: str) -> PerfConstants:
    """``key value`` lines (perf_model.py:237-257); a ``name`` line is ignored."""
    values = {"bandwidth": 10e9, "conv_time": 0.0, "fc_unit_time": 0.0,
              "ps_compute_time": 0.0}
    for key, args in parse_kv_text(text):
        if key == "name":
            continue
        if key not in values:
            raise ConfigError(f"unknown constants key {key!r}")
        try:
            (raw,) = args
            values[key] = float(raw)
        except ValueError:
            raise ConfigError(f"bad {key} line: expected one number, got {args!r}") from None
    return PerfConstants(**values)


def load_constants_file(path) -> PerfConstants:
    with open(path, "r", encoding="utf-8") as fh:
        return parse_constants_text(fh.read())


def format_constants_text(c: PerfConstants, name: str = "measured") -> str:
    """The format parse_constants_text reads (perf_model.py:265-275)."""
    return "".join((f"name {name}\n",
                    f"bandwidth {c.bandwidth!r}\n",
                    f"conv_time {c.conv_time!r}\n",
                    f"fc_unit_time {c.fc_unit_time!r}\n",
                    f"ps_compute_time {c.ps_compute_time!r}\n"))


# ---------------------------------------------------------------------------
# measurement on the GPU
# ---------------------------------------------------------------------------

def measure_link_bandwidth(nbytes: int = 256 << 20, reps: int = 10):
    """(bits/s, source): a device-to-device copy cuda:0 -> cuda:1 over
    NVLink timed with CUDA events, or the nominal NVLink-5 figure when this
    process sees a single GPU."""
    import torch
    if torch.cuda.device_count() < 2:
        return NVLINK5_BYTES_PER_S * 8, "nominal NVLink 5 (one GPU visible)"
    src = torch.empty(nbytes, dtype=torch.uint8, device="cuda:0")
    dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda:1")
    dst.copy_(src)
    torch.cuda.synchronize("cuda:0")
    torch.cuda.synchronize("cuda:1")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.device(0):
        e0.record()
        for _ in range(reps):
            dst.copy_(src, non_blocking=True)
        e1.record()
        e1.synchronize()
    return nbytes * reps / (e0.elapsed_time(e1) / 1e3) * 8, "measured cuda:0 -> cuda:1 copy"


def measure_constants(spec, device=None, reps: int = 7, bandwidth: float | None = None,
                      seed: int = 0):
    """(PerfConstants, info) measured on the GPU through BlockEngine:
    conv_time = CONV block forward + backward on one K batch, fc_unit_time =
    FC block forward + backward on that batch's boundary activations,
    ps_compute_time = both (the co-located model), floored at conv_time
    (harness.py:665-707).  Medians of ``reps`` CUDA-event timings after one
    warm-up; info carries the link-bandwidth source and the free HBM."""
    import numpy as np
    import torch

    from .engine import BlockEngine
    from .tensor_core import seeded_init

    dev = torch.device(device if device is not None else "cuda")
    part = split(spec)
    layers = spec.require_layers()
    cut = part.split_index
    params = seeded_init(layers, seed)
    vel = [[np.zeros_like(t) for t in row] for row in params]
    k = spec.batch_k
    a = part.boundary_activations
    conv = BlockEngine(layers[:cut], tuple(spec.input_shape), k, dev, params[:cut], vel[:cut],
                       need_input_grad=False)
    fc = BlockEngine(layers[cut:], (a,), k, dev, params[cut:], vel[cut:], need_input_grad=True)
    gen = torch.Generator(device=dev).manual_seed(seed)
    x = torch.randn((k, *spec.input_shape), generator=gen, device=dev)
    classes = layers[-2].out_dim
    y = torch.randint(0, classes, (k,), generator=gen, device=dev, dtype=torch.int32)
    acts = conv.forward(x)
    fc.forward(acts, y)
    fc.backward()
    conv.backward(fc.gin[0])
    torch.cuda.synchronize(dev)

    def timed(fn):
        out = []
        for _ in range(reps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            out.append(e0.elapsed_time(e1) / 1e3)
        return statistics.median(out)

    def conv_step():
        conv.forward(x)
        conv.backward(fc.gin[0])

    def fc_step():
        fc.forward(acts, y)
        fc.backward()

    def full_step():
        fc.forward(conv.forward(x), y)
        fc.backward()
        conv.backward(fc.gin[0])

    t_c, t_f, t_full = timed(conv_step), timed(fc_step), timed(full_step)
    src = "given"
    if bandwidth is None:
        bandwidth, src = measure_link_bandwidth()
    free, total = torch.cuda.mem_get_info(dev)
    c = PerfConstants(bandwidth=bandwidth, conv_time=t_c, fc_unit_time=t_f,
                      ps_compute_time=max(t_full, t_c))
    return c, {"bandwidth_source": src, "hbm_free_bytes": free, "hbm_total_bytes": total,
               "reps": reps, "device": str(dev)}


def measure_fc_group_time(spec, groups=(1, 3, 7), device=None, reps: int = 7,
                          seed: int = 0) -> dict:
    """Seconds for one FC worker's share of an iteration when it serves g
    CONV batches: FC block forward + backward on g*K boundary rows plus its
    momentum update (the FC worker's critical work in the pipelined step).
    The reference model charges g * T_f; on B200 the FC GEMMs run at larger M
    more efficiently, so this is what decides 7:1 vs 6:2."""
    import numpy as np
    import torch

    from .engine import BlockEngine
    from .tensor_core import seeded_init

    dev = torch.device(device if device is not None else "cuda")
    part = split(spec)
    layers = spec.require_layers()
    cut = part.split_index
    params = seeded_init(layers, seed)
    vel = [[np.zeros_like(t) for t in row] for row in params]
    a = part.boundary_activations
    classes = layers[-2].out_dim
    out = {}
    for g in groups:
        rows = g * spec.batch_k
        fc = BlockEngine(layers[cut:], (a,), rows, dev, params[cut:], vel[cut:],
                         need_input_grad=True)
        gen = torch.Generator(device=dev).manual_seed(seed)
        x = torch.randn((rows, a), generator=gen, device=dev)
        y = torch.randint(0, classes, (rows,), generator=gen, device=dev, dtype=torch.int32)

        def step():
            fc.forward(x, y)
            fc.backward()
            fc.sgd(rows, 1e-6, 0.9)

        step()
        torch.cuda.synchronize(dev)
        ts = []
        for _ in range(reps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            step()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        out[g] = statistics.median(ts)
        del fc
    return out


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--model", default="alexnet_exec")
    ap.add_argument("--batch-k", type=int, default=None)
    ap.add_argument("--nodes", type=int, default=8)
    ap.add_argument("--measure", action="store_true", help="time the constants on this GPU")
    ap.add_argument("--constants", default=None, help="constants file (key value lines)")
    ap.add_argument("--micro", type=int, default=2)
    args = ap.parse_args(argv)
    spec = builtin_model(args.model, args.batch_k)
    part = split(spec)
    mem = None
    if args.measure:
        c, info = measure_constants(spec)
        mem = info["hbm_free_bytes"]
        print(f"# {info}")
    elif args.constants:
        c = load_constants_file(args.constants)
    else:
        raise SystemExit("give --measure (on a GPU) or --constants FILE")
    print(format_constants_text(c, f"b200_{args.model}"), end="")
    print(f"{'split':>7} {'BSP img/s':>12} {'pipelined img/s':>16}")
    for n_fc in range(1, args.nodes):
        n_conv = args.nodes - n_fc
        if n_fc > n_conv:
            break
        bsp = stanza_throughput(part, n_conv, n_fc, c)
        pip = n_conv * spec.batch_k / pipelined_iter_time(part, n_conv, n_fc, c, args.micro)
        print(f"{n_conv:>4}:{n_fc:<2} {bsp:12.0f} {pip:16.0f}")
    if args.measure:
        gt = measure_fc_group_time(spec, groups=sorted({1, 2, 3, 7}))
        print("# FC worker time per iteration serving g CONV batches (fwd + bwd + update): " +
              ", ".join(f"g={g}: {t * 1e3:.3f} ms" for g, t in gt.items()))
        for n_fc in range(1, args.nodes):
            n_conv = args.nodes - n_fc
            if n_fc > n_conv:
                break
            g = -(-n_conv // n_fc)
            if g in gt:
                t = max(c.conv_time, gt[g])
                print(f"# measured-FC pipelined {n_conv}:{n_fc}: max(T_c, T_fc(g={g})) = "
                      f"{t * 1e3:.3f} ms -> {n_conv * spec.batch_k / t:.0f} img/s")
    a = assign_nodes(part, args.nodes, c, fc_memory_bytes=mem)
    p = assign_nodes(part, args.nodes, c, fc_memory_bytes=mem,
                     model=lambda *a_: pipelined_iter_time(*a_, micro=args.micro))
    print(f"assign_nodes (reference model): {a.n_conv}:{a.n_fc} {a.throughput:.0f} img/s")
    print(f"assign_nodes (pipelined model): {p.n_conv}:{p.n_fc} {p.throughput:.0f} img/s")
    return 0


if __name__ == "__main__":
    sys.exit(main())
