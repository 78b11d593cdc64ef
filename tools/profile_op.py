"""Replay ONE tagged ABI call of the AlexNet co-located step inside an NVTX
range, so ncu can capture exactly that kernel:

    ncu --nvtx --nvtx-include "replay/" --set full -o prof python tools/profile_op.py conv3_wgrad

Tags are the engine's (conv<i>_fwd / _dgrad / _wgrad, fc<i>_...; i = layer
index in the spec).  Prints the call's mean CUDA-event time over 20 replays
(run once without ncu for the time)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from contextlib import contextmanager
import torch
from paper_1812_10624_b200 import _lib
from paper_1812_10624_b200.model_partition import builtin_model
from paper_1812_10624_b200.stanza_runtime import StanzaCluster

tag = sys.argv[1]
model = sys.argv[2] if len(sys.argv) > 2 else "alexnet_exec"
k = int(sys.argv[3]) if len(sys.argv) > 3 else 128
_lib.load()
spec = builtin_model(model, k)
cl = StanzaCluster(spec, n_conv=1, n_fc=1, batch_fn=None, lr=0.01, seed=3, device="cuda:0")
x = torch.randn(cl.x.shape, device="cuda:0")
y = torch.randint(0, 1000, cl.labels.shape, device="cuda:0", dtype=torch.int32)
captured = []


@contextmanager
def hook(name, args, flops=0.0, t=None, nbytes=0.0):
    if t == tag and not captured:
        captured.append((name, args, flops))
    yield


for _ in range(2):
    cl.step(x=x, labels=y)
_lib.PROFILE_HOOK = hook
cl.step(x=x, labels=y)
_lib.PROFILE_HOOK = None
torch.cuda.synchronize()
if not captured:
    raise SystemExit(f"tag {tag!r} not found")
name, args, flops = captured[0]
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
_lib.call(name, *args)
e0.record()
for _ in range(20):
    _lib.call(name, *args)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
if os.environ.get("STZ_DIAG"):
    lib = _lib.load()
    for cl_on in (1, 0):
        lib.stz_set_cluster(cl_on)
        for flags in (0, 1, 2, 4, 1 | 2, 1 | 4, 4 | 8):
            lib.stz_set_debug(flags)
            _lib.call(name, *args)
            e0.record()
            for _ in range(20):
                _lib.call(name, *args)
            e1.record()
            torch.cuda.synchronize()
            print(f"  cluster={cl_on} debug={flags}: {e0.elapsed_time(e1) / 20:.4f} ms", flush=True)
    lib.stz_set_debug(0)
    lib.stz_set_cluster(1)
if os.environ.get("STZ_SWEEP"):   # time every tile configuration (model-chosen splits)
    lib = _lib.load()
    for bn, cl in ((64, 1), (64, 2), (96, 1), (128, 1), (192, 1), (128, 2), (192, 2), (256, 2)):
        if lib.stz_set_tile(bn, cl, 0) != 0:
            continue
        _lib.call(name, *args)
        e0.record()
        for _ in range(20):
            _lib.call(name, *args)
        e1.record()
        torch.cuda.synchronize()
        print(f"  tile bn={bn} cl={cl}: {e0.elapsed_time(e1) / 20:.4f} ms", flush=True)
    lib.stz_set_tile(0, 0, 0)
    if os.environ.get("STZ_SWEEP") == "2":   # split counts per tile as well
        for bn, cl in ((64, 1), (96, 1), (128, 1), (192, 1), (128, 2), (192, 2), (256, 2)):
            row = []
            for sp in (4, 8, 16, 24, 32, 48, 64, 96, 128, 148, 192, 256):
                if lib.stz_set_tile(bn, cl, sp) != 0:
                    continue
                try:
                    _lib.call(name, *args)
                except Exception as exc:  # workspace too small for this split count
                    row.append(f"{sp}:-")
                    continue
                e0.record()
                for _ in range(20):
                    _lib.call(name, *args)
                e1.record()
                torch.cuda.synchronize()
                row.append(f"{sp}:{e0.elapsed_time(e1) / 20:.4f}")
            print(f"  tile bn={bn} cl={cl} splits->ms " + " ".join(row), flush=True)
        lib.stz_set_tile(0, 0, 0)
if os.environ.get("STZ_DEBUG"):   # capture a diagnostic variant (stz_set_debug flags)
    _lib.load().stz_set_debug(int(os.environ["STZ_DEBUG"]))
torch.cuda.nvtx.range_push("replay")
_lib.call(name, *args)
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print(f"{tag} {name}: {ms:.4f} ms, {flops / ms / 1e9:.1f} TFLOP/s algorithmic")
