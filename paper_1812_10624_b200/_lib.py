"""ctypes binding of the C ABI declared in include/stanza_b200.h.

There is no CPU fallback: if the library is missing or a call fails, this
module raises.  Device pointers come from torch tensors (PyTorch owns every
buffer); the stream is torch's current CUDA stream unless given.
"""

from __future__ import annotations

import ctypes
import os
import re

from .build import LIB_PATH

_HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       "include", "stanza_b200.h")

P = ctypes.c_void_p
I = ctypes.c_int
Z = ctypes.c_size_t
F = ctypes.c_float

# name -> (restype, argtypes); must match include/stanza_b200.h
SIGNATURES = {
    "stz_abi_version": (I, []),
    "stz_last_error": (ctypes.c_char_p, []),
    "stz_set_max_k_per_split": (I, [I]),
    "stz_set_tma": (I, [I]),
    "stz_set_cluster": (I, [I]),
    "stz_set_debug": (I, [I]),
    "stz_set_tile": (I, [I, I, I]),
    "stz_set_band": (I, [I]),
    "stz_set_fixup": (I, [I]),
    "stz_set_mh": (I, [I]),
    "stz_launch_count": (ctypes.c_ulonglong, []),
    "stz_conv2d_fwd": (I, [P, P, P, P, I, I, I, I, I, I, I, I, I, P, Z, P]),
    "stz_conv2d_bwd_data": (I, [P, P, P, P, I, I, I, I, I, I, I, I, P, Z, P]),
    "stz_conv2d_bwd_filter": (I, [P, P, P, P, I, I, I, I, I, I, I, I, P, Z, P]),
    "stz_fc_fwd": (I, [P, P, P, P, I, I, I, I, P, Z, P]),
    "stz_fc_bwd_data": (I, [P, P, P, P, I, I, I, P, Z, P]),
    "stz_fc_bwd_weight": (I, [P, P, P, P, I, I, I, P, Z, P]),
    "stz_maxpool2d_fwd": (I, [P, P, P, I, I, I, I, I, I, P]),
    "stz_maxpool2d_bwd": (I, [P, P, P, P, I, I, I, I, I, I, P]),
    "stz_relu_fwd": (I, [P, P, Z, P]),
    "stz_relu_bwd": (I, [P, P, P, Z, P]),
    "stz_softmax_ce": (I, [P, P, P, P, I, I, P]),
    "stz_sum_f32": (I, [P, Z, P, I, P]),
    "stz_sgd_momentum": (I, [P, P, P, Z, F, F, F, P]),
    "stz_vec_add": (I, [P, P, Z, P]),
    # split-plane hot path
    "stzx_pack_nchw": (I, [P, P, Z, I, I, I, I, I, P]),
    "stzx_unpack_nhwc": (I, [P, Z, P, I, I, I, I, I, P]),
    "stzx_pack_rows": (I, [P, P, Z, I, I, I, P]),
    "stzx_unpack_rows": (I, [P, Z, P, I, I, I, P]),
    "stzx_pack_conv_w": (I, [P, P, Z, P, Z, I, I, I, I, I, P]),
    "stzx_nhwc_to_flat": (I, [P, Z, P, Z, I, I, I, I, I, I, P]),
    "stzx_flat_to_nhwc": (I, [P, Z, P, Z, I, I, I, I, I, I, P]),
    "stzx_conv_fwd": (I, [P, Z, P, Z, P, P, Z, I, I, I, I, I, I, I, I, I, I, P, Z, P]),
    "stzx_conv_dgrad": (I, [P, Z, P, Z, P, Z, P, I, I, I, I, I, I, I, I, I, P, Z, P]),
    "stzx_conv_wgrad": (I, [P, Z, P, Z, P, P, I, I, I, I, I, I, I, I, I, I, I, P, Z, P]),
    "stzx_fc_fwd": (I, [P, Z, P, Z, P, P, Z, P, I, I, I, I, I, I, P, Z, P]),
    "stzx_fc_dgrad": (I, [P, Z, P, Z, P, Z, P, I, I, I, I, P, Z, P]),
    "stzx_fc_wgrad": (I, [P, Z, P, Z, P, P, I, I, I, I, I, I, P, Z, P]),
    "stzx_colsum": (I, [P, Z, I, I, I, P, I, P, Z, P]),
    "stzx_fc_wgrad_sgd": (I, [P, Z, P, Z, P, P, P, Z, P, P, P, P, I, I, I, I, I, I, F, F, F,
                              P, Z, P]),
    "stzx_maxpool_fwd": (I, [P, Z, P, Z, P, I, I, I, I, I, I, I, I, P]),
    "stzx_maxpool_bwd": (I, [P, Z, P, P, Z, P, I, I, I, I, I, I, I, I, P]),
    "stzx_relu_fwd": (I, [P, Z, P, Z, Z, P]),
    "stzx_relu_bwd": (I, [P, Z, P, P, Z, Z, P]),
    "stzx_softmax_ce": (I, [P, P, P, P, Z, I, I, I, P]),
    "stzx_pack_s2d": (I, [P, P, Z, I, I, I, I, I, I, I, I, I, P]),
    "stzx_pack_conv_w_s2d": (I, [P, P, Z, I, I, I, I, I, P]),
    "stzx_conv_fwd_s2d": (I, [P, Z, P, Z, P, P, Z, I, I, I, I, I, I, I, I, I, P, Z, P]),
    "stzx_conv_wgrad_s2d": (I, [P, Z, P, Z, P, P, I, I, I, I, I, I, I, I, I, I, P, Z, P]),
    "stzx_bn_fwd": (I, [P, Z, P, P, P, Z, P, Z, P, I, I, I, I, I, F, I, P, Z, P]),
    "stzx_bn_bwd": (I, [P, Z, P, P, Z, P, P, P, P, P, I, P, Z, I, I, I, I, I, P, Z, P]),
    "stzx_gap_fwd": (I, [P, Z, P, Z, I, I, I, P]),
    "stzx_gap_bwd": (I, [P, Z, P, Z, I, I, I, P]),
    "stzx_add": (I, [P, Z, P, Z, P, P, Z, Z, P]),
    # Inception-V3 kinds
    "stzx_pack_conv2_w": (I, [P, P, Z, P, Z, I, I, I, I, I, I, P]),
    "stzx_conv2_fwd": (I, [P, Z, P, Z, P, P, Z, I, I, I, I, I, I, I, I, I, I, I, I, P, Z, P]),
    "stzx_conv2_dgrad": (I, [P, Z, P, Z, P, Z, P, I, I, I, I, I, I, I, I, I, I, I, P, Z, P]),
    "stzx_conv2_wgrad": (I, [P, Z, P, Z, P, P, I, I, I, I, I, I, I, I, I, I, I, I, I, P, Z, P]),
    "stzx_avgpool_fwd": (I, [P, Z, P, Z, I, I, I, I, I, I, I, P]),
    "stzx_avgpool_bwd": (I, [P, Z, P, Z, I, I, I, I, I, I, I, P]),
    "stzx_copy_channels": (I, [P, Z, I, I, P, Z, I, I, Z, I, P, I, I, P]),
    "stzx_add_n": (I, [P, P, I, P, Z, Z, P]),
    "stzx_pack_conv_w_multi": (I, [P, I, P]),
    # exchange + update over NVLink peer memory
    "stz_ipc_handle": (I, [P, P, P]),
    "stz_ipc_open": (I, [P, P]),
    "stz_ipc_close": (I, [P]),
    "stz_set_peer_timeout_ms": (I, [ctypes.c_ulonglong]),
    "stz_peer_barrier": (I, [P, I, I, P]),
    "stz_peer_reduce_push": (I, [P, P, I, I, Z, P]),
    "stz_sgd_momentum_pack": (I, [P, P, P, Z, F, F, F, P, I, P]),
    "stz_allreduce_sgd": (I, [P, P, P, I, I, P, P, Z, F, F, F, P, I, P]),
    # CONV <-> FC link over peer memory
    "stz_link_begin": (I, [P, P]),
    "stz_link_put": (I, [P, Z, I, I, I, P, P, P, P, P, P]),
    "stz_link_get": (I, [P, I, I, P, Z, I, P, I, I, I, P]),
}


class ConvPack(ctypes.Structure):
    """stz_conv_pack (include/stanza_b200.h)."""
    _fields_ = [("w", P), ("wf", P), ("wd", P), ("psf", Z), ("psd", Z), ("O", I), ("C", I),
                ("kh", I), ("kw", I), ("C8", I), ("O8", I)]


MAX_CONV_PACK = 160


class PlaneRange(ctypes.Structure):
    """stz_plane_range (include/stanza_b200.h)."""
    _fields_ = [("off", Z), ("len", Z), ("planes", P), ("ps", Z), ("D", I), ("D8", I)]


IPC_HANDLE_BYTES = 64
PEER_FLAG_WORDS = 32
PEER_FLAG_STATUS = 17          # exchange block: != 0 after a barrier timed out
LINK_FLAG_WORDS = 256
LINK_SLOTS = 192
LINK_EPOCH = 240
LINK_STATUS = 241              # link block: kStatusLink | slot after a get timed out


def ptr_array(ptrs) -> ctypes.Array:
    """Host array of device pointers (keep the returned object alive for the call)."""
    return (P * len(ptrs))(*[int(p) for p in ptrs])


def range_array(ranges) -> ctypes.Array:
    """Host array of stz_plane_range from (off, len, planes_ptr, ps, D, D8) tuples."""
    return (PlaneRange * max(len(ranges), 1))(*[PlaneRange(*r) for r in ranges])


class StanzaCudaError(RuntimeError):
    """A C-ABI call returned a CUDA / launch failure."""


class StanzaLibraryMissing(ImportError):
    """libstz_b200.so is not built -- there is no fallback path."""


def header_symbols(path: str = _HEADER) -> list[str]:
    """Every function the public header declares."""
    with open(path, "r", encoding="utf-8") as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(stzx?_[a-z0-9_]+)\s*\(", text)))


_lib = None


def load(path: str | None = None):
    """Load (once) and type the library.  Raises StanzaLibraryMissing."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("STZ_LIB", LIB_PATH)
    if not os.path.exists(path):
        raise StanzaLibraryMissing(
            f"{path} not found; build it with `python -m paper_1812_10624_b200.build` "
            "(the CUDA path is the only path)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if os.environ.get("STZ_BAND"):          # experiments: shifted-window kernel selection
        lib.stz_set_band(int(os.environ["STZ_BAND"]))
    if os.environ.get("STZ_FIXUP"):         # experiments: split-K in-kernel fixup on / off
        lib.stz_set_fixup(int(os.environ["STZ_FIXUP"]))
    _lib = lib
    return lib


# Optional per-call hook (bench.py): callable(name, args) -> context manager
# that brackets the call with CUDA events on the launching stream.
PROFILE_HOOK = None

# STZ_SYNC_CHECK=1 (debugging): synchronize after every call made outside a
# CUDA-graph capture and raise on the first asynchronous fault, naming the call
_SYNC_CHECK = os.environ.get("STZ_SYNC_CHECK") == "1"


def _sync_check(name: str) -> int:
    import torch
    if torch.cuda.is_current_stream_capturing():
        return 0
    try:
        torch.cuda.current_stream().synchronize()
    except Exception as e:  # noqa: BLE001
        raise StanzaCudaError(f"{name}: asynchronous fault: {e}") from e
    return 0


# Measured GEMM tile choices: (name, tag, flops) -> (BN, CL) for stz_set_tile,
# filled by autotune_tiles(); calls not in it use the library's cost model.
TILE_TABLE: dict = {}

_TILE_CANDIDATES = ((64, 1), (96, 1), (128, 1), (192, 1), (128, 2), (192, 2), (256, 2))
# split-K counts tried per tile with STZ_AUTOTUNE_SPLITS=1 (0: the cost
# model's count for that tile; counts under the accumulation cap are raised
# to it by the library).  Off by default: the isolated-call wins did not
# carry into the step (AlexNet 36,953 vs 37,084, ResNet-50 2,495 vs 2,483
# images/s, profiles/r02/autotune_splits/)
_SPLIT_CANDIDATES = (0, 2, 4, 8, 16, 32, 64, 148) \
    if os.environ.get("STZ_AUTOTUNE_SPLITS", "0") == "1" else (0,)


def autotune_tiles(run_step, reps: int = 5, gain: float = 0.97) -> dict:
    """Time every GEMM call of one step under each tile shape and split-K
    count and keep the measured winner (BN, CL, splits) where it beats the
    cost model's pick by > 3%.

    ``run_step()`` runs one EAGER step (no graph replay: replays bypass this
    module and record nothing); its GEMM calls (every call carrying
    algorithmic FLOPs) are recorded with their arguments and replayed with
    CUDA events on the stream each call was launched on -- like a
    convolution autotuner, the replays overwrite that step's outputs, so run
    it before real training steps (or before the warm-up).  A forced tile
    keeps the accumulation cap per work item; splits = 0
    lets the library derive the split count for the forced width (the fp32
    summation order of the split-K partials follows the split count, within
    the GEMM tolerance of DESIGN.md 3.2).  Returns and installs the
    table; when the step recorded no GEMM the installed table is left
    unchanged."""
    global PROFILE_HOOK
    import torch
    from contextlib import contextmanager
    seen = {}

    @contextmanager
    def record(name, args, flops=0.0, tag=None, nbytes=0.0):
        if flops > 0 and (name, tag, flops) not in seen:
            seen[(name, tag, flops)] = args
        yield

    prev, PROFILE_HOOK = PROFILE_HOOK, record
    try:
        run_step()
    finally:
        PROFILE_HOOK = prev
    if not seen:
        return {}
    lib = load()
    torch.cuda.synchronize()

    def timed(name, args):
        fn = getattr(lib, name)
        st = args[-1]                          # every GEMM entry ends with its stream
        stream = torch.cuda.ExternalStream(int(st.value or 0)) if isinstance(
            st, ctypes.c_void_p) and st.value else torch.cuda.current_stream()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        if fn(*args) != 0:
            return None
        e0.record(stream)
        for _ in range(reps):
            fn(*args)
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1) / reps

    table = {}
    for key, args in seen.items():
        name = key[0]
        lib.stz_set_tile(0, 0, 0)
        base = timed(name, args)
        if base is None:
            continue
        best, best_ms = None, base * gain
        for bn, cl in _TILE_CANDIDATES:
            for sp in _SPLIT_CANDIDATES:
                if lib.stz_set_tile(bn, cl, sp) != 0:
                    break
                try:
                    ms = timed(name, args)
                except Exception:   # e.g. the call's workspace is too small for sp
                    ms = None
                if ms is not None and ms < best_ms:
                    best, best_ms = (bn, cl, sp), ms
        lib.stz_set_tile(0, 0, 0)
        if best is not None:
            table[key] = best
    TILE_TABLE.clear()
    TILE_TABLE.update(table)
    return table


def call(name: str, *args, flops: float = 0.0, tag: str | None = None,
         nbytes: float = 0.0) -> None:
    """Invoke an ABI function and raise on a non-zero status.  ``flops`` /
    ``nbytes`` / ``tag`` (algorithmic FLOPs or HBM bytes, layer label) are
    only seen by PROFILE_HOOK (and key TILE_TABLE)."""
    lib = load()
    tile = TILE_TABLE.get((name, tag, flops)) if TILE_TABLE else None
    if tile is not None:
        lib.stz_set_tile(tile[0], tile[1], tile[2] if len(tile) > 2 else 0)
    try:
        if PROFILE_HOOK is not None:
            with PROFILE_HOOK(name, args, flops, tag, nbytes=nbytes):
                rc = getattr(lib, name)(*args)
        else:
            rc = getattr(lib, name)(*args)
    finally:
        if tile is not None:
            lib.stz_set_tile(0, 0, 0)
    if rc == 0 and _SYNC_CHECK:
        rc = _sync_check(name)
    if rc != 0:
        msg = lib.stz_last_error().decode(errors="replace")
        if rc == 1:
            from .tensor_core import ShapeMismatch
            raise ShapeMismatch(f"{name}: {msg}")
        raise StanzaCudaError(f"{name} failed ({rc}): {msg}")
