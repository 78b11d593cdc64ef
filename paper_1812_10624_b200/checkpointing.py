"""Training-state snapshots in the reference's byte formats.

``TrainState`` (iteration, params, velocities) is what ``StanzaCluster.state``
returns -- nested fp32 numpy arrays in reference layouts -- so the
reference's ``param_digest`` / ``max_param_dev`` apply unchanged.  The STZT
parameter blob (tensor_core.py:395-460) and the STZC state blob
(checkpointing.py:20-65 of the reference) are re-implemented here so a
digest computed on B200 output equals one computed by the reference.
"""

from __future__ import annotations

import hashlib
import struct
from dataclasses import dataclass

import numpy as np

from .tensor_core import CorruptCheckpoint

_STZT, _STZT_VERSION = b"STZT", 1
_STZC, _STZC_VERSION = b"STZC", 1
_STZC_HEAD = "<HQQQ"


@dataclass
class TrainState:
    """Everything needed to resume at an iteration boundary."""
    iteration: int
    params: list
    velocities: list

    def copy(self) -> "TrainState":
        return TrainState(self.iteration,
                          [[t.copy() for t in layer] for layer in self.params],
                          [[t.copy() for t in layer] for layer in self.velocities])


def serialize_params(params) -> bytes:
    """STZT: magic, u32 version, u32 tensor count, u32 layer count, u32 per
    layer tensor counts, then per tensor u32 ndim, u32 dims, raw LE fp32."""
    sizes = [len(layer) for layer in params]
    flat = [np.ascontiguousarray(t, dtype="<f4") for layer in params for t in layer]
    parts = [_STZT, struct.pack("<III", _STZT_VERSION, len(flat), len(sizes)),
             struct.pack(f"<{len(sizes)}I", *sizes)]
    for a in flat:
        parts.append(struct.pack(f"<I{a.ndim}I", a.ndim, *a.shape))
        parts.append(a.tobytes())
    return b"".join(parts)


def deserialize_params(blob: bytes) -> list:
    """Inverse of serialize_params; CorruptCheckpoint on malformed data."""
    try:
        if blob[:4] != _STZT:
            raise CorruptCheckpoint("bad magic")
        version, count, n_layers = struct.unpack_from("<III", blob, 4)
        if version != _STZT_VERSION:
            raise CorruptCheckpoint(f"unsupported version {version}")
        off = 16
        sizes = struct.unpack_from(f"<{n_layers}I", blob, off)
        off += 4 * n_layers
        if sum(sizes) != count:
            raise CorruptCheckpoint("tensor count disagrees with layer table")
        tensors = []
        for _ in range(count):
            (ndim,) = struct.unpack_from("<I", blob, off)
            shape = struct.unpack_from(f"<{ndim}I", blob, off + 4)
            off += 4 + 4 * ndim
            size = int(np.prod(shape)) if ndim else 1
            if off + 4 * size > len(blob):
                raise CorruptCheckpoint("truncated tensor data")
            tensors.append(np.frombuffer(blob, "<f4", size, off).reshape(shape)
                           .astype(np.float32))
            off += 4 * size
        if off != len(blob):
            raise CorruptCheckpoint(f"{len(blob) - off} trailing bytes")
    except struct.error as exc:
        raise CorruptCheckpoint(str(exc)) from exc
    out, i = [], 0
    for n in sizes:
        out.append(tensors[i:i + n])
        i += n
    return out


def param_digest(params) -> str:
    """sha256 of the STZT blob (order and bytes exact)."""
    return hashlib.sha256(serialize_params(params)).hexdigest()


def state_to_bytes(state: TrainState) -> bytes:
    p = serialize_params(state.params)
    v = serialize_params(state.velocities)
    return _STZC + struct.pack(_STZC_HEAD, _STZC_VERSION, state.iteration, len(p), len(v)) + p + v


def stzc_blob_len(shapes) -> int:
    """Byte length of state_to_bytes for a block whose tensors have the
    nested ``shapes`` [layer][tensor] -- without building the blob."""
    stzt = 16 + 4 * len(shapes) + sum(4 + 4 * len(s) + 4 * int(np.prod(s, dtype=np.int64))
                                      for row in shapes for s in row)
    return 4 + struct.calcsize(_STZC_HEAD) + 2 * stzt


def state_from_bytes(blob: bytes) -> TrainState:
    head = 4 + struct.calcsize(_STZC_HEAD)
    if len(blob) < head or blob[:4] != _STZC:
        raise CorruptCheckpoint("not a training-state snapshot")
    version, iteration, p_len, v_len = struct.unpack(_STZC_HEAD, blob[4:head])
    if version != _STZC_VERSION:
        raise CorruptCheckpoint(f"unsupported snapshot version {version}")
    if len(blob) != head + p_len + v_len:
        raise CorruptCheckpoint("snapshot length does not match header")
    params = deserialize_params(blob[head:head + p_len])
    vel = deserialize_params(blob[head + p_len:])
    if [len(l) for l in params] != [len(l) for l in vel]:
        raise CorruptCheckpoint("parameter/velocity structure mismatch")
    return TrainState(iteration, params, vel)
