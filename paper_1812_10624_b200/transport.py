"""Traffic accounting of the layer-separated step, with the reference's surface.

The reference moves every tensor through a simulated in-process network and
reads its ``TrafficLedger`` (transport.py:157-262): phase log, payload bytes
per message tag, per-node wire bytes, collective rounds, the logical clock.
Its callers (tests/test_stanza_runtime.py:133-200, harness.py:517-555) read
``StanzaResult.transport.ledger``.  On B200 the data moves through device
kernels (peer-memory link and exchange, or NCCL), so this module keeps the
*accounting* surface: ``DeviceTransport.ledger`` logs, per iteration, the
messages the reference protocol defines for the same (n_conv, n_fc) --
activations + labels per CONV worker, boundary gradients per CONV worker,
the recursive-doubling / surplus allreduce rounds of each role group
(collectives.py:1-157) -- and advances the logical clock with the
reference's bottleneck formula for the given ``NetConfig``.  What the GPUs
actually did (device milliseconds per phase, bytes over NVLink) sits next
to it on ``PhaseRecord.device_ms`` and ``DeviceTransport.device_bytes``.

Names and values follow the reference so its callers run unchanged:
``Role``, ``NodeId``, ``Tag`` (values "Activations", ...), ``NetConfig``,
``PhaseRecord(label, elapsed, messages, payload_bytes)``,
``TrafficLedger.{phases, tag_payload_bytes, tag_messages, bytes_for_tags,
total_payload_bytes, rounds_for_op, assert_conserved, summary, export_csv,
export_summary_json}``.
"""

from __future__ import annotations

import csv
import json
import random
from dataclasses import dataclass
from enum import Enum
from typing import Iterable

HEADER_BYTES = 32          # wire header per message (reference transport.py:42)
BYTES_PER_ELEMENT = 4


class Role(Enum):
    CONV_WORKER = "conv"
    FC_WORKER = "fc"
    PS_SERVER = "server"
    PS_WORKER = "worker"
    CONTROLLER = "controller"


@dataclass(frozen=True)
class NodeId:
    role: Role
    index: int

    def __str__(self):
        return f"{self.role.value}{self.index}"


def _order(n: NodeId):
    return (n.role.value, n.index)


class Tag(Enum):
    ACTIVATIONS = "Activations"
    BOUNDARY_GRADS = "BoundaryGrads"
    GRAD_PUSH = "GradPush"
    PARAM_PULL = "ParamPull"
    ALLREDUCE_CHUNK = "AllreduceChunk"
    CHECKPOINT = "Checkpoint"
    CONTROL = "Control"


class Timeout(TimeoutError):
    """A wait for a peer exceeded its deadline (reference transport.Timeout)."""


@dataclass
class NetConfig:
    """Logical network of the reference's clock (bits/s per node per
    direction); only the ledger's logical clock uses it."""
    bandwidth: float = 10e9
    per_message_latency: float = 0.0
    full_duplex: bool = True
    default_timeout: float = 30.0


@dataclass
class PhaseRecord:
    label: str
    elapsed: float               # logical seconds (reference clock)
    messages: int
    payload_bytes: int
    device_ms: float | None = None   # CUDA-event time of the phase (time_phases=True)


@dataclass
class MessageRecord:
    phase: str
    phase_index: int
    link_seq: int
    src: NodeId
    dst: NodeId
    tag: Tag
    op: str | None
    round: int | None
    payload_bytes: int


def phase_elapsed(transfers: Iterable[tuple], net: NetConfig) -> float:
    """Busiest direction of the busiest node at ``net.bandwidth`` plus one
    latency when anything moved (reference transport.py:265-289)."""
    sent: dict = {}
    recv: dict = {}
    count = 0
    for src, dst, nbytes in transfers:
        sent[src] = sent.get(src, 0) + nbytes
        recv[dst] = recv.get(dst, 0) + nbytes
        count += 1
    if not count:
        return 0.0
    load = max((max(sent.get(n, 0), recv.get(n, 0)) if net.full_duplex
                else sent.get(n, 0) + recv.get(n, 0)) for n in set(sent) | set(recv))
    return load * 8.0 / net.bandwidth + net.per_message_latency


class TrafficLedger:
    """Message / phase log with the reference TrafficLedger's queries."""

    def __init__(self):
        self.node_sent: dict = {}
        self.node_received: dict = {}
        self.link_bytes: dict = {}
        self.tag_payload_bytes = {t: 0 for t in Tag}
        self.tag_messages = {t: 0 for t in Tag}
        self.logical_clock = 0.0
        self.phases: list[PhaseRecord] = []
        self.messages: list[MessageRecord] = []
        self._seq: dict = {}

    def observe(self, src: NodeId, dst: NodeId, tag: Tag, payload: int, phase: str,
                phase_index: int, op: str | None = None, rnd: int | None = None) -> None:
        wire = payload + HEADER_BYTES
        self.node_sent[src] = self.node_sent.get(src, 0) + wire
        self.node_received[dst] = self.node_received.get(dst, 0) + wire
        self.link_bytes[(src, dst)] = self.link_bytes.get((src, dst), 0) + wire
        self.tag_payload_bytes[tag] += payload
        self.tag_messages[tag] += 1
        key = (src, dst, tag)
        seq = self._seq.get(key, 0)
        self._seq[key] = seq + 1
        self.messages.append(MessageRecord(phase, phase_index, seq, src, dst, tag, op, rnd,
                                           payload))

    @property
    def total_sent(self) -> int:
        return sum(self.node_sent.values())

    @property
    def total_received(self) -> int:
        return sum(self.node_received.values())

    def bytes_for_tags(self, tags: Iterable[Tag]) -> int:
        return sum(self.tag_payload_bytes[t] for t in tags)

    @property
    def total_payload_bytes(self) -> int:
        return self.bytes_for_tags(Tag)

    def rounds_for_op(self, op: str) -> list[int]:
        return sorted({m.round for m in self.messages if m.op == op and m.round is not None})

    def assert_conserved(self) -> None:
        if self.total_sent != self.total_received:
            raise AssertionError(f"byte conservation violated: {self.total_sent} != "
                                 f"{self.total_received}")

    def export_csv(self, path) -> None:
        """phase, src, dst, tag, bytes, elapsed_s per message, deterministic order."""
        elapsed = {i: p.elapsed for i, p in enumerate(self.phases)}
        rows = sorted(self.messages, key=lambda m: (m.phase_index, _order(m.src), _order(m.dst),
                                                    m.tag.value, m.link_seq))
        with open(path, "w", newline="", encoding="utf-8") as fh:
            w = csv.writer(fh)
            w.writerow(["phase", "src", "dst", "tag", "bytes", "elapsed_s"])
            for m in rows:
                w.writerow([m.phase, str(m.src), str(m.dst), m.tag.value, m.payload_bytes,
                            repr(elapsed.get(m.phase_index, 0.0))])

    def summary(self) -> dict:
        nodes = sorted(set(self.node_sent) | set(self.node_received), key=_order)
        return {
            "logical_clock_s": self.logical_clock,
            "total_wire_bytes_sent": self.total_sent,
            "total_wire_bytes_received": self.total_received,
            "total_payload_bytes": self.total_payload_bytes,
            "per_node": {str(n): {"sent": self.node_sent.get(n, 0),
                                  "received": self.node_received.get(n, 0)} for n in nodes},
            "per_tag_payload_bytes": {t.value: self.tag_payload_bytes[t] for t in Tag
                                      if self.tag_messages[t]},
            "phases": len(self.phases),
            "messages": len(self.messages),
        }

    def export_summary_json(self, path) -> None:
        with open(path, "w", encoding="utf-8") as fh:
            json.dump(self.summary(), fh, indent=2, sort_keys=True)
            fh.write("\n")


# -- the reference's allreduce schedule (collectives.py:1-157), for accounting --

def round_count(n: int) -> int:
    if n < 1:
        raise ValueError("group size must be positive")
    if n == 1:
        return 0
    m = n.bit_length() - 1
    return m if n == 1 << m else m + 2


def allreduce_messages(members: list, seed: int):
    """(src, dst, round) of every message of one recursive-doubling
    allreduce over ``members`` (group order = rank); non-power-of-two groups
    pre-send surplus members to seeded-random core donors (round 0) and
    return the result after the doubling rounds (round m + 1)."""
    n = len(members)
    if n == 1:
        return []
    m = n.bit_length() - 1
    out = []
    core, donors = list(members), {}
    if n != 1 << m:
        rng = random.Random(seed)
        surplus_idx = sorted(rng.sample(range(n), n - (1 << m)))
        core = [x for i, x in enumerate(members) if i not in set(surplus_idx)]
        picks = rng.sample(range(1 << m), len(surplus_idx))
        donors = {members[s]: core[d] for s, d in zip(surplus_idx, picks)}
        out += [(s, d, 0) for s, d in donors.items()]
    for r in range(m):
        for rank, node in enumerate(core):
            out.append((node, core[rank ^ (1 << r)], r + 1))
    out += [(d, s, m + 1) for s, d in donors.items()]
    return out


def allreduce_seed(seed: int, iteration: int) -> int:
    """reference stanza_runtime.py:59-61"""
    return seed * 1_000_003 + iteration


class DeviceTransport:
    """``StanzaResult.transport``: the reference-shaped ledger of the
    protocol's messages plus what the devices measured."""

    def __init__(self, net: NetConfig | None = None):
        self.net = net or NetConfig()
        self.ledger = TrafficLedger()
        self.device_bytes: dict = {}      # link -> bytes the kernels moved over NVLink
        self._phase = None
        self._transfers: list = []
        self._payload = 0
        self._messages = 0

    # phases (reference SimTransport.begin_phase / end_phase / advance_compute)
    def begin_phase(self, label: str) -> None:
        self._phase, self._transfers, self._payload, self._messages = label, [], 0, 0

    def send(self, src: NodeId, dst: NodeId, tag: Tag, payload: int, op: str | None = None,
             rnd: int | None = None) -> None:
        self.ledger.observe(src, dst, tag, payload, self._phase, len(self.ledger.phases), op, rnd)
        self._transfers.append((src, dst, payload))
        self._payload += payload
        self._messages += 1

    def end_phase(self) -> PhaseRecord:
        el = phase_elapsed(self._transfers, self.net)
        self.ledger.logical_clock += el
        rec = PhaseRecord(self._phase, el, self._messages, self._payload)
        self.ledger.phases.append(rec)
        self._phase = None
        return rec

    def advance_compute(self, seconds: float, label: str) -> PhaseRecord:
        if seconds < 0:
            raise ValueError("compute time must be nonnegative")
        self.ledger.logical_clock += seconds
        rec = PhaseRecord(label, seconds, 0, 0)
        self.ledger.phases.append(rec)
        return rec

    # convenience for callers that read the ledger fields off the transport
    @property
    def phases(self):
        return self.ledger.phases

    @property
    def tag_payload_bytes(self):
        return self.ledger.tag_payload_bytes

    @property
    def tag_messages(self):
        return self.ledger.tag_messages


def record_iteration(tr: DeviceTransport, *, conv_ids, fc_ids, conv_to_fc, k: int, a: int,
                     conv_params: int, fc_params: int, seed: int, iteration: int,
                     conv_time: float, fc_unit_time: float, max_group: int) -> list:
    """Log one iteration of the reference schedule (stanza_runtime.py:352-375)
    on ``tr``; returns the six PhaseRecords in order."""
    recs = [tr.advance_compute(conv_time, "conv_compute")]
    tr.begin_phase("activations")
    for i, c in enumerate(conv_ids):
        dst = fc_ids[conv_to_fc[i]]
        tr.send(c, dst, Tag.ACTIVATIONS, k * a * BYTES_PER_ELEMENT, op="activations")
        tr.send(c, dst, Tag.CONTROL, k * BYTES_PER_ELEMENT, op="labels")
    recs.append(tr.end_phase())
    recs.append(tr.advance_compute(max_group * fc_unit_time, "fc_compute"))
    tr.begin_phase("boundary")
    for j, f in enumerate(fc_ids):
        for i, g in enumerate(conv_to_fc):
            if g == j:
                tr.send(f, conv_ids[i], Tag.BOUNDARY_GRADS, k * a * BYTES_PER_ELEMENT,
                        op="boundary")
    recs.append(tr.end_phase())
    tr.begin_phase("exchange")
    ar = allreduce_seed(seed, iteration)
    groups = [(conv_ids, conv_params, "conv_allreduce")]
    if len(fc_ids) > 1:
        groups.append((fc_ids, fc_params, "fc_allreduce"))
    for members, count, op in groups:
        for src, dst, rnd in allreduce_messages(list(members), ar):
            tr.send(src, dst, Tag.ALLREDUCE_CHUNK, count * BYTES_PER_ELEMENT, op=op, rnd=rnd)
    recs.append(tr.end_phase())
    tr.begin_phase("update")
    recs.append(tr.end_phase())
    return recs
