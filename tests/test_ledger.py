"""The runtime's traffic ledger against the reference's own
(tests/golden/ledger.json, made by oracle/make_ledger_golden.py from the
unmodified reference): for every (n_conv, n_fc) the B200 runtime logs, per
iteration, exactly the messages, phase records, logical clock, allreduce
rounds and checkpoint payload the reference's transport.ledger reports
(reference transport.py:157-262; pinned by its tests/test_stanza_runtime.py
:158-200).  Host-only: transport.record_iteration is what
StanzaCluster._record calls each step."""

import json
import os

import pytest

from paper_1812_10624_b200 import model_partition as mp
from paper_1812_10624_b200.checkpointing import stzc_blob_len
from paper_1812_10624_b200.roles import plan_groups
from paper_1812_10624_b200.tensor_core import param_shapes
from paper_1812_10624_b200.transport import (DeviceTransport, NetConfig, NodeId, Role, Tag,
                                             allreduce_messages, record_iteration, round_count)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "ledger.json")))


def _replay(nc, nf):
    """The ledger a StanzaCluster(tiny_cnn, nc, nf) logs over train(2),
    checkpoint(), train(1) -- the golden scenario."""
    spec = mp.tiny_cnn()
    part = mp.split(spec)
    tr = DeviceTransport(NetConfig(**GOLD["net"]))
    conv_ids = [NodeId(Role.CONV_WORKER, i) for i in range(nc)]
    fc_ids = [NodeId(Role.FC_WORKER, j) for j in range(nf)]
    c2f = plan_groups(nc, nf)
    kw = dict(conv_ids=conv_ids, fc_ids=fc_ids, conv_to_fc=c2f, k=spec.batch_k,
              a=part.boundary_activations, conv_params=part.conv_params,
              fc_params=part.fc_params, seed=GOLD["seed"], conv_time=GOLD["conv_time"],
              fc_unit_time=GOLD["fc_unit_time"], max_group=max(c2f.count(j) for j in range(nf)))
    for it in range(2):
        record_iteration(tr, iteration=it, **kw)
    import random
    holder = random.Random((GOLD["seed"] << 32) ^ 2).randrange(nc)
    fc_shapes = [param_shapes(l) for l in spec.layers[part.split_index:]]
    tr.begin_phase("checkpoint")
    tr.send(fc_ids[0], conv_ids[holder], Tag.CHECKPOINT, stzc_blob_len(fc_shapes),
            op="checkpoint")
    tr.end_phase()
    record_iteration(tr, iteration=2, **kw)
    return tr.ledger, stzc_blob_len(fc_shapes)


@pytest.mark.parametrize("case", sorted(GOLD["runs"]))
def test_ledger_matches_reference(case):
    g = GOLD["runs"][case]
    led, blob_len = _replay(g["n_conv"], g["n_fc"])
    assert blob_len == g["blob_len"]
    assert [[p.label, p.messages, p.payload_bytes] for p in led.phases] == \
        [[p[0], p[2], p[3]] for p in g["phases"]]
    for p, q in zip(led.phases, g["phases"]):
        assert p.elapsed == pytest.approx(q[1], rel=1e-12, abs=1e-15)
    assert led.rounds_for_op("conv_allreduce") == g["rounds_conv"]
    assert led.rounds_for_op("fc_allreduce") == g["rounds_fc"]
    msgs = sorted([m.phase, str(m.src), str(m.dst), m.tag.value, m.op or "",
                   -1 if m.round is None else m.round, m.payload_bytes] for m in led.messages)
    assert msgs == [list(m) for m in g["messages"]]
    s = led.summary()
    ref = g["summary"]
    assert s["logical_clock_s"] == pytest.approx(ref["logical_clock_s"], rel=1e-12)
    for key in ("total_wire_bytes_sent", "total_wire_bytes_received", "total_payload_bytes",
                "per_node", "per_tag_payload_bytes", "phases", "messages"):
        assert s[key] == ref[key], key
    led.assert_conserved()


def test_tag_values_and_queries():
    led, _ = _replay(3, 1)
    spec = mp.tiny_cnn()
    k, a = spec.batch_k, 256
    assert Tag.ACTIVATIONS.value == "Activations"
    assert led.tag_payload_bytes[Tag.ACTIVATIONS] == 3 * 3 * a * k * 4
    assert led.tag_payload_bytes[Tag.CONTROL] == 3 * 3 * k * 4
    assert led.bytes_for_tags([Tag.ACTIVATIONS, Tag.BOUNDARY_GRADS]) == 2 * 3 * 3 * a * k * 4
    assert led.total_payload_bytes == sum(led.tag_payload_bytes.values())


@pytest.mark.parametrize("n", range(1, 10))
def test_allreduce_schedule_rounds(n):
    """collectives.py:1-157: log2 n rounds for powers of two, floor(log2 n)
    + 2 otherwise; every member sends once per doubling round; surplus
    members send once and receive once."""
    members = list(range(n))
    msgs = allreduce_messages(members, seed=123)
    rounds = sorted({r for _, _, r in msgs})
    assert len(rounds) == round_count(n)
    sent = {m: 0 for m in members}
    recv = {m: 0 for m in members}
    for s, d, _ in msgs:
        sent[s] += 1
        recv[d] += 1
    assert sent == recv


def test_export_csv_and_summary_json(tmp_path):
    led, _ = _replay(4, 2)
    led.export_csv(tmp_path / "t.csv")
    led.export_summary_json(tmp_path / "s.json")
    rows = (tmp_path / "t.csv").read_text().splitlines()
    assert rows[0] == "phase,src,dst,tag,bytes,elapsed_s"
    assert len(rows) == 1 + len(led.messages)
    assert json.loads((tmp_path / "s.json").read_text())["messages"] == len(led.messages)
