"""Golden ledgers of the reference's own StanzaCluster (tests/golden/ledger.json).

Run in the build container (the only place /root/reference exists):

    python oracle/make_ledger_golden.py

For each (n_conv, n_fc) the unmodified reference trains tiny_cnn for two
iterations under a NetConfig, checkpoints, trains one more, and the script
stores what its ``transport.ledger`` reports: ``summary()``, the phase list
(label, logical elapsed, messages, payload bytes), ``rounds_for_op`` of both
allreduce ops and the sorted message multiset.  tests/test_ledger.py checks
that ``paper_1812_10624_b200.transport.record_iteration`` (the B200
runtime's ledger) reproduces them exactly.  Test infrastructure only.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden", "ledger.json")
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

from stanza.model_partition import tiny_cnn  # noqa: E402
from stanza.stanza_runtime import StanzaCluster  # noqa: E402
from stanza.transport import NetConfig  # noqa: E402
from trainers import make_batch_fn  # noqa: E402

SHAPES = [(1, 1), (2, 1), (3, 1), (3, 2), (4, 2), (5, 1), (6, 2), (7, 1), (8, 1), (5, 3)]
NET = dict(bandwidth=1e9, per_message_latency=2e-6)
CONV_TIME, FC_UNIT_TIME, SEED = 0.01, 0.002, 3


def run(nc, nf):
    spec = tiny_cnn()
    cl = StanzaCluster(spec, n_conv=nc, n_fc=nf, batch_fn=make_batch_fn(spec, 7), lr=0.05,
                       momentum=0.9, seed=SEED, net=NetConfig(**NET), conv_time=CONV_TIME,
                       fc_unit_time=FC_UNIT_TIME)
    cl.train(2)
    cl.checkpoint()
    res = cl.train(1)
    led = res.transport.ledger
    led.assert_conserved()
    msgs = sorted((m.phase, str(m.src), str(m.dst), m.tag.value, m.op or "",
                   -1 if m.round is None else m.round, m.payload_bytes) for m in led.messages)
    return {
        "n_conv": nc, "n_fc": nf,
        "summary": led.summary(),
        "phases": [[p.label, p.elapsed, p.messages, p.payload_bytes] for p in led.phases],
        "rounds_conv": led.rounds_for_op("conv_allreduce"),
        "rounds_fc": led.rounds_for_op("fc_allreduce"),
        "messages": msgs,
        "blob_len": len(next(iter(cl.replica_snapshots.values()))),
    }


def main():
    out = {"net": NET, "conv_time": CONV_TIME, "fc_unit_time": FC_UNIT_TIME, "seed": SEED,
           "model": "tiny_cnn", "batch_k": tiny_cnn().batch_k, "runs": {}}
    for nc, nf in SHAPES:
        out["runs"][f"{nc}x{nf}"] = run(nc, nf)
    with open(OUT, "w") as fh:
        json.dump(out, fh, indent=0, sort_keys=True, default=lambda o: float(o)
                  if isinstance(o, np.floating) else int(o))
    print(f"wrote {OUT}: {len(SHAPES)} ledgers")


if __name__ == "__main__":
    main()
