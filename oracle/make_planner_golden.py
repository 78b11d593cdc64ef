"""Golden vectors for the node-assignment planner, from the REFERENCE itself.

    python oracle/make_planner_golden.py        # build container only

Imports the unmodified reference perf model (read-only,
/root/reference/pkg/src/stanza/perf_model.py) and records, for the profile
and executable models, window(n), stanza_iter_time / stanza_throughput over
every (n_conv, n_fc) split of up to 16 nodes, assign_nodes (with and without
an FC memory bound, and the Infeasible cases) under several constant sets,
and the constants text format.  paper_1812_10624_b200/planner.py restates
these formulas; tests/test_cpu_host.py checks it against this file.  Test
infrastructure only.
"""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden", "planner.json")
sys.path.insert(0, "/root/reference/pkg/src")

from stanza.model_partition import builtin_model, split  # noqa: E402
from stanza.perf_model import (Infeasible, PerfConstants, assign_nodes,  # noqa: E402
                               format_constants_text, stanza_iter_time,
                               stanza_throughput, v100_class_constants, window)

CONSTANTS = {
    "zero_10g": PerfConstants(bandwidth=10e9),
    "v100": v100_class_constants(),
    "b200_like": PerfConstants(bandwidth=900e9 * 8, conv_time=4.1e-3, fc_unit_time=0.35e-3,
                               ps_compute_time=4.6e-3),
    "fc_heavy": PerfConstants(bandwidth=100e9, conv_time=0.01, fc_unit_time=0.02,
                              ps_compute_time=0.02),
}
MODELS = ["alexnet", "vgg16", "vgg19", "inception_v3", "resnet152", "tiny_cnn"]


def main() -> None:
    out = {"window": {n: window(n) for n in range(1, 34)}, "constants": {}, "models": {}}
    for cname, c in CONSTANTS.items():
        out["constants"][cname] = {"bandwidth": c.bandwidth, "conv_time": c.conv_time,
                                   "fc_unit_time": c.fc_unit_time,
                                   "ps_compute_time": c.ps_compute_time,
                                   "text": format_constants_text(c, cname)}
    for mname in MODELS:
        part = split(builtin_model(mname))
        rec = {"conv_params": part.conv_params, "fc_params": part.fc_params,
               "boundary": part.boundary_activations, "batch_k": part.spec.batch_k,
               "iter_time": {}, "throughput": {}, "assign": {}}
        for cname, c in CONSTANTS.items():
            it, th, asg = {}, {}, {}
            for total in range(2, 17):
                for n_fc in range(1, total):
                    n_conv = total - n_fc
                    if n_fc > n_conv:
                        break
                    it[f"{n_conv},{n_fc}"] = stanza_iter_time(part, n_conv, n_fc, c)
                    th[f"{n_conv},{n_fc}"] = stanza_throughput(part, n_conv, n_fc, c)
                held = part.spec.batch_k * part.boundary_activations * 4
                for mem_name, mem in (("none", None), ("2x", 2.5 * held), ("tiny", 0.5 * held)):
                    try:
                        a = assign_nodes(part, total, c, fc_memory_bytes=mem)
                        asg[f"{total},{mem_name}"] = [a.n_conv, a.n_fc, a.throughput]
                    except Infeasible:
                        asg[f"{total},{mem_name}"] = None
            rec["iter_time"][cname], rec["throughput"][cname] = it, th
            rec["assign"][cname] = asg
        out["models"][mname] = rec
    with open(OUT, "w", encoding="utf-8") as fh:
        json.dump(out, fh, indent=0, sort_keys=True)
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
