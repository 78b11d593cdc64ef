"""Summarise the per-call timings a bench line carries (roofline.calls).

    python tools/bench_calls.py gpurun_out/bres.jsonl [more.jsonl ...]

Groups ABI calls by kind (conv fwd / dgrad / wgrad, BN fwd / bwd, ...) and
prints the total ms per kind, plus the median GB/s of the HBM-bound kinds.
"""
import json
import statistics
import sys


def kind(tag):
    last = tag.split(".")[-1]
    if last.startswith("bn"):
        return "bn_" + last.rsplit("_", 1)[-1]
    return last.rsplit("_", 1)[-1] if "_" in last else last


def main(paths):
    for path in paths:
        for line in open(path):
            d = json.loads(line)
            calls = d["roofline"].get("calls", {})
            fam, gbs = {}, {}
            for tag, c in calls.items():
                k = kind(tag)
                fam[k] = fam.get(k, 0.0) + c["total_ms"]
                if c.get("GBps"):
                    gbs.setdefault(k, []).append(c["GBps"])
            print(f"{path}: {d['config'].get('model')} {d['value']:.1f} {d['unit']} "
                  f"{d['ms_per_step']:.2f} ms/step (sum of call means {sum(fam.values()):.2f} ms)")
            for k, ms in sorted(fam.items(), key=lambda kv: -kv[1])[:12]:
                med = f"  median {statistics.median(gbs[k]):.0f} GB/s" if k in gbs else ""
                print(f"  {k:12s} {ms:7.2f} ms{med}")


if __name__ == "__main__":
    main(sys.argv[1:])
