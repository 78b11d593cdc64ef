"""Group an ncu launch list (--metrics gpu__time_duration.sum --csv) by
kernel family and print the serialised device time per family.

    python tools/launch_summary.py gpurun_out/prof/step_launches.csv
"""
import csv
import re
import sys
from collections import defaultdict


def family(name):
    name = re.sub(r"\(.*", "", name)              # drop the argument list
    name = re.sub(r"^void ", "", name)
    base = re.sub(r"<.*", "", name).replace("stz::", "")
    return base + ("<" + name.split("<", 1)[1] if "<" in name and base == "tgemm_kernel" else "")


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        f = family(r[ki])
        tot[f] += float(r[vi].replace(",", ""))
        cnt[f] += 1
    unit = "ns"
    all_t = sum(tot.values())
    print(f"{len(rows) - 1} launches, {all_t / 1e3:.1f} us serialised")
    for f, t in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{t / 1e3:9.1f} us {100 * t / all_t:5.1f}%  n={cnt[f]:4d}  {f[:110]}")


if __name__ == "__main__":
    main(sys.argv[1])
