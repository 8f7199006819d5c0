"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per kernel the launch count, mean time and share of all launches, and the
two frame kernels' share of a frame.

    python tools/ncu_launches.py gpurun_out/launches.csv
"""

import collections
import csv
import sys


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if r]
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    kn, mn, mv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    t = collections.defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > mv and r[mn] == "gpu__time_duration.sum":
            name = r[kn].split("(")[0].replace("<unnamed>::", "").strip()
            t[name].append(float(r[mv].replace(",", "")) / 1e3)  # ns -> us
    total = sum(sum(v) for v in t.values())
    frame = sum(sum(v) for k, v in t.items() if "fused_" in k)
    for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1])):
        line = f"{k[:48]:48s} launches={len(v):4d} mean={sum(v) / len(v):9.2f} us  share_of_all={100 * sum(v) / total:5.1f}%"
        if "fused_" in k:
            line += f"  share_of_frame={100 * sum(v) / frame:5.1f}%"
        print(line)


if __name__ == "__main__":
    main()
