"""Aggregate an ncu source page (--page source --csv --print-source cuda,sass)
per CUDA source line: warp instructions executed and stall samples, the
heaviest lines first.  The file/line context comes from the inlined source
the SASS rows follow.

    ncu -i rep --page source --csv --print-source cuda,sass -k regex:NAME > x.csv
    python tools/ncu_lines.py x.csv [top]
"""
import csv
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    inst = defaultdict(int)
    samp = defaultdict(int)
    thr = defaultdict(int)
    text = {}
    cur_file = None
    cur = None
    total_i = total_s = 0
    with open(path, newline="") as f:
        for row in csv.reader(f):
            if not row:
                continue
            if row[0] == "File Path":
                cur_file = row[1].split("/")[-1]
                continue
            if row[0] in ("Function Name", "Line No", "Kernel Name"):
                continue
            # per-line aggregate rows: "Line No", "Source", "-", "-", metrics...
            if row[0] != "" and len(row) > 8 and row[2] == "-":
                k = (cur_file, int(row[0]))
                text[k] = row[1].strip()[:90]
                try:
                    i = int(row[7] or 0)
                    s_ = int(row[4] or 0)
                    t = int(row[8] or 0)
                except ValueError:
                    continue
                inst[k] += i
                samp[k] += s_
                thr[k] += t
                total_i += i
                total_s += s_
    print(f"total warp instructions {total_i}, stall samples {total_s}")
    for k in sorted(inst, key=lambda k: -inst[k])[:top]:
        print(f"{inst[k] / total_i:6.1%} inst {samp[k] / max(total_s, 1):6.1%} samp  thr/inst {thr[k] / max(inst[k], 1):5.1f}"
              f"  {k[0]}:{k[1]}  {text.get(k, '')}")


if __name__ == "__main__":
    main()
