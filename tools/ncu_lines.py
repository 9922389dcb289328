"""Aggregate ncu warp-stall samples per CUDA source line.

usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > s.csv
       python tools/ncu_lines.py s.csv [top]
"""
import csv
import sys
from collections import Counter


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    fname, hdr, agg, stall_cols = None, None, Counter(), {}
    per_reason = {}
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            stall_cols = {i: h for i, h in enumerate(hdr) if h.startswith("stall_")}
            continue
        if hdr is None or len(r) != len(hdr) or r[0] in ("", "Line No"):
            continue
        try:
            s = int(r[4])
        except ValueError:
            continue
        if s:
            key = (fname, r[0], r[1].strip()[:80])
            agg[key] += s
            pr = per_reason.setdefault(key, Counter())
            for i, h in stall_cols.items():
                try:
                    pr[h] += int(r[i])
                except ValueError:
                    pass
    tot = sum(agg.values())
    print("total samples", tot)
    for (f, ln, src), s in agg.most_common(top):
        reasons = ", ".join(f"{k[6:]}={v}" for k, v in per_reason[(f, ln, src)].most_common(2) if v)
        print(f"{100 * s / tot:5.1f}% {f}:{ln} {src}  [{reasons}]")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
