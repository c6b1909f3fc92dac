"""Per-source-line summary of an ncu capture (stall samples, warp-instructions).

    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_lines.py src.csv scl.cu [--frames F] [--phase name:a-b ...] [--top 40]

Lines of inlined helpers from other files are reported under their own file.
"""
from __future__ import annotations

import argparse
import csv


def _int(v):
    try:
        return int(v)
    except ValueError:
        return 0


def load(path):
    out = {}  # (file, line) -> [samples, inst, text]
    cur = None
    hdr = None
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].rsplit("/", 1)[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if r[0] in ("Function Name",) or hdr is None or r[0] == "":
            continue
        try:
            line = int(r[0])
        except ValueError:
            continue
        s = _int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        i = _int(r[hdr.index("Instructions Executed")])
        e = out.setdefault((cur, line), [0, 0, r[1]])
        e[0] += s
        e[1] += i
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("file")
    ap.add_argument("--frames", type=int, default=1)
    ap.add_argument("--phase", action="append", default=[])
    ap.add_argument("--top", type=int, default=40)
    a = ap.parse_args()
    d = load(a.csv)
    S = sum(v[0] for v in d.values()) or 1
    I = sum(v[1] for v in d.values()) or 1
    print(f"total stall samples {S}, warp-instructions {I} ({I / a.frames:.0f} per frame)")
    for ph in a.phase:
        name, rng = ph.split(":")
        lo, hi = (int(x) for x in rng.split("-"))
        s = sum(v[0] for (f, ln), v in d.items() if f == a.file and lo <= ln <= hi)
        i = sum(v[1] for (f, ln), v in d.items() if f == a.file and lo <= ln <= hi)
        print(f"  {name:24s} {100 * s / S:5.1f}% samp {100 * i / I:5.1f}% inst {i / a.frames:9.0f} inst/frame")
    others = {}
    for (f, ln), v in d.items():
        if f != a.file:
            o = others.setdefault(f, [0, 0])
            o[0] += v[0]
            o[1] += v[1]
    for f, v in others.items():
        print(f"  [{f}] {100 * v[0] / S:5.1f}% samp {100 * v[1] / I:5.1f}% inst")
    print()
    for (f, ln), v in sorted(d.items(), key=lambda kv: -kv[1][0])[: a.top]:
        print(f"{100 * v[0] / S:5.1f}% samp {100 * v[1] / I:5.1f}% inst  {f}:{ln:<5d} {v[2].strip()[:100]}")


if __name__ == "__main__":
    main()
