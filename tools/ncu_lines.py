"""Aggregate ncu cuda,sass source-view stall samples per CUDA source line."""
import csv
import subprocess
import sys
from collections import defaultdict


def main(rep, top=30, kern=None):
    filt = ["--kernel-name", f"regex:{kern}", "--launch-count", "1"] if kern else []
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"] + filt,
                         capture_output=True, text=True).stdout
    cur_file, hdr = None, None
    agg = defaultdict(lambda: [0.0, 0.0, ""])
    cur_line = None
    for r in csv.reader(txt.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name",):
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        if r[0] not in ("", "-"):
            cur_line = (cur_file, r[0], r[1])
        samp = r[4]
        inst = r[7]
        try:
            a = agg[(cur_line[0], cur_line[1])]
            a[0] += float(samp)
            a[1] += float(inst)
            a[2] = cur_line[2]
        except (ValueError, TypeError):
            pass
    tot = sum(v[0] for v in agg.values()) or 1
    print(f"total warp instructions {sum(v[1] for v in agg.values()):.0f}")
    for (f, ln), (s, n, src) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{s / tot * 100:5.1f}% inst={n:10.0f} {f[:14]}:{ln:>4} {src.strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30, sys.argv[3] if len(sys.argv) > 3 else None)
