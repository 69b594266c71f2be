"""Summarise an ncu --page source --csv --print-source sass dump: hottest SASS per kernel."""
import csv
import subprocess
import sys


def main(rep, top=25, kernel_filter=""):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    kernels, cur, hdr = [], None, None
    for row in csv.reader(txt.splitlines()):
        if not row:
            continue
        if row[0] == "Kernel Name":
            cur = {"name": row[1], "rows": []}
            kernels.append(cur)
            hdr = None
            continue
        if row[0] == "Address":
            hdr = row
            continue
        if cur is not None and hdr:
            cur["rows"].append(dict(zip(hdr, row)))
    for k in kernels:
        if kernel_filter not in k["name"]:
            continue
        rows = k["rows"]
        tot = sum(int(r.get("Warp Stall Sampling (All Samples)", 0) or 0) for r in rows)
        inst = sum(int(r.get("Instructions Executed", 0) or 0) for r in rows)
        print(f"=== {k['name'][:110]}\n    samples={tot} warp-instructions={inst}")
        hot = sorted(rows, key=lambda r: -int(r.get("Warp Stall Sampling (All Samples)", 0) or 0))[:top]
        for r in hot:
            print(f"  {int(r['Warp Stall Sampling (All Samples)']):6d} {r['Address'][-5:]} {r['Source'].strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25, sys.argv[3] if len(sys.argv) > 3 else "")
