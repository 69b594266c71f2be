"""Turn the gpurun_out ncu artefacts into the committed profiles/ summaries.

    python tools/summarize_profiles.py <round-tag>

Writes profiles/<tag>_launches.csv (kernel, launches, avg/total device us, share; from the
bench command's `--metrics gpu__time_duration.sum` pass), profiles/<tag>_kernels.md (one
`--set full` capture per hot kernel: duration, DRAM bytes, tensor-pipe / issue activity,
top stall reasons) and profiles/dram_traffic.json (per-launch DRAM bytes, read by bench.py
for roofline.traffic).
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

SHORT = [("EpiGeluQuantT", "ffn1_i8"), ("EpiQKV", "qkv_i8"), ("EpiGeluQuant", "ffn1_i8"), ("EpiResLN", "ln_i8"), ("EpiF16Out", "f16out"),
         ("attention_kernel<0", "attention_i8"), ("attention_kernel<1", "attention_f16"),
         ("embed_kernel", "embed"), ("pooler_kernel", "pooler"), ("classifier_kernel", "classifier")]


def short(name):
    for k, v in SHORT:
        if k in name:
            if v == "ln_i8" and "<0," not in name:
                return "ln_f16"
            return v
    return name[:40]


def launches(tag):
    rows = list(csv.reader(open(os.path.join(OUT, "bench_launches.csv"))))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hdr]
    agg = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) != len(h):
            continue
        d = dict(zip(h, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = short(d["Kernel Name"])
        v = float(d["Metric Value"]) / (1000.0 if d["Metric Unit"] == "ns" else 1.0)
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    path = os.path.join(PROF, f"{tag}_launches.csv")
    with open(path, "w") as fh:
        fh.write("kernel,launches,avg_us,total_us,share\n")
        for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            fh.write(f"{k},{n},{t / n:.2f},{t:.1f},{t / tot:.4f}\n")
    return agg


def full(tag):
    txt = subprocess.run(["ncu", "-i", os.path.join(OUT, "prof_full.ncu-rep"), "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, units = rows[0], rows[1]
    g = lambda r, k: r[h.index(k)] if k in h else ""  # noqa: E731
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3}

    def num(r, k):  # bytes or microseconds, unit-aware
        v = g(r, k)
        return float(v) * scale.get(units[h.index(k)], 1.0) if v else 0.0
    lines = [f"# {tag}: ncu --set full, one launch per hot kernel (BERT-base FULLY_QUANT, batch 32 x 128)", "",
             "| kernel | grid | dur (us) | DRAM read+write (MB) | tensor pipe % | issue active % | warps active % | top stalls |",
             "|---|---|---|---|---|---|---|---|"]
    traffic = {}
    for r in rows[2:]:
        if not g(r, "Kernel Name"):
            continue
        name = short(g(r, "Kernel Name"))
        stalls = [(k[33:], float(g(r, k) or 0)) for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled")
                  and not k.endswith("not_issued")]
        tot = sum(v for _, v in stalls) or 1
        top = ", ".join(f"{k} {v / tot * 100:.0f}%" for k, v in sorted(stalls, key=lambda kv: -kv[1])[:3])
        rd = num(r, "dram__bytes_read.sum")
        wr = num(r, "dram__bytes_write.sum")
        traffic.setdefault(name, rd + wr)
        tensor = g(r, "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active") or \
            g(r, "sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active")
        lines.append(f"| {name} | {g(r, 'launch__grid_size')} | {num(r, 'gpu__time_duration.sum'):.1f} | "
                     f"{(rd + wr) / 1e6:.1f} | {tensor[:5]} | "
                     f"{g(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active')[:5]} | "
                     f"{g(r, 'sm__warps_active.avg.pct_of_peak_sustained_active')[:5]} | {top} |")
    with open(os.path.join(PROF, f"{tag}_kernels.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    with open(os.path.join(PROF, "dram_traffic.json"), "w") as fh:
        json.dump({"source": f"{tag} ncu --set full (dram__bytes_read.sum + dram__bytes_write.sum per launch)",
                   **{k: int(v) for k, v in traffic.items()}}, fh, indent=1)


if __name__ == "__main__":
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    os.makedirs(PROF, exist_ok=True)
    launches(tag)
    full(tag)
    print(open(os.path.join(PROF, f"{tag}_launches.csv")).read())
    print(open(os.path.join(PROF, f"{tag}_kernels.md")).read())
