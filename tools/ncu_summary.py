"""Key ncu --set full metrics of every kernel in a report (time, instructions, issue,
pipes, smem wavefronts/conflicts, stall reasons per issue, DRAM bytes).

    python tools/ncu_summary.py gpurun_out/prof_x.ncu-rep
"""
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time_us"),
    ("smsp__inst_executed.sum", "warp_inst"),
    ("sm__cycles_active.avg", "sm_active_cyc"),
    ("sm__cycles_elapsed.avg", "sm_elapsed_cyc"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
    ("smsp__warps_active.avg.per_cycle_active", "warps/smsp"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu%"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma%"),
    ("sm__inst_executed_pipe_xu.sum.pct_of_peak_sustained_active", "xu%"),
    ("sm__inst_executed_pipe_lsu.sum.pct_of_peak_sustained_active", "lsu%"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem_wf%"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "bank_conf"),
    ("sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active", "tensor%"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
]


def main(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        name = v[h.index("Kernel Name")][:90]
        print(f"== {name}")
        out = []
        for k, lab in KEYS:
            if k in h:
                out.append(f"{lab}={v[h.index(k)]}{'' if u[h.index(k)] in ('', '%', 'inst', 'cycle') else u[h.index(k)]}")
        print("   " + "  ".join(out))
        st = [(n.split("issue_stalled_")[1].split("_per_issue")[0], float(v[i]))
              for i, n in enumerate(h) if n.startswith("smsp__average_warps_issue_stalled_") and
              n.endswith("_per_issue_active.ratio") and v[i] not in ("", "n/a")]
        st = sorted(st, key=lambda x: -x[1])[:9]
        print("   stalls/issue: " + "  ".join(f"{a}={b:.2f}" for a, b in st))


if __name__ == "__main__":
    main(sys.argv[1])
