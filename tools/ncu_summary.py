"""Summarize an ncu --set full report into profiles/*.json.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/ncu_rXX_vY_summary.json "label" [--headline]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "smsp__inst_executed.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__maximum_warps_per_active_cycle_pct",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(rep, out, label, headline=False):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    kernels = []
    for r in rows[2:]:
        d = {"kernel": r[idx["Kernel Name"]]}
        for k in KEYS:
            if k in idx:
                d[k] = r[idx[k]] + (" " + units[idx[k]] if units[idx[k]] else "")
        kernels.append(d)
    json.dump({"report": rep, "label": label, "kernels": kernels}, open(out, "w"), indent=1)
    if headline:
        k = [x for x in kernels if "k_exhaustive_pfx<12" in x["kernel"]][0]

        def b(v):
            num, unit = v.split()
            return float(num) * SCALE[unit]

        traffic = b(k["dram__bytes_read.sum"]) + b(k["dram__bytes_write.sum"])
        json.dump({"kernel": k["kernel"], "dram_bytes_per_launch": traffic,
                   "issue_active_pct": float(k["sm__inst_issued.avg.pct_of_peak_sustained_active"].split()[0]),
                   "fp64_pipe_active_pct": float(
                       k["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"].split()[0]),
                   "alu_pipe_active_pct": float(
                       k["sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"].split()[0]),
                   "warp_exec_efficiency": float(
                       k["smsp__thread_inst_executed_per_inst_executed.ratio"].split()[0]) / 32,
                   "achieved_occupancy_pct": float(
                       k["sm__warps_active.avg.pct_of_peak_sustained_active"].split()[0]),
                   "theoretical_occupancy_pct": float(k["sm__maximum_warps_per_active_cycle_pct"].split()[0]),
                   "warp_instructions_per_launch": float(k["smsp__inst_executed.sum"].split()[0]),
                   "source": out}, open("profiles/ncu_headline.json", "w"), indent=1)
    print(json.dumps(kernels, indent=1)[:3000])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], "--headline" in sys.argv)
