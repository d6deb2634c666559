"""Summarise one kernel of an .ncu-rep into the profiles/ JSON format.

usage: python tools/ncu_summary.py REP.ncu-rep OUT.json "command" "note"
"""
import csv, io, json, subprocess, sys

KEYS = [
    "Kernel Name", "dram__bytes.sum.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpc__cycles_elapsed.avg.per_second", "gpu__time_duration.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "launch__block_size",
    "launch__grid_size", "launch__occupancy_limit_registers", "launch__registers_per_thread",
    "lts__t_sector_hit_rate.pct", "sm__cycles_active.avg",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
]


def main():
    rep, out, cmd, note = sys.argv[1:5]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True,
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, vals = rows[0], rows[1], rows[2]
    res = {k: {"value": vals[head.index(k)], "unit": units[head.index(k)]}
           for k in KEYS if k in head}
    res["_command"], res["_note"] = cmd, note
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    for k in ("gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "dram__bytes.sum.per_second", "launch__registers_per_thread"):
        if k in res:
            print(k, res[k])


if __name__ == "__main__":
    main()
