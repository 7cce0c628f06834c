"""Summarise an ncu --set full report of zgemm3m launches: the longest launch's
DMMA pipe utilisation, FP64 tensor ops per cycle, DRAM traffic, occupancy and
warp-stall samples.  python tools/ncu_full_summary.py report.ncu-rep out.json "source note"
"""
import csv
import io
import json
import subprocess
import sys


def num(s):
    try:
        return float(s.replace(",", ""))
    except (ValueError, AttributeError):
        return None


def main():
    rep, out, note = sys.argv[1], sys.argv[2], sys.argv[3]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, data = rows[0], rows[2:]
    it = h.index("gpu__time_duration.sum")
    r = max(data, key=lambda x: num(x[it]) or 0.0)
    g = {c: r[i] for i, c in enumerate(h)}
    pre = "smsp__pcsamp_warps_issue_stalled_"
    stalls = {c[len(pre):]: num(g[c]) for c in h
              if c.startswith(pre) and not c.endswith("_not_issued") and num(g[c])}
    stalls = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:10])
    s = {
        "source": note,
        "launches_in_report": len(data),
        "kernel": g["Kernel Name"], "grid": g["Grid Size"], "block": g["Block Size"],
        "registers_per_thread": num(g["launch__registers_per_thread"]),
        "time": num(g["gpu__time_duration.sum"]),
        "dmma_pipe_pct_of_peak_active":
            num(g["sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"]),
        "fp64_tensor_ops_per_cycle_per_sm":
            num(g["sm__ops_path_tensor_src_fp64.avg.per_cycle_elapsed"]),
        "fp64_tensor_ops_peak_per_cycle_per_sm": 128,
        "dram_read": num(g["dram__bytes_read.sum"]),
        "dram_write": num(g["dram__bytes_write.sum"]),
        "warps_active_pct": num(g["sm__warps_active.avg.pct_of_peak_sustained_active"]),
        "stall_samples_top": stalls,
        "units": {"dram_read": rows[1][h.index("dram__bytes_read.sum")],
                  "dram_write": rows[1][h.index("dram__bytes_write.sum")], "time": rows[1][it]},
    }
    json.dump(s, open(out, "w"), indent=1)
    print(json.dumps(s, indent=1))


if __name__ == "__main__":
    main()
