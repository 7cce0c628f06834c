"""Achieved HBM bandwidth of the streaming kernels from an ncu metrics CSV
(gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum,
dram__throughput.avg.pct_of_peak_sustained_elapsed per launch), against the
measured copy bandwidth in MEASURED_PEAKS.json.

  python tools/stream_summary.py out.json source-note a.csv [b.csv ...]
"""
import collections
import csv
import json
import os
import sys

PEAK = 6546.2  # GB/s, MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth)


def per_launch(path):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    h = rows[0]
    ik, inm, iv, iid = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    d = collections.OrderedDict()
    for r in rows[1:]:
        e = d.setdefault(r[iid], {"kernel": r[ik].split("(")[0].replace("void ", "")})
        e[r[inm]] = float(r[iv].replace(",", ""))
    return list(d.values())


def main():
    out, note, paths = sys.argv[1], sys.argv[2], sys.argv[3:]
    peak = PEAK
    mp = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                      "MEASURED_PEAKS.json")
    if os.path.exists(mp):
        peak = json.load(open(mp)).get("hbm_gbs", PEAK)
    agg = collections.OrderedDict()
    for p in paths:
        for e in per_launch(p):
            if e["kernel"].startswith("at::"):  # torch fixture kernels (building A)
                continue
            a = agg.setdefault(e["kernel"], collections.Counter())
            a["launches"] += 1
            a["ns"] += e["gpu__time_duration.sum"]
            a["read"] += e["dram__bytes_read.sum"]
            a["write"] += e["dram__bytes_write.sum"]
            a["pct_sum"] += e.get("dram__throughput.avg.pct_of_peak_sustained_elapsed", 0.0)
    ks = []
    for k, a in agg.items():
        gbs = (a["read"] + a["write"]) / a["ns"]
        ks.append({"kernel": k, "launches": int(a["launches"]),
                   "us_per_launch": round(a["ns"] / a["launches"] / 1e3, 2),
                   "dram_read_MB_per_launch": round(a["read"] / a["launches"] / 1e6, 3),
                   "dram_write_MB_per_launch": round(a["write"] / a["launches"] / 1e6, 3),
                   "achieved_GBps": round(gbs, 1), "frac_of_hbm_peak": round(gbs / peak, 3),
                   "ncu_dram_pct_of_peak_mean": round(a["pct_sum"] / a["launches"], 1)})
    ks.sort(key=lambda x: -x["launches"] * x["us_per_launch"])
    json.dump({"source": note, "hbm_peak_GBps": peak, "kernels": ks}, open(out, "w"), indent=1)
    for x in ks:
        print(x)


if __name__ == "__main__":
    main()
