"""DRAM traffic of the GEMM launches of one filter application, from an ncu
metrics pass, against their algorithmic bytes:
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none -k regex:zgemm --csv --log-file gpurun_out/zt.csv \
      python tools/one_app.py 4 lu 1
  python tools/zgemm_traffic.py gpurun_out/zt.csv 4 > profiles/ncu_zgemm_traffic_cfg4_r02.json
The JSON records the sha256 of the library's sources the capture ran on;
bench.py uses the figure only when that digest is the benched sources'."""
import collections
import csv
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1605_08771_b200 import configs as CF  # noqa: E402


from paper_1605_08771_b200._lib import source_digest  # noqa: E402


def trailing_algorithmic_bytes(N, nodes, kb):
    """Trailing updates of one LU per node, outer blocks of kb columns: C read +
    written once (32 B per complex entry), L21 / U12 and their sum planes read
    once (24 B per entry), the sum planes written and their sources read by zsum."""
    c = ops = 0.0
    for k0 in range(0, N, kb):
        rest = N - k0 - kb
        if rest <= 0:
            break
        c += 32.0 * rest * rest
        ops += 24.0 * 2 * rest * kb
    return nodes * c, nodes * ops


def main(path, cfg):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ik, im, iv, iu, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("ID")
    per = collections.defaultdict(lambda: collections.defaultdict(float))
    ids = collections.defaultdict(set)
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3,
             "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}
    for r in rows[hi + 1:]:
        if len(r) <= iv:
            continue
        name = r[ik].split("(")[0].replace("void ", "").replace("fl::", "")
        try:
            v = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
        except ValueError:
            continue
        per[name][r[im]] += v
        ids[name].add(r[iid])
    c = CF.CONFIGS[cfg]
    N = (c.n + 63) // 64 * 64
    kb = 1024 if N >= 12288 else 256
    calg, oalg = trailing_algorithmic_bytes(N, c.n_c, kb)
    out = {"source": f"{path}: ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum of one "
                     f"cfg{cfg} LU filter application (node chunks on one stream)",
           "src_sha256": source_digest(), "cfg": cfg, "kernels": {}}
    for name, m in per.items():
        n = len(ids[name])
        rd, wr = m.get("dram__bytes_read.sum", 0.0), m.get("dram__bytes_write.sum", 0.0)
        out["kernels"][name] = {"launches": n, "ms": round(m.get("gpu__time_duration.sum", 0.0), 2),
                                "dram_read_bytes": rd, "dram_write_bytes": wr,
                                "dram_bytes_per_launch": (rd + wr) / max(n, 1)}
    tr = next((k for k in out["kernels"] if k.startswith("zgemm3s_kernel")), None)
    if tr:
        t = out["kernels"][tr]
        out["trailing_update"] = {
            "kernel": tr, "launches": t["launches"],
            "dram_bytes_per_launch": t["dram_bytes_per_launch"],
            "dram_bytes": t["dram_read_bytes"] + t["dram_write_bytes"],
            "algorithmic_bytes": calg + oalg,
            "algorithmic_note": "C read and written once (32 B per complex entry) + L21, U12 and their sum planes read once",
            "traffic_over_algorithmic": round((t["dram_read_bytes"] + t["dram_write_bytes"]) / (calg + oalg), 3),
            "write_over_algorithmic_c_write": round(t["dram_write_bytes"] / (calg / 2), 3)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))
