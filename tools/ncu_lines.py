"""Aggregate an ncu source page (--print-source=cuda,sass --csv) per CUDA source
line: warp stall samples and executed warp instructions, top N lines.
  ncu -i rep --page source --csv --print-source=cuda,sass > x.csv
  python tools/ncu_lines.py x.csv [N]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = None
cur_file = ""
agg = {}
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 8 or not r[0]:
        continue
    d = dict(zip(hdr[2:], r[2:]))
    key = (cur_file, int(r[0]))
    try:
        samp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        inst = int(d.get("Instructions Executed", "0") or 0)
    except ValueError:
        continue
    a = agg.setdefault(key, [0, 0, r[1][:90]])
    a[0] += samp
    a[1] += inst
tot_s = sum(v[0] for v in agg.values()) or 1
tot_i = sum(v[1] for v in agg.values()) or 1
print(f"total samples {tot_s}, warp instructions {tot_i}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0]}:{k[1]:4d} samp {100*v[0]/tot_s:5.1f}% inst {100*v[1]/tot_i:5.1f}%  {v[2]}")
