"""Summarise ncu outputs into profiles/: launch-list shares and key metrics."""
import csv, collections, json, sys

def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    h = rows[hi]; ik = h.index('Kernel Name'); iv = h.index('Metric Value')
    tot = collections.Counter(); cnt = collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= iv: continue
        name = r[ik].split('(')[0].replace('void ', '')
        try: v = float(r[iv].replace(',', ''))
        except ValueError: continue
        tot[name] += v; cnt[name] += 1
    T = sum(tot.values())
    return [{"kernel": k, "launches": cnt[k], "ms": round(v / 1e6, 3), "share": round(v / T, 4)}
            for k, v in tot.most_common()], T / 1e6

if __name__ == "__main__":
    rows, T = launches(sys.argv[1])
    print(json.dumps({"source": sys.argv[1], "total_ms": round(T, 3), "kernels": rows[:25]}, indent=1))
