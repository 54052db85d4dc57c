"""Aggregate an ncu --metrics gpu__time_duration.sum CSV by kernel name: count, total ms, share."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r and r[0] == "ID": hdr = r; continue
    if hdr is None or len(r) != len(hdr): continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum": continue
    name = d["Kernel Name"].split("(")[0][:90]
    v = float(d["Metric Value"].replace(",", ""))
    unit = d.get("Metric Unit", "ns")
    ms = v / 1e6 if unit == "ns" else (v / 1e3 if unit in ("us", "usecond") else v)
    agg[name][0] += 1; agg[name][1] += ms
tot = sum(v[1] for v in agg.values())
print(f"total {tot:.2f} ms over {sum(v[0] for v in agg.values())} launches")
for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1])[:30]:
    print(f"{ms:10.2f} ms {100*ms/tot:5.1f}% n={n:6d} avg={1e3*ms/n:8.1f}us  {k}")
