"""Summarise an ncu launch list (gpu__time_duration.sum CSV): per-kernel launch count, time and share."""
import csv, collections, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
H = rows[hdr]; ix = {h: i for i, h in enumerate(H)}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hdr + 1:]:
    if len(r) < len(H) or r[ix["Metric Name"]] != "gpu__time_duration.sum": continue
    name = r[ix["Kernel Name"]]
    short = re.sub(r"\(.*", "", name)
    short = re.sub(r"^void ", "", short)[:90]
    ns = float(r[ix["Metric Value"]].replace(",", ""))
    scale = {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(r[ix["Metric Unit"]], 1)
    agg[short][0] += 1; agg[short][1] += ns * scale
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':92s} {'launches':>8s} {'total_ms':>10s} {'avg_us':>10s} {'share':>7s}")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:92s} {n:8d} {t/1e6:10.3f} {t/n/1e3:10.1f} {100*t/tot:6.1f}%")
