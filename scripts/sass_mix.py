"""Summarise an ncu source-page CSV (SASS): executed instructions and stall samples per opcode."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
ex = collections.Counter(); st = collections.Counter(); tot_s = 0
for r in rows[2:]:
    if len(r) < len(hdr): continue
    op = r[ix["Source"]].strip().split()[0] if r[ix["Source"]].strip() else "?"
    if op.startswith("@"): op = r[ix["Source"]].strip().split()[1]
    op = op.split(".")[0]
    n = int(r[ix["Instructions Executed"]] or 0); s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    ex[op] += n; st[op] += s; tot_s += s
tot = sum(ex.values())
print(f"total warp-instructions {tot:,}  stall samples {tot_s:,}")
for op, n in ex.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"{op:10s} {n:14,d} {100*n/tot:6.2f}%   stall {100*st[op]/max(tot_s,1):6.2f}%")
