"""Stall breakdown of one kernel from an ncu source-page CSV (ncu -i X --page source --csv)."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h) and r[0].startswith("0x")]
if len(data) > 2 and data[0][0] == data[len(data) // 2][0]:
    data = data[:len(data) // 2]
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = collections.Counter()
for r in data:
    for c in cols:
        try:
            tot[c] += int(r[h.index(c)] or 0)
        except ValueError:
            pass
s = sum(tot.values())
print("stall reasons (% of samples):", ", ".join(f"{c[6:]}={100*v/s:.1f}" for c, v in tot.most_common(10)))
iS = h.index("Source"); iW = h.index("Warp Stall Sampling (All Samples)"); iI = h.index("Instructions Executed")
top = sorted(data, key=lambda r: -int(r[iW] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]
for r in top:
    why = max(cols, key=lambda c: int(r[h.index(c)] or 0))
    print(f"  {int(r[iW]):6d} {why[6:]:14s} {r[iS].strip()[:64]:64s} exec={r[iI]}")
