"""Print an ncu launch list (--metrics gpu__time_duration.sum --csv) as kernel, time (us)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]; ix = {k: i for i, k in enumerate(h)}
seq = [(r[ix["Kernel Name"]].split("(")[0].replace("void ", ""), float(r[ix["Metric Value"]]), r[ix["Metric Unit"]], r[ix["Grid Size"]])
       for r in rows[hi + 1:] if r and r[ix["Metric Name"]] == "gpu__time_duration.sum"]
skip = int(sys.argv[2]) if len(sys.argv) > 2 else len(seq) // 2
tot = 0.0
for name, v, u, g in seq[skip:]:
    us = v / 1000.0 if u == "ns" else (v if u == "us" else v * 1000.0)
    tot += us
    print(f"{us:10.1f} us  grid={g:>18s}  {name}")
print(f"{tot:10.1f} us  total")
