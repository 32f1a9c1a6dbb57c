"""Per-launch DRAM traffic of each kernel family from an ncu --set full report -> JSON for
profiles/ (read by bench.py for roofline.traffic).  usage: traffic_json.py REPORT SOURCE_NOTE"""
import csv, io, json, re, subprocess, sys
from collections import defaultdict

# the library's profile scope "scatter" brackets a level's two scatter kernels (stable, then
# terminal): their traffic is summed per level
FAMILY = {"k_scatter_stable": "scatter", "k_scatter_term": "scatter", "k_term_fused": "scatter",
          "k_base_warp": "base_warp",
          "k_classify_scan": "classify_scan", "k_base_sort": "base_sort",
          "k_gather_fit": "gather_fit", "k_fit_small": "fit_small", "k_emit": "emit",
          "k_fill": "fill"}


def main(rep, note):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, data = rows[0], rows[1], rows[2:]
    iK = h.index("Kernel Name")
    iR, iW = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    per = defaultdict(list)
    for r in data:
        fam = next((v for k, v in FAMILY.items() if k in r[iK]), None)
        if fam is None:
            continue
        rd = float(r[iR]) * scale[units[iR]]
        wr = float(r[iW]) * scale[units[iW]]
        if ("k_scatter_term" in r[iK] or "k_term_fused" in r[iK]) and per[fam]:
            per[fam][-1][0] += int(rd)
            per[fam][-1][1] += int(wr)
        else:
            per[fam].append([int(rd), int(wr)])
    res = {"source": note, "kernels": {}}
    for fam, l in per.items():
        res["kernels"][fam] = {"dram_bytes_per_launch": int(sum(a + b for a, b in l) / len(l)),
                               "launches": len(l), "per_launch": l}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
