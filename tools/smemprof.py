"""Per-CUDA-line shared-memory wavefronts (actual vs ideal) of one kernel launch from an ncu
report (dev tool).  usage: python tools/smemprof.py REPORT KERNEL_REGEX [TOP]  (SKIP=n)"""
import csv, io, os, subprocess, sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + kre, "--launch-count", "1", "--launch-skip",
                      os.environ.get("SKIP", "0")], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, agg = "", None, []
for r in rows:
    if len(r) == 2 and r[0] == "File Name":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and r and len(r) == len(hdr):
        iw, ii = hdr.index("L1 Wavefronts Shared"), hdr.index("L1 Wavefronts Shared Ideal")
        try:
            w, wi, ln = int(r[iw] or 0), int(r[ii] or 0), int(r[0])
        except ValueError:
            continue
        if w:
            agg.append((w, wi, fname, ln, r[1].strip()))
tw = sum(a[0] for a in agg) or 1
print(f"total shared wavefronts {tw}, ideal {sum(a[1] for a in agg)}")
for w, wi, f, ln, src in sorted(agg, reverse=True)[:top]:
    print(f"{100*w/tw:5.1f}%  {w:>11d} (ideal {wi:>11d})  {f}:{ln:<5} {src[:80]}")
