"""Per-CUDA-line profile of one kernel from an ncu report (dev tool).

usage: python tools/srcprof.py REPORT.ncu-rep KERNEL_REGEX [TOP]
Prints the source lines with the most warp-stall samples and executed warp instructions
(ncu --page source --print-source cuda,sass; needs -lineinfo)."""
import csv, io, os, subprocess, sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + kre, "--launch-count", "1", "--launch-skip", os.environ.get("SKIP","0")], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = []
fname = ""
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and r and r[0] not in ("", "File Path", "Function Name") and len(r) >= 8:
        try:
            agg.append((fname, int(r[0]), r[1].strip(), int(r[4] or 0), int(r[7] or 0)))
        except ValueError:
            pass
ts = sum(a[3] for a in agg) or 1
ti = sum(a[4] for a in agg) or 1
print(f"total stall samples {ts}, warp instructions {ti}")
for a in sorted(agg, key=lambda a: -a[3])[:top]:
    print(f"{100*a[3]/ts:5.1f}% smp {100*a[4]/ti:5.1f}% ins  {a[0]}:{a[1]:<5d} {a[2][:90]}")
