"""BASELINE.md §4 results table (dev tool, on the GPU box): per BASELINE config C1-C5 the GPU
sort time (median of REPS, L2 flushed before each), keys/s, the whole-sort roofline fraction
(48 B/key model at C2-C5, 32 B/key at C1, against 8 TB/s and against the measured copy peak),
bit-exactness against the CPU oracle's output, the oracle's single-thread time, torch.sort
(context) and, with --dram DIR, the ncu DRAM bytes of one sort (DIR/dram_<cfg>.csv from
`ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --csv python tools/one_sort.py CFG 1`).
Writes profiles/r02_results.json and prints the markdown rows."""
import csv, io, json, math, os, statistics, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_2208_06902_b200 as ipls
from paper_2208_06902_b200 import datagen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
reps = int(os.environ.get("REPS", "10"))
dram_dir = sys.argv[sys.argv.index("--dram") + 1] if "--dram" in sys.argv else None
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
cpu = "unknown"
try:
    for line in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines():
        if line.startswith("Model name"):
            cpu = line.split(":", 1)[1].strip()
except Exception:
    pass
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
rows = []
for name in ["C1", "C2", "C3", "C4", "C5"]:
    cfg = datagen.CONFIGS[name]
    a = datagen.generate(name)
    n = a.size
    kt = 0 if a.dtype == np.float64 else 1
    src = torch.from_numpy(a.view(np.int64)).cuda()
    t = torch.empty_like(src)
    ts = []
    for r in range(reps + 3):
        t.copy_(src)
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ipls.sort(t, k=cfg.k, base_case=cfg.base_case, key_type=kt)
        e1.record()
        torch.cuda.synchronize()
        if r >= 3:
            ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    got = t.cpu().numpy()
    tt = []
    for _ in range(3):
        flush.fill_(2)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); torch.sort(src.view(torch.float64) if kt == 0 else src); e1.record()
        torch.cuda.synchronize()
        tt.append(e0.elapsed_time(e1))
    oms = []
    for _ in range(3 if name == "C1" else 1):
        w = a.copy()
        t0 = time.perf_counter()
        assert oracle.sort(w, k=cfg.k, base_case=cfg.base_case).status == 0
        oms.append(1e3 * (time.perf_counter() - t0))
    exact = got.tobytes() == w.view(np.int64).tobytes()
    Ls = math.ceil(math.log(math.ceil(n / cfg.base_case), cfg.k))
    mb = 2 * 8 * n * (Ls + 1)
    row = {"cfg": name, "n": n, "ms": round(ms, 3), "keys_per_s": n / (ms / 1e3),
           "model_bytes_per_key": 16 * (Ls + 1), "frac_8TBps": round(mb / 8e12 / (ms / 1e3), 4),
           "frac_measured_copy": round(mb / (peak * 1e9) / (ms / 1e3), 4),
           "bit_exact_vs_oracle": exact, "oracle_ms_1core": round(statistics.median(oms), 1),
           "torch_sort_ms": round(statistics.median(tt), 3), "host_cpu": cpu,
           "nproc": os.cpu_count(), "all_ms": [round(x, 3) for x in ts]}
    if dram_dir:
        p = os.path.join(dram_dir, f"dram_{name}.csv")
        if os.path.exists(p):
            txt = open(p).read()
            txt = txt[txt.index('"ID"'):] if '"ID"' in txt else txt
            tot = 0.0
            for rr in csv.DictReader(io.StringIO(txt)):
                if rr.get("Metric Name", "").startswith("dram__bytes"):
                    v = float(rr["Metric Value"].replace(",", ""))
                    u = rr.get("Metric Unit", "byte")
                    tot += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            row["ncu_dram_bytes"] = tot
            row["ncu_dram_bytes_per_key"] = round(tot / n, 2)
    rows.append(row)
    print(json.dumps(row), flush=True)
    del src, t
    torch.cuda.empty_cache()
with open(os.path.join(ROOT, "profiles", "r02_results.json"), "w") as f:
    json.dump({"rows": rows, "reps": reps, "peak_hbm_gbs": peak}, f, indent=1)
for r in rows:
    print(f"| {r['cfg']} | {r['ms']} | {r['keys_per_s']/1e9:.2f} G | {r['frac_8TBps']} | "
          f"{r['frac_measured_copy']} | {r.get('ncu_dram_bytes_per_key', '-')} B/key | "
          f"{'yes' if r['bit_exact_vs_oracle'] else 'NO'} | {r['oracle_ms_1core']} | "
          f"{r['host_cpu']} / {r['nproc']} |")
