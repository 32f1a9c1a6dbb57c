"""Per-phase clock breakdown of k_scatter (dev tool): builds a timing variant of libipls.so
(-DIPLS_SCATTER_TIMING) under /tmp, sorts a BASELINE config, prints cycles per tile per phase."""
import ctypes, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2208_06902_b200 import build as B
so = os.path.join(ROOT, "tools", "libipls_timing.so")
if not os.path.exists(so):
    subprocess.check_call([B.nvcc(), *B.NVCC_FLAGS, "-DIPLS_SCATTER_TIMING", "-o", so, *B.SOURCES])
import numpy as np, torch
import paper_2208_06902_b200 as ipls
ipls._LIB_PATH = so
from paper_2208_06902_b200 import datagen
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = datagen.CONFIGS[name]
a = datagen.generate(name)
if os.environ.get("ORDER") == "sorted":  # presorted input (K3, dense tiles)
    a = np.sort(a)
kt = 0 if a.dtype == np.float64 else 1
src = torch.from_numpy(a.view(np.int64)).cuda()
t = torch.empty_like(src)
lib = ipls.lib()
ph = (ctypes.c_ulonglong * 32)()
for rep in range(2):
    t.copy_(src)
    torch.cuda.synchronize()
    lib.ipls_debug_scatter_phases(ph, 1)
    ipls.sort(t, k=cfg.k, base_case=cfg.base_case, key_type=kt)
    torch.cuda.synchronize()
lib.ipls_debug_scatter_phases(ph, 1)
tr = ipls.sort_trace(src.clone(), k=cfg.k, base_case=cfg.base_case, key_type=kt) if False else None
ns, nt = max(ph[28], 1), max(ph[29], 1)
print(f"stable scatter: {ph[28]} tiles; cycles per tile (thread 0): ranks {ph[0]/ns:.0f} offsets {ph[1]/ns:.0f} "
      f"place {ph[2]/ns:.0f} writeout {ph[3]/ns:.0f}")
print(f"terminal scatter: {ph[29]} tiles; cycles per tile (thread 0): slots {ph[4]/nt:.0f} offsets {ph[5]/nt:.0f} "
      f"place {ph[6]/nt:.0f} writeout {ph[7]/nt:.0f}")
print(f"large-sample fit (1 CTA, cycles): gather {ph[16]} sort {ph[17]} fmcd {ph[18]}")
print("fit cycle sums over all CTAs of the last sort (x1e6): gather", ph[8] / 1e6, "sort", ph[9] / 1e6,
      "fmcd", ph[10] / 1e6)
print("all phase counters:", [int(x) for x in ph])
