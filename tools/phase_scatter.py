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
tiles = sum((int(n) + 8191) // 8192 for n in [a.size]) * 2  # approx: 2 levels over all keys
print("scatter cycles per tile (thread 0):", " ".join(f"{i}:{ph[i] / tiles:.0f}" for i in range(7)))
nt = max(ph[15], 1)
print(f"unstable scatter: {ph[15]} tiles; cycles per tile (thread 0): zero {ph[11]/nt:.0f} count {ph[12]/nt:.0f} "
      f"scan {ph[13]/nt:.0f} place {ph[14]/nt:.0f} writeout {ph[7]/nt:.0f}")
print(f"large-sample fit (1 CTA, cycles): gather {ph[16]} sort {ph[17]} fmcd {ph[18]}")
print("small-sample fit sort sub-phases (cycles summed):", [ph[i] for i in range(22, 27)])
print(f"small-sample fit (cycles summed over CTAs): gather {ph[19]} sort {ph[20]} fmcd {ph[21]}")
print("fit cycle sums over all CTAs of the last sort (x1e6): gather", ph[8] / 1e6, "sort", ph[9] / 1e6,
      "fmcd", ph[10] / 1e6)
