"""Times a few workloads under each terminal-path mode (dev tool): ipls_debug_term_mode
0 auto, 1 fused, 2 separate, 3 window sort; median of 8 sorts, CUDA events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2208_06902_b200 as ipls
from paper_2208_06902_b200 import datagen
names = sys.argv[1:] or ["C2", "P:twodups", "P:zipf"]
for name in names:
    a = datagen.paper_workload(name[2:], 100_000_000) if name.startswith("P:") else datagen.generate(name)
    kt = 0 if a.dtype == np.float64 else 1
    src = torch.from_numpy(a.view(np.int64)).cuda(); t = torch.empty_like(src)
    row = []
    for mode in (0, 1, 2):
        ipls.lib().ipls_debug_term_mode(mode)
        ts = []
        for r in range(8):
            t.copy_(src); torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); ipls.sort(t, k=1024, base_case=4096, key_type=kt, model=int(os.environ.get("MODEL", "0"))); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        row.append(f"mode{mode} {np.median(ts[2:]):.3f}")
    ipls.lib().ipls_debug_term_mode(0)
    print(name, " ".join(row), flush=True)
