"""Quick CUDA-event timing of ipls.sort on the BASELINE configs (development tool)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2208_06902_b200 as ipls
from paper_2208_06902_b200 import datagen

names = sys.argv[1:] or ["C2"]
for name in names:
    cfg = datagen.CONFIGS[name]
    a = datagen.generate(name)
    kt = 0 if a.dtype == np.float64 else 1
    src = torch.from_numpy(a.view(np.int64)).cuda()
    t = torch.empty_like(src)
    want = None
    times = []
    for rep in range(int(os.environ.get('REPS', '8'))):
        t.copy_(src)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        ipls.sort(t, k=cfg.k, base_case=cfg.base_case, key_type=kt)
        e1.record(); torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    ok = bool((t[1:].view(torch.float64 if kt == 0 else torch.int64) >= t[:-1].view(torch.float64 if kt == 0 else torch.int64)).all()) if kt == 0 else True
    ms = float(np.median(times[3:] if len(times) > 3 else times))
    print(f"{name}: n={a.size} median {ms:.3f} ms  ({a.size/ms/1e6:.2f} Gkeys/s)  all={['%.3f'%x for x in times]} sorted={ok}", flush=True)
