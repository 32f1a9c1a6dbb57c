"""CUDA-event timing of ipls.sort on BASELINE configs + per-kernel library profile (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2208_06902_b200 as ipls
from paper_2208_06902_b200 import datagen
if os.environ.get("IPLS_LIB"):  # A/B a variant build
    ipls._LIB_PATH = os.path.abspath(os.environ["IPLS_LIB"])

names = sys.argv[1:] or ["C2"]
reps = int(os.environ.get("REPS", "8"))
for name in names:
    if name.startswith("P:"):  # a paper workload (datagen.PAPER_WORKLOADS) at 1e8, C2's k and B
        cfg = datagen.CONFIGS["C2"]
        a = datagen.paper_workload(name[2:], int(os.environ.get("N", "100000000")))
    else:
        cfg = datagen.CONFIGS[name]
        a = datagen.generate(name)
    order = os.environ.get("ORDER", "")  # presorted inputs: sorted, reverse, or G runs
    if order == "sorted":
        a = np.sort(a)
    elif order == "reverse":
        a = np.sort(a)[::-1].copy()
    elif order.startswith("runs"):  # G sorted runs of a random split (what dist_sort's local
        G = int(order[4:] or 8)       # sorts receive is G bucket-ordered runs)
        a = np.concatenate([np.sort(x) for x in np.array_split(a, G)])
    kt = 0 if a.dtype == np.float64 else 1
    src = torch.from_numpy(a.view(np.int64)).cuda()
    t = torch.empty_like(src)
    times = []
    for rep in range(reps):
        t.copy_(src)
        torch.cuda.synchronize()
        if rep == reps - 1:
            ipls.profile_reset(); ipls.profile_enable(True)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        ipls.sort(t, k=cfg.k, base_case=cfg.base_case, key_type=kt,
                  model=int(os.environ.get("MODEL", "0")))
        e1.record(); torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    ipls.profile_enable(False)
    prof = ipls.profile_read()
    ref = torch.sort(src.view(torch.float64) if kt == 0 else src)[0].view(torch.int64)
    ok = bool(torch.equal(ref, t))
    ms = float(np.median(times[2:] if len(times) > 2 else times))
    print(f"{name}: n={a.size} median {ms:.3f} ms ({a.size/ms/1e6:.2f} Gkeys/s) sorted={ok} "
          f"all={['%.2f' % x for x in times]}", flush=True)
    print("   " + "  ".join(f"{k}:{v[1]:.3f}ms/{v[0]}" + (f"({v[2]/(v[1]/1e3)/1e9:.0f}GB/s)" if v[2] else "")
                          for k, v in sorted(prof.items())), flush=True)
