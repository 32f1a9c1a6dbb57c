"""Time dist_sort (the multi-GPU top level) in a one-rank NCCL group against the
one-GPU sort on the same input (dev tool).  At one rank the exchange is a
device copy, so the difference is the cost of the extra top-level pass (sample, fit,
partition, copy) that a G-rank run pays before its local sorts."""
import os
import socket
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

import paper_2208_06902_b200 as ipls
from paper_2208_06902_b200 import datagen
from paper_2208_06902_b200.distributed import SymmPeers, dist_sort

s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = datagen.CONFIGS[name]
a = datagen.generate(name)
src = torch.from_numpy(a.view(np.int64)).cuda()
if a.dtype == np.float64:
    src = src.view(torch.float64)
work = torch.empty_like(src)
reps = int(os.environ.get("REPS", "8"))


def timed(fn):
    ts = []
    for _ in range(reps):
        work.copy_(src)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); out = fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts[2:])), out


ms1, _ = timed(lambda: ipls.sort(work, k=cfg.k, base_case=cfg.base_case))
want = torch.sort(src)[0]
for label, kw in [("all-to-all path", dict(fused=False)),
                  ("fused exchange, buffer allocated per call", dict(fused=True)),
                  ("fused exchange, buffer reused", dict(fused=True, peers=SymmPeers(reuse=True)))]:
    msd, res = timed(lambda: dist_sort(work, k=cfg.k, base_case=cfg.base_case, **kw))
    ok = torch.equal(res.keys, want)
    work.copy_(src); torch.cuda.synchronize()
    ipls.profile_reset(); ipls.profile_enable(True)
    dist_sort(work, k=cfg.k, base_case=cfg.base_case, **kw)
    ipls.profile_enable(False)
    prof = ipls.profile_read()
    for _ in range(3):
        work.copy_(src); torch.cuda.synchronize()
        marks = []
        dist_sort(work, k=cfg.k, base_case=cfg.base_case, marks=marks, **kw)
        torch.cuda.synchronize()
    print(f"{name}, {label}: one-GPU sort {ms1:.3f} ms, dist_sort (1 rank) {msd:.3f} ms "
          f"(+{msd - ms1:.3f} ms top-level pass), sorted={ok}", flush=True)
    print("  phases: " + "  ".join(f"{n}:{marks[i - 1][1].elapsed_time(e):.3f}ms"
                                   for i, (n, e) in enumerate(marks) if i), flush=True)
    print("  library kernels in one dist_sort: " + "  ".join(
        f"{k}:{v[1]:.3f}ms/{v[0]}" for k, v in sorted(prof.items())), flush=True)
dist.destroy_process_group()
