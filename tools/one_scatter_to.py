"""One ipls_partition_count + ipls_partition_scatter_to of a whole workload into a local
receive buffer (G = 1 plan), for ncu captures of k_scatter_peer (dev tool):
python tools/one_scatter_to.py CFG REPS"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2208_06902_b200 as ipls
from paper_2208_06902_b200 import datagen
from paper_2208_06902_b200.distributed import fused_plan
name, reps = sys.argv[1], int(sys.argv[2])
cfg = datagen.CONFIGS[name]
a = datagen.generate(name)
kt = 0 if a.dtype == np.float64 else 1
t = torch.from_numpy(a.view(np.int64)).cuda()
S = ipls.sample_size(a.size, cfg.k)
smp = torch.zeros(S, dtype=torch.int64, device="cuda")
ipls.sample_strata(t, 0, a.size, S, smp)
m = ipls.fit_fmcd(smp, cfg.k, key_type=kt, presorted=False)
buf = torch.empty_like(t)
for _ in range(reps):
    cnt = np.diff(ipls.partition_count(t, m, key_type=kt).cpu().numpy())[None, :]
    _, _, owner, offset, recv = fused_plan(cnt, 1)
    addr = torch.from_numpy(buf.data_ptr() + 8 * offset[0]).cuda()
    ipls.partition_scatter_to(t, m, addr, key_type=kt)
torch.cuda.synchronize()
ref = torch.empty_like(t)
ipls.partition_level(t, ref, m, key_type=kt)
print("same as ipls_partition_level:", bool(torch.equal(buf, ref)))
