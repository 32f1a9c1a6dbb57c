"""One warm sort of a BASELINE config (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2208_06902_b200 as ipls
from paper_2208_06902_b200 import datagen
if os.environ.get("IPLS_LIB"):  # A/B a variant build
    ipls._LIB_PATH = os.path.abspath(os.environ["IPLS_LIB"])
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = datagen.CONFIGS[name]
a = datagen.generate(name)
kt = 0 if a.dtype == np.float64 else 1
src = torch.from_numpy(a.view(np.int64)).cuda()
t = torch.empty_like(src)
for _ in range(reps):
    t.copy_(src)
    ipls.sort(t, k=cfg.k, base_case=cfg.base_case, key_type=kt)
torch.cuda.synchronize()
print("ok", name, reps)
