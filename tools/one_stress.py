"""One sort of a base-case stress input (tests/test_gpu_parity.py::test_base_case_stress_parity)
for compute-sanitizer runs (dev tool): python tools/one_stress.py KIND N K"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2208_06902_b200 as ipls
from paper_2208_06902_b200 import datagen
kind, n, k = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
a = datagen.stress_array(np.random.default_rng(n + k + len(kind)), n, kind)
t = torch.from_numpy(a.view(np.int64).copy()).cuda()
ipls.sort(t, k=k, base_case=4096, key_type=0 if a.dtype == np.float64 else 1)
ok = np.array_equal(t.cpu().numpy().view(a.dtype), np.sort(a))
print("sorted:", ok)
