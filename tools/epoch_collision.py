"""Stale lookback status words (dev tool / regression): sorts clustered f64 inputs whose keys
carry top-16-bit patterns equal to the level epoch tags, with the epoch counter forced to
those values, and checks every output.  IPLS_LIB=<so> runs a variant build."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2208_06902_b200 as ipls
if os.environ.get("IPLS_LIB"):
    ipls._LIB_PATH = os.path.abspath(os.environ["IPLS_LIB"])
L = ipls.lib()
has_hook = hasattr(L, "ipls_debug_set_epoch")
bad = 0
rng = np.random.default_rng(5)
for tag in (0x3FF0, 0x3FF4, 0xBFF0, 0x4000):
    # keys whose bits 63..48 == tag and bits 47..46 != 0: count field = low 32 bits
    base = np.uint64(tag) << np.uint64(48)
    vals = (base | (np.uint64(3) << np.uint64(46)) |
            rng.integers(0, 1 << 20, 40).astype(np.uint64)).view(np.float64)
    a = vals[rng.integers(0, vals.size, 3_000_000)]
    a = np.concatenate([a, rng.normal(0, 1, 1_000_000)])
    rng.shuffle(a)
    for e0 in range(tag - 3, tag + 1):
        if has_hook:
            L.ipls_debug_set_epoch(e0)
        t = torch.from_numpy(a.view(np.int64).copy()).cuda()
        try:
            ipls.sort(t, k=1024, base_case=4096, key_type=ipls.KEY_F64)
            ok = np.array_equal(t.cpu().numpy().view(np.float64), np.sort(a))
        except ipls.IPLSError as ex:
            ok = False
            print("error", ex)
        bad += not ok
        print(f"tag {tag:#06x} epoch {e0:#06x}: {'ok' if ok else 'WRONG'}", flush=True)
print("hook" if has_hook else "no hook (old build: epochs not forced)", "bad:", bad)
