"""SURVEY §8(f) NEXT #4 (dev tool, run on the GPU box): the paper's nine synthetic workloads at
N = 1e8 and the Normal size sweep 1e4..1e9, k = 1024, B = 4096.

Per case: median ms over timed reps (CUDA events around ipls.sort on its stream; D2D restore
of the pristine input outside the events), keys/s, and the whole-sort roofline fraction
(16 n (L*+1) bytes / 8 TB/s).  Every output is checked on the GPU against
torch.sort of the input in ordering-key order (sorted, same multiset).  Inputs: the paper
workloads from datagen.paper_workload (numpy PCG64(7)); the sweep draws Normal(0,1) on the GPU
with torch.Generator(cuda).manual_seed(11) (1e9 keys would take a minute on the host).

usage: python tools/sweep.py [--part workloads|sizes|models|all] [--out FILE]
  models: C1-C5 with the FMCD linear model (IPLS) and with the splitter tree (IPS4o's
  classifier, IPLS_FLAG_TREE_MODEL) on the same framework.
"""
import argparse, json, math, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2208_06902_b200 as ipls
from paper_2208_06902_b200 import datagen

K, B = 1024, 4096
SIGN = -(1 << 63)


def signed_order(t, f64):
    """int64 tensor whose signed order is the ordering-key order of the keys."""
    if f64:
        ok = torch.where(t < 0, ~t, t | SIGN)  # ok as unsigned, stored in int64
        return ok ^ SIGN
    return t ^ SIGN


def run_case(x, f64, reps, warm=3, k=K, base_case=B, model=ipls.MODEL_LINEAR):
    work = torch.empty_like(x)
    kt = ipls.KEY_F64 if f64 else ipls.KEY_U64
    times = []
    for i in range(warm + reps):
        work.copy_(x)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ipls.sort(work, k=k, base_case=base_case, key_type=kt, model=model)
        e1.record()
        torch.cuda.synchronize()
        if i >= warm:
            times.append(e0.elapsed_time(e1))
    got = signed_order(work, f64)
    ok_sorted = bool((got[1:] >= got[:-1]).all())
    ref = torch.sort(signed_order(x, f64))[0]
    same = bool(torch.equal(ref, got))
    del ref, got, work
    n = x.numel()
    ms = statistics.median(times)
    lstar = max(1, math.ceil(math.log(math.ceil(n / base_case), k))) if n > base_case else 0
    model = 16 * n * (lstar + 1)
    return {"n": n, "ms": round(ms, 4), "keys_per_s": n / (ms / 1e3),
            "frac_of_8TBps": round(model / 8e12 / (ms / 1e3), 4), "L*": lstar,
            "reps": reps, "correct": ok_sorted and same}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--part", default="all")
    ap.add_argument("--out", default=None)
    ap.add_argument("--n", type=int, default=100_000_000)
    args = ap.parse_args()
    res = {"k": K, "base_case": B, "device": torch.cuda.get_device_name(0)}
    if args.part in ("workloads", "all"):
        res["workloads"] = {}
        for name, (dt, desc) in datagen.PAPER_WORKLOADS.items():
            a = datagen.paper_workload(name, args.n)
            x = torch.from_numpy(a.view(np.int64)).cuda()
            r = run_case(x, dt == "f64", reps=10)
            r["desc"] = desc
            res["workloads"][name] = r
            print(name, json.dumps(r), flush=True)
            del x
    if args.part in ("models", "all"):
        res["models"] = {}
        for name in ["C1", "C2", "C3", "C4", "C5"]:
            cfg = datagen.CONFIGS[name]
            a = datagen.generate(name)
            x = torch.from_numpy(a.view(np.int64)).cuda()
            for model, mname in [(ipls.MODEL_LINEAR, "fmcd"), (ipls.MODEL_TREE, "tree"),
                                 (ipls.MODEL_TREE_EQ, "tree_eq")]:
                r = run_case(x, a.dtype == np.float64, reps=10, k=cfg.k, base_case=cfg.base_case,
                             model=model)
                res["models"][f"{name}/{mname}"] = r
                print(name, mname, json.dumps(r), flush=True)
            del x
    if args.part in ("sizes", "all"):
        res["normal_sizes"] = []
        g = torch.Generator(device="cuda")
        g.manual_seed(11)
        for n in [10**4, 10**5, 10**6, 10**7, 10**8, 10**9]:
            x = torch.randn(n, dtype=torch.float64, device="cuda", generator=g).view(torch.int64)
            r = run_case(x, True, reps=50 if n <= 10**7 else (10 if n <= 10**8 else 5))
            res["normal_sizes"].append(r)
            print("normal", json.dumps(r), flush=True)
            del x
            torch.cuda.empty_cache()
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
