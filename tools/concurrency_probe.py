"""Headroom probe (dev tool): two C2 sorts on two streams from two host threads at once against
the same two sorts back to back.  A large gain means the kernels leave SM resources idle that
another CTA in a different phase could use."""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2208_06902_b200 as ipls
from paper_2208_06902_b200 import datagen
a = datagen.generate("C2")
src = torch.from_numpy(a.view(np.int64)).cuda()
bufs = [torch.empty_like(src) for _ in range(2)]
streams = [torch.cuda.Stream() for _ in range(2)]
def one(i):
    with torch.cuda.stream(streams[i]):
        ipls.sort(bufs[i], k=1024, base_case=4096, key_type=0)
    streams[i].synchronize()
for rep in range(6):
    for b in bufs: b.copy_(src)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); one(0); one(1); t1 = time.perf_counter()
    for b in bufs: b.copy_(src)
    torch.cuda.synchronize()
    th = [threading.Thread(target=one, args=(i,)) for i in range(2)]
    t2 = time.perf_counter()
    for x in th: x.start()
    for x in th: x.join()
    t3 = time.perf_counter()
    print(f"serial {1e3*(t1-t0):.3f} ms  concurrent {1e3*(t3-t2):.3f} ms", flush=True)
