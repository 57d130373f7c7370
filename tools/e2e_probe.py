import time, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
import paper_2502_01985_b200 as fl
wl = bench.WORKLOADS["c3"]
dev = torch.device("cuda")
sh = bench.make_shard(torch, wl, 0, 1, dev)
maps, c_t = bench.col_maps(wl)
def pinned(t):
    p = torch.empty(t.shape, dtype=t.dtype, pin_memory=True); p.copy_(t); return p
host = [pinned(sh["fact"])] + [pinned(d) for d in sh["dims"]]
fks = [pinned(f) for f in sh["fks"]]
torch.cuda.synchronize()
for j in range(4):
    t0 = time.perf_counter()
    h2 = fl.TargetHandle.from_arrays([t.numpy() for t in host], [None] + [f.numpy() for f in fks], maps, sh["rows"], c_t)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    from paper_2502_01985_b200.trainers import KMeansSession, kmeans_init
    c0 = kmeans_init(h2, wl["k"], 0); t2 = time.perf_counter()
    s2 = KMeansSession(h2, wl["k"], c0); torch.cuda.synchronize(); t3 = time.perf_counter()
    s2.run(100); torch.cuda.synchronize(); t4 = time.perf_counter()
    r = s2.result(100); t5 = time.perf_counter()
    s2.close(); del h2; torch.cuda.empty_cache()
    print(f"job {j}: upload {t1-t0:.4f} init {t2-t1:.4f} session {t3-t2:.4f} run {t4-t3:.4f} result {t5-t4:.4f}", flush=True)
