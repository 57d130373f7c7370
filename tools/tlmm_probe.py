"""One C2-size transpose_lmm (1 column) after a warm-up, for an ncu launch list:
ncu --metrics gpu__time_duration.sum python tools/tlmm_probe.py"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2502_01985_b200 as fl  # noqa: E402

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
sh = bench.make_shard(torch, wl, 0, 1, torch.device("cuda"))
h = bench.build_handle(fl, wl, sh)
del sh
y = torch.rand((h.shape[0], 1), device="cuda")
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _ in range(2):
    h.transpose_lmm(y, traced=False)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
