"""Phase timing of the C2 table upload from pinned host buffers (what bounds
bench.py's e2e; PROBE_PAGEABLE=1: from plain numpy memory, a drop-in user's case).  Run with FL_TRACE_UPLOAD=1 for the library's own
finalize-phase timestamps."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2502_01985_b200 as fl  # noqa: E402
from paper_2502_01985_b200.trainers import GlmSession  # noqa: E402


def main():
    wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
    sh = bench.make_shard(torch, wl, 0, 1, torch.device("cuda"))
    maps, c_t = bench.col_maps(wl)

    def pinned(t):
        if os.environ.get("PROBE_PAGEABLE"):   # plain numpy-owned (pageable) host memory
            return torch.from_numpy(t.cpu().numpy().copy())
        p = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        p.copy_(t)
        return p

    host = [pinned(sh["fact"])] + [pinned(d) for d in sh["dims"]]
    fks = [pinned(f) for f in sh["fks"]]
    y_h = pinned(sh["y"])
    del sh
    torch.cuda.empty_cache()
    nbytes = sum(t.numel() * t.element_size() for t in host + fks)
    for j in range(int(os.environ.get('PROBE_JOBS', '4'))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        c0 = time.process_time()
        h = fl.TargetHandle.from_arrays([t.numpy() for t in host],
                                        [None] + [f.numpy() for f in fks], maps,
                                        host[0].shape[0], c_t)
        ta = time.perf_counter()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        print(f"  from_arrays returned {1e3 * (ta - t0):.1f} ms, sync {1e3 * (t1 - ta):.1f} ms, "
              f"process cpu {1e3 * (time.process_time() - c0):.1f} ms", flush=True)
        s = GlmSession(h, wl["model"], y_h.numpy(), 1e-9)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        s.close()
        del h
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        print(f"job {j}: upload {1e3 * (t1 - t0):.1f} ms ({nbytes / (t1 - t0) / 1e9:.1f} GB/s), "
              f"session {1e3 * (t2 - t1):.1f} ms, teardown {1e3 * (t3 - t2):.1f} ms", flush=True)


if __name__ == "__main__":
    main()
