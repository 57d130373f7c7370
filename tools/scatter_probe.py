"""Random-row HBM bandwidth on the B200 (decides the lmm output strategy):
100M rows, rows written to / read from a random permutation of positions,
128-byte rows (32 fp32: a k = 32 lmm output row) and 80-byte rows (20 fp32:
a C2 fact row), against the sequential copy.  CUDA-event medians."""
import torch


def timed(fn, reps=5):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(reps)]
    fn()
    torch.cuda.synchronize()
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a, b in ev)[reps // 2]


n = 100_000_000
perm = torch.randperm(n, device="cuda")
for w in (32, 20):
    src = torch.rand((n, w), device="cuda")
    dst = torch.empty_like(src)
    gb = 2 * n * w * 4 / 1e9
    t_seq = timed(lambda: dst.copy_(src))
    t_sc = timed(lambda: dst.index_copy_(0, perm, src))
    t_ga = timed(lambda: torch.index_select(src, 0, perm, out=dst))
    print(f"rows of {w * 4} B: copy {t_seq:.2f} ms ({gb / t_seq:.0f} TB/s... GB/ms), "
          f"scatter {t_sc:.2f} ms, gather {t_ga:.2f} ms  ({gb:.1f} GB moved each)", flush=True)
    del src, dst
    torch.cuda.empty_cache()
