"""Host->device copy bandwidth on the GPU box (what bounds bench.py's e2e).

Times an 8 GB pinned fp32 buffer (the C2 fact block) copied to the device
as one cudaMemcpyAsync, and split into chunks on 1, 2 and 4 streams.
"""
import time

import torch


def main():
    n = 2_000_000_000                      # 8 GB of fp32
    h = torch.empty(n, dtype=torch.float32, pin_memory=True)
    h.fill_(1.0)
    d = torch.empty(n, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    for streams in (1, 2, 4):
        for chunks in (1, 8, 32):
            if chunks < streams:
                continue
            ss = [torch.cuda.Stream() for _ in range(streams)]
            step = (n + chunks - 1) // chunks
            best = 1e9
            for _ in range(3):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                for c in range(chunks):
                    with torch.cuda.stream(ss[c % streams]):
                        d[c * step:(c + 1) * step].copy_(h[c * step:(c + 1) * step], non_blocking=True)
                torch.cuda.synchronize()
                best = min(best, time.perf_counter() - t0)
            print(f"streams {streams} chunks {chunks}: {4 * n / best / 1e9:.1f} GB/s", flush=True)
    # device -> host for reference
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    print(f"d2h: {4 * n / (time.perf_counter() - t0) / 1e9:.1f} GB/s")


if __name__ == "__main__":
    main()
