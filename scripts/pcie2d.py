"""PCIe copy rates for the shapes a tile-granular sk_execute pipeline would use:
contiguous vs 2-D strips (B column panels of 256 bf16 columns = 512 B rows, C
blocks of 256 fp32 columns = 1 KB rows), H2D and D2H, alone.

  python scripts/pcie2d.py
"""
import json
import time

import torch
from cuda.bindings import runtime as rt


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return best


def main():
    n = k = 8192
    Bh = torch.empty(k, n, dtype=torch.bfloat16).pin_memory()
    Bd = torch.empty(k, n, dtype=torch.bfloat16, device="cuda")
    Ch = torch.empty(8192, n, dtype=torch.float32).pin_memory()
    Cd = torch.empty(8192, n, dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    H2D, D2H = rt.cudaMemcpyKind.cudaMemcpyHostToDevice, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost
    out = {}
    out["h2d_contig_GBps"] = Bh.numel() * 2 / timed(lambda: Bd.copy_(Bh, non_blocking=True)) / 1e9
    for cols in (256, 1024):
        def panels(cols=cols):
            for c in range(0, n, cols):
                rt.cudaMemcpy2DAsync(Bd.data_ptr() + c * 2, n * 2, Bh.data_ptr() + c * 2, n * 2, cols * 2, k,
                                     H2D, s)
        out[f"h2d_2d_{cols * 2}B_rows_GBps"] = Bh.numel() * 2 / timed(panels) / 1e9
    out["d2h_contig_GBps"] = Ch.numel() * 4 / timed(lambda: Ch.copy_(Cd, non_blocking=True)) / 1e9
    for cols, rows in ((256, 2048), (1024, 2048)):
        def blocks(cols=cols, rows=rows):
            for r in range(0, 8192, rows):
                for c in range(0, n, cols):
                    off = (r * n + c) * 4
                    rt.cudaMemcpy2DAsync(Ch.data_ptr() + off, n * 4, Cd.data_ptr() + off, n * 4, cols * 4, rows,
                                         D2H, s)
        out[f"d2h_2d_{cols * 4}B_rows_GBps"] = Ch.numel() * 4 / timed(blocks) / 1e9
    print(json.dumps({k: round(v, 1) for k, v in out.items()}))


if __name__ == "__main__":
    main()
