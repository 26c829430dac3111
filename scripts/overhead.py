"""Where a short launch spends its time (single-wave data-parallel shapes).

For each shape: event time of one launch (after warm-up, back-to-back pairs so
PDL overlap is included), and from the device stamps of a traced launch:
  prologue_to_mac   first CTA start stamp (after barrier init / TMEM alloc /
                    grid-dependency wait) -> first mainloop start
  mainloop          mainloop start -> accumulator ready (median over tiles)
  epilogue          accumulator ready -> tile stored (median)
  teardown          last tile stored -> last CTA end stamp
  device_span       first CTA start stamp -> last CTA end stamp

  python scripts/overhead.py [--shapes 256x256x256,1024x1024x1024,...]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2301_03598_b200 as sk  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="256x256x256,512x512x1024,1024x1024x1024,2048x2048x512,4096x4096x256")
    ap.add_argument("--strategy", default="data_parallel")
    args = ap.parse_args()
    out = []
    for spec in args.shapes.split(","):
        m, n, k = (int(x) for x in spec.split("x"))
        A = (torch.rand(m, k, device="cuda") * 2 - 1).bfloat16()
        B = (torch.rand(k, n, device="cuda") * 2 - 1).bfloat16()
        C = torch.empty(m, n, device="cuda")
        blk = sk.kernel_blocking(sk.DType.BFloat16, sk.Variant.TwoSM)
        prob = sk.GemmProblem(m, n, k)
        a = sk.data_parallel(prob, blk) if args.strategy == "data_parallel" else sk.stream_k(prob, blk, 74)
        g = sk.Gemm(a, sk.DType.BFloat16, sk.Variant.TwoSM)
        for _ in range(20):
            g.run(A, B, C)
        torch.cuda.synchronize()
        s = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 200
        e0.record(s)
        for _ in range(reps):
            g.run(A, B, C)
        e1.record(s)
        torch.cuda.synchronize()
        per_launch = e0.elapsed_time(e1) / reps * 1e3
        # graph of the same launches (what the sweep times)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for _ in range(50):
                g.run(A, B, C)
        graph.replay()
        torch.cuda.synchronize()
        e0.record(s)
        for _ in range(4):
            graph.replay()
        e1.record(s)
        torch.cuda.synchronize()
        per_graph_launch = e0.elapsed_time(e1) / 200 * 1e3
        t = sk.Gemm(a, sk.DType.BFloat16, sk.Variant.TwoSM, trace=True, timeline=True)
        for _ in range(5):
            t.run(A, B, C)
        torch.cuda.synchronize()
        rec = t.timeline()
        clk = t.cta_clocks.view(-1, 4).cpu().numpy()
        clk = clk[(clk[:, 1] > 0) & (clk[:, 3] > 0)]
        start, end = clk[:, 1].min(), clk[:, 3].max()
        us = lambda x: float(x) / 1e3  # noqa: E731
        out.append({
            "shape": [m, n, k], "tiles": a.grid.total_tiles, "ipt": a.grid.iters_per_tile,
            "event_us_per_launch": round(per_launch, 2),
            "graph_us_per_launch": round(per_graph_launch, 2),
            "device_span_us": round(us(end - start), 2),
            "prologue_to_mac_us": round(us(rec[:, 4].min() - start), 2),
            "mainloop_us": round(us(np.median(rec[:, 5] - rec[:, 4])), 2),
            "epilogue_us": round(us(np.median(rec[:, 7] - rec[:, 5])), 2),
            "teardown_us": round(us(end - rec[:, 7].max()), 2),
            "cta_start_spread_us": round(us(clk[:, 1].max() - start), 2),
        })
        print(json.dumps(out[-1]), flush=True)


if __name__ == "__main__":
    main()
