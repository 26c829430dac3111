"""compute-sanitizer driver for this round's paths (run from the repo root):
cooperative fixup (>= 8 contributors), grouped tile ids, pieces outside C
skipped (ragged shapes), die-aware lanes, and the tile-block transfer pipeline
(pinned host buffers: B panels, A rows, C blocks, DP slot permutation).
Integer-valued operands: every result must be bit-exact."""
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2301_03598_b200 as sk  # noqa: E402

port = oracle.Oracle("port")
ok = True
for V in (sk.Variant.OneSM, sk.Variant.TwoSM):
    blk = sk.kernel_blocking(sk.DType.BFloat16, V)
    for (m, n, k), mk in (((256, 520, 8192), lambda P: sk.stream_k(P, blk, 60)),      # coop
                          ((300, 700, 700), lambda P: sk.stream_k(P, blk, 13)),       # ragged
                          ((1100, 900, 300), lambda P: sk.hybrid(P, blk, 5, sk.HybridVariant.TwoTileSkDp))):
        P = sk.GemmProblem(m, n, k)
        A = port.random_matrix(m, k, 1, "int64") >> 2
        B = port.random_matrix(k, n, 2, "int64") >> 2
        want = (A.astype(np.float64) @ B.astype(np.float64)).astype(np.float32)
        a = mk(P)
        got = sk.execute(a, A.astype(np.float32), B.astype(np.float32), compute=sk.DType.BFloat16, variant=V)
        r = np.array_equal(got, want)
        ok &= r
        print(int(V), m, n, k, sk.strategy_name(a.strategy), "pageable", r, flush=True)
        # pinned fp16 buffers: the tile-block transfer pipeline
        At = torch.empty((m, k), dtype=torch.float16, pin_memory=True)
        Bt = torch.empty((k, n), dtype=torch.float16, pin_memory=True)
        Ct = torch.empty((m, n), dtype=torch.float32, pin_memory=True)
        At.numpy()[...] = A.astype(np.float16)
        Bt.numpy()[...] = B.astype(np.float16)
        got = sk.execute(a, At.numpy(), Bt.numpy(), compute=sk.DType.Float16, variant=V, out=Ct.numpy())
        r = np.array_equal(got, want)
        ok &= r
        print(int(V), m, n, k, sk.strategy_name(a.strategy), "pinned", r, flush=True)
os.environ["SKB200_DIE_AWARE"] = "1"
blk = sk.kernel_blocking(sk.DType.BFloat16, sk.Variant.TwoSM)
P = sk.GemmProblem(2048, 2048, 256)
A = port.random_matrix(2048, 256, 3, "int64") >> 2
B = port.random_matrix(256, 2048, 4, "int64") >> 2
want = (A.astype(np.float64) @ B.astype(np.float64)).astype(np.float32)
for a in (sk.data_parallel(P, blk), sk.hybrid(P, blk, 74, sk.HybridVariant.TwoTileSkDp)):
    got = sk.execute(a, A.astype(np.float32), B.astype(np.float32), compute=sk.DType.BFloat16)
    r = np.array_equal(got, want)
    ok &= r
    print("die-aware", sk.strategy_name(a.strategy), r, flush=True)
print("ALL_OK" if ok else "MISMATCH")
