import os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, 'oracle')
import paper_2301_03598_b200 as sk, oracle
port = oracle.Oracle('port')
for V, ab in ((sk.Variant.OneSM, sk.DType.BFloat16), (sk.Variant.TwoSM, sk.DType.BFloat16), (sk.Variant.Auto, sk.DType.Float64)):
    blk = sk.kernel_blocking(ab, V)
    m, n, k = 300, 520, 700
    A = port.random_matrix(m, k, 1, 'int64'); B = port.random_matrix(k, n, 2, 'int64')
    want = (A.astype(np.float64) @ B.astype(np.float64))
    P = sk.GemmProblem(m, n, k)
    dt = np.float64 if ab == sk.DType.Float64 else np.float32
    for a in (sk.stream_k(P, blk, 13), sk.fixed_split(P, blk, 3), sk.hybrid(P, blk, 5, sk.HybridVariant.TwoTileSkDp)):
        got = sk.execute(a, A.astype(dt), B.astype(dt), compute=ab, variant=V)
        print(V, ab, sk.strategy_name(a.strategy), np.array_equal(got, want.astype(dt)))
