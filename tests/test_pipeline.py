"""sk_execute with pinned host buffers overlaps H2D, compute and D2H (A arrives
by tile rows and B by column panels behind flags the producer waits on; finished
blocks of C leave on a copy stream while the kernel runs).  The schedule is
unchanged, so on integer-valued data C must be bit-identical to the serial path
and to the oracle."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def pinned(torch, arr):
    t = torch.empty(arr.shape, dtype={np.float32: torch.float32, np.float64: torch.float64,
                                      np.float16: torch.float16}[arr.dtype.type], pin_memory=True)
    out = t.numpy()
    out[...] = arr
    return t, out


def run(sk, a, A, B, compute, variant, pipeline, out):
    old = os.environ.get("SKB200_PIPELINE")
    os.environ["SKB200_PIPELINE"] = "1" if pipeline else "0"
    sk.reload_env()  # the library reads SKB200_* once
    try:
        out[...] = np.nan
        return sk.execute(a, A, B, compute=compute, variant=variant, out=out).copy()
    finally:
        if old is None:
            del os.environ["SKB200_PIPELINE"]
        else:
            os.environ["SKB200_PIPELINE"] = old
        sk.reload_env()


@pytest.mark.parametrize("var", ["1sm", "2sm", "fp64"])
@pytest.mark.parametrize("shape", [(1000, 1000, 520), (2048, 768, 1024), (777, 1300, 333),
                                   (2100, 2600, 700)])
def test_pipelined_execute_bit_identical(sk, port, torch_cuda, var, shape):
    torch = torch_cuda
    m, n, k = shape
    if var == "fp64":
        dt, v, hdt = sk.DType.Float64, sk.Variant.Auto, np.float64
    else:
        dt, v, hdt = sk.DType.Float16, (sk.Variant.OneSM if var == "1sm" else sk.Variant.TwoSM), np.float16
    blk = sk.kernel_blocking(dt, v)
    P = sk.GemmProblem(m, n, k)
    Ai = port.random_matrix(m, k, 21, "int64") >> 2
    Bi = port.random_matrix(k, n, 22, "int64") >> 2
    _ta, A = pinned(torch, Ai.astype(hdt))
    _tb, B = pinned(torch, Bi.astype(hdt))
    _tc, Cp = pinned(torch, np.zeros((m, n), np.float64 if var == "fp64" else np.float32))
    for a in (sk.data_parallel(P, blk), sk.stream_k(P, blk, 9),
              sk.hybrid(P, blk, 7, sk.HybridVariant.TwoTileSkDp), sk.fixed_split(P, blk, 3)):
        want = port.execute(sk.strategy_name(a.strategy), a.param, Ai, Bi, blk.blk_m, blk.blk_n, blk.blk_k)
        serial = run(sk, a, A, B, dt, v, False, Cp)
        piped = run(sk, a, A, B, dt, v, True, Cp)
        assert np.array_equal(serial, piped), sk.strategy_name(a.strategy)
        assert np.array_equal(piped, want.astype(piped.dtype)), sk.strategy_name(a.strategy)


def test_pipelined_explicit_table_with_unstarted_tiles(sk, port, torch_cuda):
    from test_explicit import assignment, random_table

    torch = torch_cuda
    blk = sk.kernel_blocking(sk.DType.Float16, sk.Variant.TwoSM)
    P = sk.GemmProblem(1100, 900, 700)
    grid = sk.tile_grid(P, blk)
    rng = np.random.default_rng(3)
    tbl = random_table(rng, grid.total_iters, grid.iters_per_tile, 23, drop=0.35)
    a = assignment(sk, P, blk, tbl)
    Ai = port.random_matrix(P.m, P.k, 5, "int64") >> 2
    Bi = port.random_matrix(P.k, P.n, 6, "int64") >> 2
    _ta, A = pinned(torch, Ai.astype(np.float16))
    _tb, B = pinned(torch, Bi.astype(np.float16))
    _tc, Cp = pinned(torch, np.zeros((P.m, P.n), np.float32))
    want = port.execute_ranges(tbl, Ai, Bi, blk.blk_m, blk.blk_n, blk.blk_k).astype(np.float32)
    for _ in range(2):
        got = run(sk, a, A, B, sk.DType.Float16, sk.Variant.TwoSM, True, Cp)
        assert np.array_equal(got, want)
