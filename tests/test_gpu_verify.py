"""GPU parity at BASELINE sizes and on the reference's own inputs.

* sk_random_matrix (the device restatement of random_matrix<T>, matrix.hpp:
  39-68) reproduces the reference generator value for value.
* Float C at BASELINE config 2 (8192^3) and config 3 sizes: the reference's
  random_matrix<float>(42), (43) rounded to bf16 feed both sides; >= 256 seeded
  rows of C are checked against the reference's gemm_reference<float>
  (executor.hpp:22-54) under its verify bound 8 eps_f32 k max(|ref|, 1)
  (executor.hpp:217-239), for DP, stream_k(p), two_tile_sk_dp(p) and the
  policy on every tcgen05 variant (1-SM, 2-SM, 2-SM wide).
* The tile -> C map: the device-recorded storer of every block of C is the
  owner (fixup_peers_of front) of tile row * tiles_n + col -- the reference's
  row-major map (executor.hpp:69-70) -- and the pinned (transfer-pipelined)
  and pageable sk_execute paths return identical C.
* Config 1 echo: 384 x 384 x 128 on an explicit 4-CTA persistent grid, DP vs
  stream_k(4), against the reference executor.
* The sweep's per-row verification (sweep.Verifier) passes on config-3 /
  corpus samples.
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
EPS32 = float(np.finfo(np.float32).eps)


def to_bf16_f32(x):
    u = np.ascontiguousarray(x, np.float32).view(np.uint32)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


@pytest.fixture(scope="module")
def checker():
    import oracle

    return oracle.Oracle("reference" if oracle.have_reference() else "port")


def test_random_matrix_device_matches_reference(sk, port, torch_cuda):
    torch = torch_cuda
    for rows, cols, seed in ((37, 53, 5), (1000, 777, 2 ** 63 + 12345)):
        i64 = port.random_matrix(rows, cols, seed, "int64")
        f32 = port.random_matrix(rows, cols, seed, "float32")
        f64 = port.random_matrix(rows, cols, seed, "float64")
        got = sk.random_matrix_device(rows, cols, seed, sk.DType.Int64, sk.DType.Float32).cpu().numpy()
        assert np.array_equal(got, i64.astype(np.float32))
        got = sk.random_matrix_device(rows, cols, seed, sk.DType.Int64, sk.DType.BFloat16, shift=3)
        assert np.array_equal(got.float().cpu().numpy(), (i64 >> 3).astype(np.float32))
        got = sk.random_matrix_device(rows, cols, seed, sk.DType.Float32, sk.DType.Float32).cpu().numpy()
        assert np.array_equal(got.view(np.uint32), f32.view(np.uint32))
        got = sk.random_matrix_device(rows, cols, seed, sk.DType.Float32, sk.DType.BFloat16)
        assert np.array_equal(got.float().cpu().numpy().view(np.uint32), to_bf16_f32(f32).view(np.uint32))
        got = sk.random_matrix_device(rows, cols, seed, sk.DType.Float32, sk.DType.Float16)
        assert np.array_equal(got.cpu().numpy(), f32.astype(np.float16))
        got = sk.random_matrix_device(rows, cols, seed, sk.DType.Float64, sk.DType.Float64).cpu().numpy()
        assert np.array_equal(got.view(np.uint64), f64.view(np.uint64))
    torch.cuda.synchronize()


def _rows_reference(checker, Arows, Bh, blk):
    """gemm_reference<float> on a row sample: each element is the same
    sequential-k sum it has in the full matrix (executor.hpp:33-50)."""
    with ThreadPoolExecutor(max_workers=16) as ex:
        parts = list(ex.map(lambda i: checker.gemm_reference(np.ascontiguousarray(Arows[i:i + 1]), Bh,
                                                             blk.blk_m, blk.blk_n, blk.blk_k),
                            range(Arows.shape[0])))
    return np.concatenate(parts, axis=0)


BASELINE_SHAPES = [(8192, 8192, 8192), (1024, 1024, 32768), (1280, 3840, 4096), (1024, 4864, 4096)]


@pytest.mark.parametrize("shape", BASELINE_SHAPES)
def test_float_parity_baseline_sizes(sk, torch_cuda, checker, shape):
    import oracle

    torch = torch_cuda
    m, n, k = shape
    rng = np.random.default_rng(m + n + k)
    rows = np.sort(rng.choice(m, size=256, replace=False))
    ridx = torch.from_numpy(rows).cuda()
    A = sk.random_matrix_device(m, k, 42, sk.DType.Float32, sk.DType.BFloat16)
    B = sk.random_matrix_device(k, n, 43, sk.DType.Float32, sk.DType.BFloat16)
    Bh = B.float().cpu().numpy()
    want = None
    for V, p in ((sk.Variant.TwoSM, 74), (sk.Variant.OneSM, 148), (sk.Variant.TwoSMWide, 74)):
        blk = sk.kernel_blocking(sk.DType.BFloat16, V)
        if want is None:
            want = _rows_reference(checker, A[ridx].float().cpu().numpy(), Bh, blk)
        P = sk.GemmProblem(m, n, k)
        for a in (sk.data_parallel(P, blk), sk.stream_k(P, blk, p),
                  sk.hybrid(P, blk, p, sk.HybridVariant.TwoTileSkDp), sk.auto_stream_k(P, blk, p)):
            C = torch.full((m, n), float("nan"), device="cuda")
            g = sk.Gemm(a, variant=V)
            g.run(A, B, C)
            g.check()
            ok, max_abs, max_rel = oracle.verify(C[ridx].cpu().numpy(), want, k, EPS32)
            assert ok, (shape, V, sk.strategy_name(a.strategy), a.param, max_abs, max_rel)
            assert not bool(torch.isnan(C).any())


@pytest.mark.parametrize("var", ["1sm", "2sm", "2smw"])
def test_trace_blocks_follow_row_major_map(sk, torch_cuda, var):
    """Trace section 3: the unit that stored block (r, c) is the owner of tile id
    r * tiles_n + c (executor.hpp:69-70); with the opt-in grouped layout the
    storer follows sk_tile_block instead."""
    torch = torch_cuda
    V = {"1sm": sk.Variant.OneSM, "2sm": sk.Variant.TwoSM, "2smw": sk.Variant.TwoSMWide}[var]
    p = 148 if var == "1sm" else 74
    blk = sk.kernel_blocking(sk.DType.BFloat16, V)
    for shape in ((8192, 8192, 1024), (1280, 3840, 512), (2304, 2304, 2048), (1000, 3008, 704)):
        P = sk.GemmProblem(*shape)
        A = torch.zeros(P.m, P.k, dtype=torch.bfloat16, device="cuda")
        B = torch.zeros(P.k, P.n, dtype=torch.bfloat16, device="cuda")
        C = torch.empty(P.m, P.n, device="cuda")
        for a in (sk.hybrid(P, blk, p, sk.HybridVariant.TwoTileSkDp), sk.stream_k(P, blk, p),
                  sk.data_parallel(P, blk), sk.hybrid(P, blk, p, sk.HybridVariant.DpOneTileSk)):
            owners = np.array([pr[0] for pr in sk.fixup_peers_of(a)])
            tm, tn = a.grid.tiles_m, a.grid.tiles_n
            g = sk.Gemm(a, variant=V, trace=True)
            g.run(A, B, C)
            g.check()
            assert np.array_equal(g.block_storers(), owners.reshape(tm, tn)), (shape, a.strategy)
            g2 = sk.Gemm(a, variant=V, trace=True, tile_group=-1)
            g2.run(A, B, C)
            g2.check()
            blocks = sk.tile_blocks(a, variant=V, tile_group=-1)
            want = np.full((tm, tn), -1)
            want[blocks[:, 0], blocks[:, 1]] = owners
            assert np.array_equal(g2.block_storers(), want), (shape, a.strategy)


def test_pinned_and_pageable_execute_agree(sk, torch_cuda, checker):
    """The transfer-pipelined (pinned) and plain sk_execute paths hand the same
    WorkAssignment's blocks of C to the same units: identical float C."""
    torch = torch_cuda
    m, n, k = 2048, 3072, 1536
    A = to_bf16_f32(checker.random_matrix(m, k, 11, "float32"))
    B = to_bf16_f32(checker.random_matrix(k, n, 12, "float32"))
    Ab = torch.from_numpy(A).to(torch.bfloat16)
    Bb = torch.from_numpy(B).to(torch.bfloat16)
    An, Bn = Ab.view(torch.int16).numpy().view(np.uint16), Bb.view(torch.int16).numpy().view(np.uint16)
    Ap = Ab.pin_memory().view(torch.int16).numpy().view(np.uint16)
    Bp = Bb.pin_memory().view(torch.int16).numpy().view(np.uint16)
    Cp = torch.empty(m, n).pin_memory().numpy()
    blk = sk.kernel_blocking(sk.DType.BFloat16, sk.Variant.TwoSM)
    P = sk.GemmProblem(m, n, k)
    for a in (sk.hybrid(P, blk, 74, sk.HybridVariant.TwoTileSkDp), sk.stream_k(P, blk, 74)):
        pageable = sk.execute(a, An, Bn)
        pinned = sk.execute(a, Ap, Bp, out=Cp)
        assert np.array_equal(pageable, pinned), sk.strategy_name(a.strategy)


def test_config1_echo_four_cta_grid(sk, torch_cuda, checker):
    """BASELINE config 1 on the device: 384 x 384 x 128 on an explicit 4-CTA
    persistent grid (num_ctas = 4), data-parallel vs stream_k(4); C against
    the reference executor, ownership against fixup_peers_of."""
    import oracle

    torch = torch_cuda
    m = n = 384
    k = 128
    blk = sk.kernel_blocking(sk.DType.BFloat16, sk.Variant.OneSM)  # 128 x 256 x 64: 6 tiles, ipt 2
    P = sk.GemmProblem(m, n, k)
    Af = to_bf16_f32(checker.random_matrix(m, k, 31, "float32"))
    Bf = to_bf16_f32(checker.random_matrix(k, n, 32, "float32"))
    Ai = checker.random_matrix(m, k, 31, "int64")
    Bi = checker.random_matrix(k, n, 32, "int64")
    for a in (sk.data_parallel(P, blk), sk.stream_k(P, blk, 4)):
        want_f = checker.execute(int(a.strategy), a.param, Af, Bf, blk.blk_m, blk.blk_n, blk.blk_k, threads=4)
        want_i = checker.execute(int(a.strategy), a.param, Ai, Bi, blk.blk_m, blk.blk_n, blk.blk_k, threads=4)
        g = sk.Gemm(a, variant=sk.Variant.OneSM, num_ctas=4, trace=True)
        for X, Y, want, exact in ((Ai, Bi, want_i, True), (Af, Bf, want_f, False)):
            A = torch.from_numpy(X.astype(np.float32)).cuda().to(torch.bfloat16)
            B = torch.from_numpy(Y.astype(np.float32)).cuda().to(torch.bfloat16)
            C = torch.full((m, n), float("nan"), device="cuda")
            g.run(A, B, C)
            g.check()
            got = C.cpu().numpy()
            if exact:
                assert np.array_equal(got, want.astype(np.float32))
            else:
                ok, _, mr = oracle.verify(got, want, k, EPS32)
                assert ok, mr
        owners = np.array([pr[0] for pr in sk.fixup_peers_of(a)])
        assert np.array_equal(g.block_storers().ravel(), owners)


def test_persistent_capacity(sk, torch_cuda):
    sms = torch_cuda.cuda.get_device_properties(0).multi_processor_count
    assert sk.persistent_capacity(sk.DType.BFloat16, sk.Variant.OneSM) == sms
    assert sk.persistent_capacity(sk.DType.BFloat16, sk.Variant.TwoSM) == sms // 2
    assert sk.persistent_capacity(sk.DType.Float64, sk.Variant.Auto) == 2 * sms


@pytest.mark.parametrize("which", ["config3", "corpus"])
def test_sweep_rows_verified(sk, torch_cuda, which):
    from paper_2301_03598_b200 import sweep as sw

    if which == "config3":
        shapes, seeds, full = sw.CONFIG3[1:4], None, True
    else:
        c = sk.corpus(0, 24)
        shapes, seeds, full = [tuple(int(x) for x in r[:3]) for r in c], [int(r[3]) for r in c], False
    rows = sw.run(shapes, ["data_parallel", "stream_k:auto", "stream_k"], sk.Variant.TwoSM, "bf16",
                  seeds=seeds, verify=True, force_full=full)
    assert rows and all(r["verified"] == "pass" for r in rows), [
        (r["m"], r["n"], r["k"], r["strategy"], r["int_exact"], r["max_rel_err"]) for r in rows
        if r["verified"] != "pass"]
    if full:
        assert all(r["float_check"] == "full" and r["cpu_time_s"] > 0 for r in rows)
    for r in rows:
        assert len(sw.csv_line(r).split(",")) == len(sw.COLUMNS)


@pytest.mark.parametrize("var", ["1sm", "2sm"])
def test_cluster_capacity_and_policy(sk, torch_cuda, checker, var):
    """The policy takes fixed_split(S) on the DSMEM cluster fixup when t * S
    units fit as clusters of S and every k-chunk has >= 8 iterations (1-SM
    CTAs / 2-SM CTA pairs); the wide tile never does.  The result is verified
    against the reference executor on a row sample."""
    import oracle

    torch = torch_cuda
    V = sk.Variant.OneSM if var == "1sm" else sk.Variant.TwoSM
    p = 148 if var == "1sm" else 74
    caps = {S: sk.cluster_capacity(S, V) for S in range(2, 9)}
    assert all(0 <= caps[S] <= p and caps[S] % S == 0 for S in caps), caps
    assert caps[2] > 0
    blk = sk.kernel_blocking(sk.DType.BFloat16, V)
    min_iters = sk.default_cost_params(variant=V).cluster_min_iters
    # 32, 16, 20, 40 tiles on the 1-SM kernel (128 x 10240: S = 3 when 4 does not fit)
    for m, n, k in ((128, 8192, 8192), (128, 4096, 16384), (64, 5120, 8192), (128, 10240, 8192)):
        a = sk.auto_stream_k(sk.GemmProblem(m, n, k), blk, p)
        t, ipt = a.grid.total_tiles, a.grid.iters_per_tile
        want_s = next((S for S in (8, 4, 3, 2) if t * S <= caps[S] and -(-ipt // S) >= min_iters
                       and (S - 1) * -(-ipt // S) < ipt), None)
        if want_s is None:
            assert a.strategy != sk.Strategy.FixedSplit, (m, n, k, caps)
        else:
            assert (a.strategy, a.param) == (sk.Strategy.FixedSplit, want_s), (m, n, k, caps)
    m, n, k = 128, 8192, 8192
    a = sk.auto_stream_k(sk.GemmProblem(m, n, k), blk, p)
    bw = sk.kernel_blocking(sk.DType.BFloat16, sk.Variant.TwoSMWide)
    aw = sk.auto_stream_k(sk.GemmProblem(m, n, k), bw, 74, sk.default_cost_params(variant=sk.Variant.TwoSMWide))
    assert aw.strategy != sk.Strategy.FixedSplit
    A = sk.random_matrix_device(m, k, 42, sk.DType.Float32, sk.DType.BFloat16)
    B = sk.random_matrix_device(k, n, 43, sk.DType.Float32, sk.DType.BFloat16)
    C = torch.full((m, n), float("nan"), device="cuda")
    g = sk.Gemm(a, variant=V)
    g.run(A, B, C)
    g.check()
    rows = np.arange(0, m, 8)
    want = _rows_reference(checker, A[torch.from_numpy(rows).cuda()].float().cpu().numpy(),
                           B.float().cpu().numpy(), blk)
    ok, max_abs, max_rel = oracle.verify(C[torch.from_numpy(rows).cuda()].cpu().numpy(), want, k, EPS32)
    assert ok, (max_abs, max_rel)
