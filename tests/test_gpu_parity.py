"""GPU parity: the sm_100a Stream-K kernels against the oracle.

* Integer-valued operands (the reference's random_matrix<int64> band, exact in
  bf16/fp16, products and partial sums exact in fp32 below 2^24): C must be
  BIT-exact versus the oracle's int64 execute, for every decomposition.
* Random uniform [-1, 1) operands rounded to bf16/fp16: within the reference's
  own verify bound |c - ref| <= 8 * eps_fp32 * k * max(|ref|, 1)
  (executor.hpp:217-239), eps_fp32 = 2^-23 (fp32 accumulate), ref = oracle
  gemm_reference<float> on the same rounded values.
* Ownership: the device-recorded owner / last peer of every tile equals the
  reference's fixup_peers_of.
"""
import numpy as np
import pytest

import __graft_entry__

pytestmark = pytest.mark.gpu

NAMES = ["data_parallel", "fixed_split", "stream_k", "dp_one_tile_sk", "two_tile_sk_dp"]
EPS32 = float(np.finfo(np.float32).eps)


def strategies(sk, problem, blk, p=148):
    yield sk.data_parallel(problem, blk)
    yield sk.fixed_split(problem, blk, 3)
    yield sk.stream_k(problem, blk, p)
    yield sk.stream_k(problem, blk, 7)
    yield sk.hybrid(problem, blk, p, sk.HybridVariant.DpOneTileSk)
    yield sk.hybrid(problem, blk, p, sk.HybridVariant.TwoTileSkDp)
    yield sk.hybrid(problem, blk, 5, sk.HybridVariant.TwoTileSkDp)


def int_operands(port, m, n, k, seed, shift=0):
    A = port.random_matrix(m, k, seed, "int64") >> shift
    B = port.random_matrix(k, n, seed + 1, "int64") >> shift
    return A, B


def to_bf16_f32(x):
    """Round float32 to the nearest bfloat16 (RNE), returned as float32."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


def test_smoke():
    __graft_entry__.smoke()


VARIANTS = ["1sm", "2sm", "2smw"]


def variant(sk, name):
    return {"1sm": sk.Variant.OneSM, "2sm": sk.Variant.TwoSM, "2smw": sk.Variant.TwoSMWide}[name]


@pytest.mark.parametrize("var", VARIANTS)
@pytest.mark.parametrize("shape", [(128, 256, 64), (384, 768, 1000), (129, 257, 65),
                                   (1000, 1000, 520), (256, 512, 4096), (640, 1280, 192)])
def test_int_bit_exact_all_strategies_execute(sk, port, shape, var):
    m, n, k = shape
    V = variant(sk, var)
    blk = sk.kernel_blocking(sk.DType.BFloat16, V)
    A, B = int_operands(port, m, n, k, 1234 + m)
    want = port.execute("data_parallel", 1, A, B, blk.blk_m, blk.blk_n, blk.blk_k).astype(np.float32)
    Af, Bf = A.astype(np.float32), B.astype(np.float32)
    p = 148 if V == sk.Variant.OneSM else 74
    for a in strategies(sk, sk.GemmProblem(m, n, k), blk, p):
        got = sk.execute(a, Af, Bf, compute=sk.DType.BFloat16, variant=V)
        assert np.array_equal(got, want), (sk.strategy_name(a.strategy), a.param)


@pytest.mark.parametrize("var", VARIANTS)
def test_int_bit_exact_fp16(sk, port, var):
    m, n, k = 512, 768, 640
    V = variant(sk, var)
    blk = sk.kernel_blocking(sk.DType.Float16, V)
    A, B = int_operands(port, m, n, k, 77)
    want = (A @ B).astype(np.float32)
    for a in strategies(sk, sk.GemmProblem(m, n, k), blk):
        got = sk.execute(a, A.astype(np.float16), B.astype(np.float16), compute=sk.DType.Float16,
                         variant=V)
        assert np.array_equal(got, want), sk.strategy_name(a.strategy)


@pytest.mark.parametrize("var", VARIANTS)
def test_edge_schedules_bit_exact(sk, port, var):
    """g > total_iters (empty units), one deep-k tile split 148 ways, the
    pathological DpOneTileSk (150 tiles, p=148: 20 empty ranges, 64 peers)."""
    V = variant(sk, var)
    blk = sk.kernel_blocking(sk.DType.BFloat16, V)
    cases = [
        (sk.GemmProblem(128, 256, 128), lambda p: sk.stream_k(p, blk, 148)),
        (sk.GemmProblem(128, 256, 16384), lambda p: sk.stream_k(p, blk, 148)),
        (sk.GemmProblem(128, 256, 16384), lambda p: sk.fixed_split(p, blk, 5)),
        (sk.GemmProblem(1280, 3840, 1024), lambda p: sk.hybrid(p, blk, 148, sk.HybridVariant.DpOneTileSk)),
        (sk.GemmProblem(1280, 3840, 1024), lambda p: sk.hybrid(p, blk, 148, sk.HybridVariant.TwoTileSkDp)),
    ]
    for problem, make in cases:
        a = make(problem)
        # values in [-8, 7]: |partial sums| <= 64 * 16384 < 2^24, exact in fp32
        A, B = int_operands(port, problem.m, problem.n, problem.k, 99, shift=3)
        want = (A.astype(np.float64) @ B.astype(np.float64)).astype(np.float32)  # exact
        got = sk.execute(a, A.astype(np.float32), B.astype(np.float32), variant=V)
        assert np.array_equal(got, want), (problem, sk.strategy_name(a.strategy))


@pytest.mark.parametrize("var", VARIANTS)
def test_float_within_reference_bound(sk, port, var):
    m, n, k = 768, 1024, 2000
    V = variant(sk, var)
    blk = sk.kernel_blocking(sk.DType.BFloat16, V)
    A = to_bf16_f32(port.random_matrix(m, k, 42, "float32"))
    B = to_bf16_f32(port.random_matrix(k, n, 43, "float32"))
    ref = port.gemm_reference(A, B, blk.blk_m, blk.blk_n, blk.blk_k)
    import oracle

    for a in strategies(sk, sk.GemmProblem(m, n, k), blk):
        got = sk.execute(a, A, B, variant=V)
        ok, max_abs, max_rel = oracle.verify(got, ref, k, EPS32)
        assert ok, (sk.strategy_name(a.strategy), max_abs, max_rel)


@pytest.mark.parametrize("var", VARIANTS)
def test_device_path_deterministic_and_self_cleaning(sk, torch_cuda, var):
    torch = torch_cuda
    m = n = 2048
    k = 4096
    V = variant(sk, var)
    blk = sk.kernel_blocking(sk.DType.BFloat16, V)
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.rand(m, k, device="cuda", generator=g).mul_(2).sub_(1).to(torch.bfloat16)
    B = torch.rand(k, n, device="cuda", generator=g).mul_(2).sub_(1).to(torch.bfloat16)
    ref = A.double() @ B.double()
    for a in (sk.stream_k(sk.GemmProblem(m, n, k), blk, 148),
              sk.hybrid(sk.GemmProblem(m, n, k), blk, 148, sk.HybridVariant.DpOneTileSk)):
        gemm = sk.Gemm(a, variant=V)
        outs = []
        for _ in range(5):
            C = torch.full((m, n), float("nan"), device="cuda")
            gemm.run(A, B, C)
            outs.append(C)
        gemm.check()
        for C in outs[1:]:
            assert torch.equal(C, outs[0])  # fixed fold order: run-to-run identical
        err = (outs[0].double() - ref).abs()
        bound = 8 * EPS32 * k * ref.abs().clamp(min=1)
        assert bool((err <= bound).all())
        # flags re-armed by the owners: the whole flag region is zero again
        flags = gemm.workspace[256:256 + 4 * 512].view(torch.int32)
        assert int(flags.abs().sum()) == 0


@pytest.mark.parametrize("var", VARIANTS)
def test_trace_ownership_equals_fixup_peers_of(sk, torch_cuda, var):
    torch = torch_cuda
    V = variant(sk, var)
    blk = sk.kernel_blocking(sk.DType.BFloat16, V)
    for problem, p in ((sk.GemmProblem(1024, 1024, 32768), 148), (sk.GemmProblem(1280, 3840, 512), 148),
                       (sk.GemmProblem(2048, 2048, 1024), 37)):
        for strat in (sk.Strategy.StreamK, sk.Strategy.FixedSplit, sk.Strategy.DpOneTileSk,
                      sk.Strategy.TwoTileSkDp, sk.Strategy.DataParallel):
            param = {sk.Strategy.FixedSplit: 3, sk.Strategy.DataParallel: 1}.get(strat, p)
            a = sk._assignment(strat, problem, blk, param)
            gemm = sk.Gemm(a, variant=V, trace=True)
            A = torch.zeros(problem.m, problem.k, dtype=torch.bfloat16, device="cuda")
            B = torch.zeros(problem.k, problem.n, dtype=torch.bfloat16, device="cuda")
            C = torch.empty(problem.m, problem.n, device="cuda")
            gemm.run(A, B, C)
            gemm.check()
            t = gemm.trace.cpu().numpy()
            T = a.grid.total_tiles
            tiles = t[:4 * T].reshape(T, 4)
            peers = sk.fixup_peers_of(a)
            for x in range(T):
                assert tiles[x, 0] == peers[x][0] and tiles[x, 1] == peers[x][-1], (strat, x)
                assert tiles[x, 2] == peers[x][0]  # stored by the owner
            # every unit whose range starts mid-tile emitted exactly one partial
            emitted = t[4 * T:4 * T + a.grid_size]
            tbl = a.range_table()
            expect = ((tbl[:, 0] % a.grid.iters_per_tile != 0) & (tbl[:, 1] > tbl[:, 0])).astype(int)
            assert np.array_equal(emitted, expect), strat


@pytest.mark.parametrize("var", VARIANTS)
def test_large_square_checksums(sk, torch_cuda, var):
    """8192^3 (BASELINE config 2): size-independent properties on integer-valued
    operands in [-2, 1]: row/column checksums exact, sampled rows exact."""
    torch = torch_cuda
    m = n = k = 8192
    V = variant(sk, var)
    blk = sk.kernel_blocking(sk.DType.BFloat16, V)
    p = 148 if V == sk.Variant.OneSM else 74
    g = torch.Generator(device="cuda").manual_seed(1)
    A = torch.randint(-2, 2, (m, k), device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randint(-2, 2, (k, n), device="cuda", generator=g).to(torch.bfloat16)
    ones = torch.ones(n, 1, device="cuda", dtype=torch.float64)
    rows = (A.double() @ (B.double() @ ones)).squeeze(1)
    cols = ((torch.ones(1, m, device="cuda", dtype=torch.float64) @ A.double()) @ B.double()).squeeze(0)
    sample = torch.arange(0, m, 997, device="cuda")
    exact_rows = A[sample].double() @ B.double()
    for a in (sk.stream_k(sk.GemmProblem(m, n, k), blk, p),
              sk.hybrid(sk.GemmProblem(m, n, k), blk, p, sk.HybridVariant.TwoTileSkDp),
              sk.data_parallel(sk.GemmProblem(m, n, k), blk)):
        C = torch.empty(m, n, device="cuda")
        gemm = sk.Gemm(a, variant=V)
        gemm.run(A, B, C)
        gemm.check()
        assert torch.equal(C.double().sum(1), rows)
        assert torch.equal(C.double().sum(0), cols)
        assert torch.equal(C[sample].double(), exact_rows)


# ---------------------------------------------------------------- FP64 (config 4)
EPS64 = float(np.finfo(np.float64).eps)


@pytest.mark.parametrize("shape", [(64, 64, 16), (200, 150, 300), (129, 65, 33), (512, 384, 1024)])
def test_fp64_int_bit_exact_all_strategies(sk, port, shape):
    m, n, k = shape
    blk = sk.kernel_blocking(sk.DType.Float64)
    assert (blk.blk_m, blk.blk_n, blk.blk_k) == (64, 64, 16)
    A, B = int_operands(port, m, n, k, 314)
    want = port.execute("data_parallel", 1, A, B, 64, 64, 16).astype(np.float64)
    for a in strategies(sk, sk.GemmProblem(m, n, k), blk, 148):
        got = sk.execute(a, A.astype(np.float64), B.astype(np.float64), compute=sk.DType.Float64)
        assert got.dtype == np.float64
        assert np.array_equal(got, want), (sk.strategy_name(a.strategy), a.param)


def test_fp64_within_reference_bound(sk, port):
    """execute<double> semantics: |c - ref| <= 8 eps64 k max(|ref|, 1) against the
    oracle's gemm_reference<double> on the same inputs (random_matrix<double>)."""
    import oracle

    m, n, k = 300, 260, 1000
    blk = sk.kernel_blocking(sk.DType.Float64)
    A = port.random_matrix(m, k, 81, "float64")
    B = port.random_matrix(k, n, 82, "float64")
    ref = port.gemm_reference(A, B, 64, 64, 16)
    for a in strategies(sk, sk.GemmProblem(m, n, k), blk, 148):
        got = sk.execute(a, A, B, compute=sk.DType.Float64)
        ok, max_abs, max_rel = oracle.verify(got, ref, k, EPS64)
        assert ok, (sk.strategy_name(a.strategy), max_abs, max_rel)


def test_fp64_trace_and_determinism(sk, torch_cuda):
    torch = torch_cuda
    problem = sk.GemmProblem(1024, 1024, 4096)
    blk = sk.kernel_blocking(sk.DType.Float64)
    g = torch.Generator(device="cuda").manual_seed(3)
    A = torch.rand(problem.m, problem.k, device="cuda", dtype=torch.float64, generator=g)
    B = torch.rand(problem.k, problem.n, device="cuda", dtype=torch.float64, generator=g)
    for a in (sk.stream_k(problem, blk, 148), sk.hybrid(problem, blk, 148, sk.HybridVariant.DpOneTileSk)):
        gemm = sk.Gemm(a, sk.DType.Float64, trace=True)
        C1 = torch.empty(problem.m, problem.n, device="cuda", dtype=torch.float64)
        C2 = torch.empty_like(C1)
        gemm.run(A, B, C1)
        gemm.run(A, B, C2)
        gemm.check()
        assert torch.equal(C1, C2)
        ref = A @ B
        assert bool(((C1 - ref).abs() <= 8 * EPS64 * problem.k * ref.abs().clamp(min=1)).all())
        T = a.grid.total_tiles
        tiles = gemm.trace.cpu().numpy()[:4 * T].reshape(T, 4)
        peers = sk.fixup_peers_of(a)
        for x in range(T):
            assert tiles[x, 0] == peers[x][0] and tiles[x, 1] == peers[x][-1]


def test_double_signal_raises_protocol_error_and_recovers(sk, torch_cuda):
    """FixupStore::signal's double-signal check (executor.hpp:108-112, :203-205):
    a flag found already set when a non-owner signals is a protocol violation
    -> ProtocolError (std::logic_error); the next launch on the same workspace
    is clean again."""
    torch = torch_cuda
    problem = sk.GemmProblem(512, 512, 2048)
    blk = sk.kernel_blocking(sk.DType.BFloat16, sk.Variant.OneSM)
    a = sk.stream_k(problem, blk, 37)
    gemm = sk.Gemm(a, sk.DType.BFloat16, sk.Variant.OneSM)
    A = torch.ones(problem.m, problem.k, dtype=torch.bfloat16, device="cuda")
    B = torch.ones(problem.k, problem.n, dtype=torch.bfloat16, device="cuda")
    C = torch.empty(problem.m, problem.n, device="cuda")
    gemm.run(A, B, C)
    gemm.check()
    assert torch.equal(C, torch.full_like(C, 2048.0))
    # corrupt: pre-set every flag (the --corrupt idea of tools/streamk_main.cpp:129)
    gemm.workspace[256:256 + 4 * 37].view(torch.int32).fill_(1)
    gemm.run(A, B, C)
    with pytest.raises(sk.ProtocolError):
        gemm.check()
    gemm.run(A, B, C)  # dirty flags are cleared before the next launch
    gemm.check()
    assert torch.equal(C, torch.full_like(C, 2048.0))


def test_pitched_views_and_alignment(sk, torch_cuda):
    """Leading dimensions larger than the row (pitched views) are honoured;
    misaligned leading dimensions are rejected (SK_EUNSUPPORTED) before launch."""
    torch = torch_cuda
    m, n, k = 300, 520, 700
    blk = sk.kernel_blocking()
    Abig = torch.randint(-8, 8, (m, 1024), device="cuda").to(torch.bfloat16)
    Bbig = torch.randint(-8, 8, (k, 768), device="cuda").to(torch.bfloat16)
    Cbig = torch.zeros(m, 640, device="cuda")
    A, B, Cv = Abig[:, :k], Bbig[:, :n], Cbig[:, :n]
    gemm = sk.Gemm(sk.stream_k(sk.GemmProblem(m, n, k), blk, 11))
    gemm.run(A, B, Cv)
    gemm.check()
    assert torch.equal(Cv, (A.double() @ B.double()).float())
    assert torch.equal(Cbig[:, n:], torch.zeros_like(Cbig[:, n:]))  # nothing written past n
    bad = torch.zeros(m, k + 1, device="cuda", dtype=torch.bfloat16)[:, :k]  # ld = 701: not 16-B
    with pytest.raises(sk.UnsupportedError):
        gemm.run(bad, B, Cv)


def test_graph_capture(sk, torch_cuda):
    """sk_gemm is stream-ordered and capturable: a CUDA graph of launches
    replays to the same result."""
    torch = torch_cuda
    m = n = 1024
    k = 4096
    blk = sk.kernel_blocking(sk.DType.BFloat16, sk.Variant.TwoSM)
    gemm = sk.Gemm(sk.auto_stream_k(sk.GemmProblem(m, n, k), blk, 74), variant=sk.Variant.TwoSM)
    A = torch.randint(-4, 4, (m, k), device="cuda").to(torch.bfloat16)
    B = torch.randint(-4, 4, (k, n), device="cuda").to(torch.bfloat16)
    C = torch.zeros(m, n, device="cuda")
    gemm.run(A, B, C)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            gemm.run(A, B, C)
    C.zero_()
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    gemm.check()
    assert torch.equal(C, (A.double() @ B.double()).float())


@pytest.mark.parametrize("var", ["1sm", "2sm", "2smw", "fp64"])
def test_random_instances_bit_exact(sk, port, var):
    """acceptance.cpp criterion 4 on the device: seeded random problems (dims up to
    700, every decomposition with random knobs) with integer-valued operands are
    bit-exact against the oracle's int64 executor."""
    rng = np.random.default_rng({"1sm": 11, "2sm": 22, "2smw": 44, "fp64": 33}[var])
    if var == "fp64":
        ab, V, dt = sk.DType.Float64, sk.Variant.Auto, np.float64
    else:
        ab, V, dt = sk.DType.BFloat16, variant(sk, var), np.float32
    blk = sk.kernel_blocking(ab, V)
    for trial in range(25):
        m, n, k = (int(x) for x in rng.integers(1, 700, 3))
        A, B = int_operands(port, m, n, k, int(rng.integers(1 << 40)))
        want = (A.astype(np.float64) @ B.astype(np.float64)).astype(dt)
        P = sk.GemmProblem(m, n, k)
        for a in (sk.data_parallel(P, blk), sk.fixed_split(P, blk, int(rng.integers(1, 6))),
                  sk.stream_k(P, blk, int(rng.integers(1, 300))),
                  sk.hybrid(P, blk, int(rng.integers(1, 160)), sk.HybridVariant.DpOneTileSk),
                  sk.hybrid(P, blk, int(rng.integers(1, 160)), sk.HybridVariant.TwoTileSkDp)):
            got = sk.execute(a, A.astype(dt), B.astype(dt), compute=ab, variant=V)
            assert np.array_equal(got, want), (trial, m, n, k, sk.strategy_name(a.strategy), a.param)


def test_device_timeline(sk, torch_cuda, tmp_path):
    """Per-segment device timeline -> reference Timeline CSV / Gantt formats:
    one record per (unit, tile segment), owners with peers carry fixup events,
    every event is inside the launch."""
    torch = torch_cuda
    from paper_2301_03598_b200 import timeline as tlm

    problem = sk.GemmProblem(1280, 3840, 4096)
    V = sk.Variant.TwoSM
    blk = sk.kernel_blocking(sk.DType.BFloat16, V)
    a = sk.stream_k(problem, blk, 74)
    g = sk.Gemm(a, variant=V, timeline=True)
    A = torch.randn(problem.m, problem.k, device="cuda").to(torch.bfloat16)
    B = torch.randn(problem.k, problem.n, device="cuda").to(torch.bfloat16)
    C = torch.empty(problem.m, problem.n, device="cuda")
    g.run(A, B, C)
    g.check()
    rec = g.timeline()
    tbl = a.range_table()
    ipt = a.grid.iters_per_tile
    nseg = sum((e - 1) // ipt - b // ipt + 1 for b, e in tbl if e > b)
    assert len(rec) == nseg
    assert (rec[:, 4] <= rec[:, 5]).all() and (rec[:, 5] <= rec[:, 6]).all() and (rec[:, 6] <= rec[:, 7]).all()
    owners = rec[(rec[:, 3] & 2) != 0]
    peers = sk.fixup_peers_of(a)
    assert len(owners) == sum(len(p) > 1 for p in peers)
    tl = tlm.from_device(rec)
    assert tl.p == 74 and 0 < tlm.utilization(tl) <= 1.0
    with open(tmp_path / "t.csv", "w") as f:
        tlm.write_timeline_csv(tl, f)
    with open(tmp_path / "t.svg", "w") as f:
        tlm.render_gantt(tl, f)
    head = open(tmp_path / "t.csv").readline().strip()
    assert head == "core_id,cta_id,kind,start,end"
    assert open(tmp_path / "t.svg").read().startswith("<svg")


def test_execute_drop_in_all_reference_types(sk, port, ref):
    """execute<int64_t>, execute<float>, execute<double> of the reference, via the
    FP64 tensor path: int64 bit-exact, float/double within the reference's bound,
    each against the reference's own executor on the same inputs."""
    import oracle

    blk = sk.kernel_blocking(sk.DType.Float64)
    m, n, k = 384, 320, 512
    for strat, param in (("stream_k", 37), ("two_tile_sk_dp", 11), ("fixed_split", 3), ("data_parallel", 1)):
        a = sk._assignment(sk.Strategy(NAMES.index(strat)), sk.GemmProblem(m, n, k), blk, param)
        Ai, Bi = int_operands(port, m, n, k, 5)
        Ci = sk.execute(a, Ai, Bi, compute=sk.DType.Float64)
        assert Ci.dtype == np.int64
        assert np.array_equal(Ci, ref.execute(strat, param, Ai, Bi, 64, 64, 16, threads=8))
        Af = port.random_matrix(m, k, 7, "float32")
        Bf = port.random_matrix(k, n, 8, "float32")
        Cf = sk.execute(a, Af, Bf, compute=sk.DType.Float64)
        assert Cf.dtype == np.float32
        ok, _, mr = oracle.verify(Cf, ref.execute(strat, param, Af, Bf, 64, 64, 16, threads=8), k, EPS32)
        assert ok, mr
        Ad = port.random_matrix(m, k, 9, "float64")
        Bd = port.random_matrix(k, n, 10, "float64")
        Cd = sk.execute(a, Ad, Bd, compute=sk.DType.Float64)
        ok, _, mr = oracle.verify(Cd, ref.execute(strat, param, Ad, Bd, 64, 64, 16, threads=8), k, EPS64)
        assert ok, mr
    big = np.full((8, 8), 2 ** 40, np.int64)
    with pytest.raises(sk.UnsupportedError):
        sk.execute(sk.data_parallel(sk.GemmProblem(8, 8, 8), blk), big, big, compute=sk.DType.Float64)


# ---------------------------------------------------------------- die-aware lanes
def test_device_topology_two_dies(sk, torch_cuda):
    """sk_device_topology: a B200 shows two dies, TPC pairs never straddle them."""
    die = sk.device_topology(0)
    sms = torch_cuda.cuda.get_device_properties(0).multi_processor_count
    assert die is not None and len(die) == sms
    assert set(die.tolist()) == {0, 1}
    assert all(die[2 * t] == die[2 * t + 1] for t in range(sms // 2))


@pytest.mark.parametrize("var", VARIANTS)
def test_die_aware_lanes_bit_exact(sk, torch_cuda, monkeypatch, var):
    """SKB200_DIE_AWARE=1 only re-maps data-parallel tiles to persistent CTAs:
    the full-grid schedules give the same C (bit-identical) with and without it,
    and the integer-valued 2048^3 result stays exact (row checksums)."""
    torch = torch_cuda
    m = n = k = 2048
    V = variant(sk, var)
    blk = sk.kernel_blocking(sk.DType.BFloat16, V)
    p = 148 if V == sk.Variant.OneSM else 74
    g = torch.Generator(device="cuda").manual_seed(3)
    A = torch.randint(-2, 2, (m, k), device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randint(-2, 2, (k, n), device="cuda", generator=g).to(torch.bfloat16)
    rows = (A.double() @ (B.double() @ torch.ones(n, 1, device="cuda", dtype=torch.float64))).squeeze(1)
    prob = sk.GemmProblem(m, n, k)
    for a in (sk.data_parallel(prob, blk), sk.hybrid(prob, blk, p, sk.HybridVariant.TwoTileSkDp),
              sk.hybrid(prob, blk, p, sk.HybridVariant.DpOneTileSk)):
        out = []
        for flag in ("0", "1"):
            monkeypatch.setenv("SKB200_DIE_AWARE", flag)
            sk.reload_env()  # the library reads SKB200_* once
            C = torch.full((m, n), float("nan"), device="cuda")
            gemm = sk.Gemm(a, variant=V)
            gemm.run(A, B, C)
            gemm.check()
            out.append(C)
        assert torch.equal(out[0], out[1])
        assert torch.equal(out[1].double().sum(1), rows)
    monkeypatch.undo()
    sk.reload_env()


# ---------------------------------------------------------------- cooperative fixup
@pytest.mark.parametrize("var", VARIANTS)
@pytest.mark.parametrize("shape,g", [((256, 512, 16384), 74), ((512, 512, 8192), 48),
                                     ((384, 640, 6000), 60), ((256, 256, 4096), 37)])
def test_cooperative_fixup_bit_exact(sk, port, torch_cuda, monkeypatch, shape, g, var):
    """Deep-k, few-tile Stream-K schedules (>= 8 contributors per tile) take the
    cooperative fixup: integer-valued C bit-exact vs the oracle, and float C
    bit-identical to the owner-fold protocol (same fold order)."""
    torch = torch_cuda
    m, n, k = shape
    V = variant(sk, var)
    blk = sk.kernel_blocking(sk.DType.BFloat16, V)
    a = sk.stream_k(sk.GemmProblem(m, n, k), blk, g)
    Ai, Bi = int_operands(port, m, n, k, 77 + k)
    want = port.execute("stream_k", g, Ai, Bi, blk.blk_m, blk.blk_n, blk.blk_k).astype(np.float32)
    rng = np.random.default_rng(k)
    Af = to_bf16_f32(rng.uniform(-1, 1, (m, k)).astype(np.float32))
    Bf = to_bf16_f32(rng.uniform(-1, 1, (k, n)).astype(np.float32))
    outs = {}
    for coop in ("1", "0"):
        monkeypatch.setenv("SKB200_COOP", coop)
        sk.reload_env()
        gemm = sk.Gemm(a, variant=V)
        for name, (X, Y) in (("int", (Ai, Bi)), ("float", (Af, Bf))):
            A = torch.from_numpy(X.astype(np.float32)).cuda().to(torch.bfloat16)
            B = torch.from_numpy(Y.astype(np.float32)).cuda().to(torch.bfloat16)
            C = torch.full((m, n), float("nan"), device="cuda")
            for _ in range(2):  # second launch: flags re-armed by the first
                gemm.run(A, B, C)
            gemm.check()
            outs[coop, name] = C.cpu().numpy()
    monkeypatch.undo()
    sk.reload_env()
    assert np.array_equal(outs["1", "int"], want)
    assert np.array_equal(outs["1", "float"], outs["0", "float"])


@pytest.mark.parametrize("var", ["1sm", "2sm"])
@pytest.mark.parametrize("shape,s", [((128, 8192, 8192), 4), ((128, 8192, 8192), 2), ((129, 264, 1024), 2),
                                     ((129, 264, 1024), 8), ((256, 512, 4096), 8), ((1000, 1000, 512), 2),
                                     ((64, 328, 2048), 4), ((300, 1000, 1000), 4),
                                     ((129, 264, 1024), 3), ((64, 328, 2048), 5), ((256, 512, 4096), 6),
                                     ((200, 600, 2048), 7), ((128, 4096, 16384), 7)])
def test_cluster_fixup_fixed_split(sk, port, torch_cuda, monkeypatch, shape, s, var):
    """fixed_split(s) with no empty k-chunk runs the cluster fixup when t * s
    units fit as clusters (the s k-chunks of a tile on one cluster, reduced
    through DSMEM; 1-SM CTAs or 2-SM CTA pairs): integer-valued C bit-exact vs
    the oracle, float C bit-identical to the global-slab owner fold
    (SKB200_CLUSTER_FIX=0), and the recorded ownership equal to the
    reference's fixup_peers_of.  (300 x 1000 x 1000, s = 4: ipt = 16 -> chunks
    of 4; ragged rows and columns.)"""
    torch = torch_cuda
    m, n, k = shape
    V = variant(sk, var)
    blk = sk.kernel_blocking(sk.DType.BFloat16, V)
    a = sk.fixed_split(sk.GemmProblem(m, n, k), blk, s)
    Ai, Bi = int_operands(port, m, n, k, 91 + k, shift=3 if k > 4096 else 0)
    want = port.execute("fixed_split", s, Ai, Bi, blk.blk_m, blk.blk_n, blk.blk_k).astype(np.float32)
    rng = np.random.default_rng(k + s)
    Af = to_bf16_f32(rng.uniform(-1, 1, (m, k)).astype(np.float32))
    Bf = to_bf16_f32(rng.uniform(-1, 1, (k, n)).astype(np.float32))
    owners = [pr[0] for pr in sk.fixup_peers_of(a)]
    outs = {}
    for on in ("1", "0"):
        monkeypatch.setenv("SKB200_CLUSTER_FIX", on)
        sk.reload_env()
        gemm = sk.Gemm(a, variant=V, trace=True)
        for name, (X, Y) in (("int", (Ai, Bi)), ("float", (Af, Bf))):
            A = torch.from_numpy(X.astype(np.float32)).cuda().to(torch.bfloat16)
            B = torch.from_numpy(Y.astype(np.float32)).cuda().to(torch.bfloat16)
            C = torch.full((m, n), float("nan"), device="cuda")
            for _ in range(2):  # the second launch sees the first one's workspace state
                gemm.run(A, B, C)
            gemm.check()
            outs[on, name] = C.cpu().numpy()
        storers = gemm.block_storers()
        assert np.array_equal(storers.reshape(-1), np.array(owners)), on
        if on == "1" and a.grid.total_tiles * s <= sk.cluster_capacity(s, V):
            # the cluster path ran: every unit's record carries S - 1 (partials
            # included; the global-slab path records 0 peers for a partial)
            tl = sk.Gemm(a, variant=V, timeline=True)
            tl.run(A, B, C)
            tl.check()
            kinds = tl.timeline()[:, 3].astype(np.int64)
            assert np.all(((kinds >> 8) & 0xFF) == s - 1), kinds[:8]
    monkeypatch.undo()
    sk.reload_env()
    assert np.array_equal(outs["1", "int"], want)
    assert np.array_equal(outs["0", "int"], want)
    assert np.array_equal(outs["1", "float"], outs["0", "float"])
