"""Explicit range tables (SK_EXPLICIT): execute<T> on a WorkAssignment that no
closed-form decomposition produces, e.g. one read back by from_text
(types.cpp:101-123).  The reference executes any table (executor.hpp:147-185):
ranges are indexed by position, a tile's starter folds every other range that
touches it in ascending id, tiles nobody starts stay zero.

CPU tests: table validation through sk_workspace_size, fixup_peers_of of a
table against the oracle port and the reference, port vs reference execute on
random tables.  GPU tests (marked): the kernels on random tables, bit-exact.
"""
import ctypes as C

import numpy as np
import pytest


def random_table(rng, total, ipt, g, drop=0.0, shuffle=True):
    """A random explicit table over [0, total): g ranges cut at random points
    (some dropped to empty ranges, leaving gaps, orphan partials and unstarted
    tiles), ids assigned by a random topological order of "a tile's starter <
    every other range touching it" -- the condition the persistent grid needs."""
    cuts = np.sort(rng.integers(0, total + 1, size=g - 1))
    bounds = np.concatenate([[0], cuts, [total]])
    pieces = [(int(bounds[i]), int(bounds[i + 1])) for i in range(g)]
    pieces = [(b, b) if rng.random() < drop else (b, e) for b, e in pieces]
    # edges: starter of each tile -> other nonempty pieces of that tile
    succ = {i: set() for i in range(g)}
    indeg = [0] * g
    tiles = {}
    for i, (b, e) in enumerate(pieces):
        if b < e:
            for t in range(b // ipt, (e - 1) // ipt + 1):
                tiles.setdefault(t, []).append(i)
    for t, lst in tiles.items():
        st = [i for i in lst if pieces[i][0] <= t * ipt]
        if st:
            for j in lst:
                if j != st[0] and j not in succ[st[0]]:
                    succ[st[0]].add(j)
                    indeg[j] += 1
    order = []
    ready = [i for i in range(g) if indeg[i] == 0]
    while ready:
        i = ready.pop(int(rng.integers(len(ready))) if shuffle else 0)
        order.append(i)
        for j in succ[i]:
            indeg[j] -= 1
            if indeg[j] == 0:
                ready.append(j)
    assert len(order) == g
    tbl = np.zeros((g, 2), np.int64)
    for new_id, i in enumerate(order):
        tbl[new_id] = pieces[i]
    return tbl


def assignment(sk, problem, blk, tbl):
    a = sk.WorkAssignment(strategy=sk.Strategy.StreamK, grid_size=len(tbl), problem=problem,
                          blocking=blk, grid=sk.tile_grid(problem, blk),
                          ranges=[sk.CtaRange(i, int(b), int(e)) for i, (b, e) in enumerate(tbl)],
                          param=0)
    return a


def desc_for(sk, problem, blk, tbl, ab=None):
    d = sk.sk_gemm_desc()
    d.problem = problem._c()
    d.blocking = blk._c()
    d.strategy = sk.SK_EXPLICIT
    d.ab_type = int(ab if ab is not None else sk.DType.BFloat16)
    d.variant = int(sk.Variant.Auto)
    tbl = np.ascontiguousarray(tbl, np.int64)
    d.ranges = tbl.ctypes.data if tbl.size else None
    d.num_ranges = tbl.shape[0]
    return d, tbl


def ws_status(sk, problem, blk, tbl):
    d, keep = desc_for(sk, problem, blk, tbl)
    n = C.c_size_t()
    st = sk.lib().sk_workspace_size(C.byref(d), C.byref(n))
    return st, n.value


# ---------------------------------------------------------------- CPU: validation
def test_validation_statuses(sk):
    blk = sk.kernel_blocking(sk.DType.BFloat16)  # 256x256x64 (2-SM)
    P = sk.GemmProblem(512, 512, 256)  # 4 tiles x 4 iterations
    ok = np.array([[0, 6], [6, 16]], np.int64)
    st, n_ok = ws_status(sk, P, blk, ok)
    assert st == sk.SK_OK
    # the table itself is part of the workspace: 2g ranges + t+1 offsets + nnz ids,
    # after the 256-B header, the flags and g units x 2 ranks x 128 KB slabs
    table = 8 * (2 * 2 + 4 + 1 + 5)
    assert n_ok >= 256 + 256 + 2 * 2 * 256 * 128 * 4 + table
    # out of bounds / reversed: mac_loop's invalid_argument
    for bad in ([[0, 17]], [[-1, 4]], [[5, 4]]):
        assert ws_status(sk, P, blk, np.array(bad, np.int64))[0] == sk.SK_EINVAL
    # tile 0 started twice: the reference would wait forever
    assert ws_status(sk, P, blk, np.array([[0, 2], [0, 4]], np.int64))[0] == sk.SK_EINVAL
    # starter (id 1) with a lower-id peer (id 0): not orderable on a persistent grid
    assert ws_status(sk, P, blk, np.array([[2, 4], [0, 2]], np.int64))[0] == sk.SK_EUNSUPPORTED
    # gaps, empty ranges and an unstarted tile are fine (the reference zero-fills)
    assert ws_status(sk, P, blk, np.array([[2, 4], [4, 4], [9, 16]], np.int64))[0] == sk.SK_OK
    # zero ranges: nothing to run, C stays zero
    assert ws_status(sk, P, blk, np.zeros((0, 2), np.int64))[0] == sk.SK_OK
    # closed-form entry points do not take SK_EXPLICIT
    g = C.c_int64()
    assert sk.lib().sk_schedule(C.byref(P._c()), C.byref(blk._c()), sk.SK_EXPLICIT, 1,
                                C.byref(g), None, 0) == sk.SK_EINVAL


def test_cta_ids_must_match_positions(sk):
    blk = sk.kernel_blocking(sk.DType.BFloat16)
    P = sk.GemmProblem(256, 256, 256)
    a = assignment(sk, P, blk, np.array([[0, 2], [2, 4]], np.int64))
    a.ranges[0] = sk.CtaRange(1, 0, 2)
    with pytest.raises(ValueError):
        sk.fixup_peers_of(a)


@pytest.mark.parametrize("seed", range(6))
def test_peers_of_table_match_oracle(sk, port, seed):
    rng = np.random.default_rng(100 + seed)
    blk = sk.BlockingFactors(128, 128, 16)
    P = sk.GemmProblem(int(rng.integers(1, 700)), int(rng.integers(1, 700)), int(rng.integers(1, 300)))
    grid = sk.tile_grid(P, blk)
    g = int(rng.integers(1, 3 * grid.total_tiles + 2))
    tbl = random_table(rng, grid.total_iters, grid.iters_per_tile, g, drop=0.2)
    got = sk.fixup_peers_of(assignment(sk, P, blk, tbl))
    off = np.zeros(grid.total_tiles + 1, np.int64)
    nnz = C.c_int64()
    f = port.lib.skor_fixup_peers
    tp = np.ascontiguousarray(tbl)
    f(tp.ctypes.data_as(C.c_void_p), C.c_int64(g), C.c_int64(grid.iters_per_tile),
      C.c_int64(grid.total_tiles), off.ctypes.data_as(C.c_void_p), None, C.c_int64(0), C.byref(nnz))
    ids = np.zeros(max(nnz.value, 1), np.int64)
    f(tp.ctypes.data_as(C.c_void_p), C.c_int64(g), C.c_int64(grid.iters_per_tile),
      C.c_int64(grid.total_tiles), off.ctypes.data_as(C.c_void_p), ids.ctypes.data_as(C.c_void_p),
      C.c_int64(ids.size), C.byref(nnz))
    want = [ids[off[t]:off[t + 1]].tolist() for t in range(grid.total_tiles)]
    assert got == want


@pytest.mark.parametrize("seed", range(4))
def test_port_execute_table_matches_reference(ref, port, seed):
    """The restatement's executor on arbitrary tables == the reference's execute
    on the same table parsed by its own from_text (int64: bit-exact)."""
    rng = np.random.default_rng(7 + seed)
    m, n, k = (int(x) for x in rng.integers(1, 200, size=3))
    bm, bn, bk = 64, 32, 8
    tiles = -(-m // bm) * -(-n // bn)
    ipt = -(-k // bk)
    tbl = random_table(rng, tiles * ipt, ipt, int(rng.integers(1, 3 * tiles + 2)), drop=0.25)
    A = port.random_matrix(m, k, 11 + seed, "int64")
    B = port.random_matrix(k, n, 12 + seed, "int64")
    want = ref.execute_ranges(tbl, A, B, bm, bn, bk, threads=1)
    got = port.execute_ranges(tbl, A, B, bm, bn, bk)
    assert np.array_equal(got, want)


# ---------------------------------------------------------------- GPU
CASES = [
    ("2sm", (640, 768, 1000), 0.0),
    ("2sm", (513, 300, 777), 0.3),
    ("1sm", (384, 768, 1000), 0.0),
    ("1sm", (300, 520, 333), 0.3),
    ("fp64", (200, 130, 260), 0.0),
    ("fp64", (129, 191, 100), 0.3),
]


@pytest.mark.gpu
@pytest.mark.parametrize("var,shape,drop", CASES)
@pytest.mark.parametrize("seed", range(3))
def test_gpu_random_tables_bit_exact(sk, port, torch_cuda, var, shape, drop, seed):
    rng = np.random.default_rng(1000 * seed + hash((var, shape)) % 997)
    m, n, k = shape
    if var == "fp64":
        dt, v = sk.DType.Float64, sk.Variant.Auto
    else:
        dt, v = sk.DType.BFloat16, (sk.Variant.OneSM if var == "1sm" else sk.Variant.TwoSM)
    blk = sk.kernel_blocking(dt, v)
    P = sk.GemmProblem(m, n, k)
    grid = sk.tile_grid(P, blk)
    g = int(rng.integers(1, 4 * grid.total_tiles + 3))
    tbl = random_table(rng, grid.total_iters, grid.iters_per_tile, g, drop=drop)
    a = assignment(sk, P, blk, tbl)
    A = port.random_matrix(m, k, 31 + seed, "int64")
    B = port.random_matrix(k, n, 32 + seed, "int64")
    want = port.execute_ranges(tbl, A, B, blk.blk_m, blk.blk_n, blk.blk_k)
    if dt == sk.DType.Float64:
        got = sk.execute(a, A.astype(np.float64), B.astype(np.float64), compute=dt, variant=v)
        assert np.array_equal(got, want.astype(np.float64))
    else:
        got = sk.execute(a, A.astype(np.float32), B.astype(np.float32), compute=dt, variant=v)
        assert np.array_equal(got, want.astype(np.float32))


@pytest.mark.gpu
def test_gpu_table_reuse_and_trace(sk, port, torch_cuda):
    """Alternating explicit tables and closed forms on the same sk_execute
    workspace (table re-upload / invalidation), and the device ownership trace
    of an explicit table against fixup_peers_of."""
    torch = torch_cuda
    blk = sk.kernel_blocking(sk.DType.BFloat16, sk.Variant.TwoSM)
    P = sk.GemmProblem(512, 768, 640)
    grid = sk.tile_grid(P, blk)
    rng = np.random.default_rng(5)
    A = port.random_matrix(P.m, P.k, 3, "int64")
    B = port.random_matrix(P.k, P.n, 4, "int64")
    Af, Bf = A.astype(np.float32), B.astype(np.float32)
    tables = [random_table(rng, grid.total_iters, grid.iters_per_tile, g, drop=d)
              for g, d in ((9, 0.0), (17, 0.2), (9, 0.0))]
    for i, tbl in enumerate(tables * 2):
        a = assignment(sk, P, blk, tbl)
        want = port.execute_ranges(tbl, A, B, blk.blk_m, blk.blk_n, blk.blk_k).astype(np.float32)
        got = sk.execute(a, Af, Bf, compute=sk.DType.BFloat16, variant=sk.Variant.TwoSM)
        assert np.array_equal(got, want), i
        sk_a = sk.stream_k(P, blk, 5 + i)
        want = port.execute("stream_k", 5 + i, A, B, blk.blk_m, blk.blk_n, blk.blk_k).astype(np.float32)
        assert np.array_equal(sk.execute(sk_a, Af, Bf, compute=sk.DType.BFloat16,
                                         variant=sk.Variant.TwoSM), want)
    # device trace: every started tile's owner and last peer
    tbl = tables[1]
    a = assignment(sk, P, blk, tbl)
    gm = sk.Gemm(a, variant=sk.Variant.TwoSM, trace=True)
    At = torch.tensor(Af).to(torch.bfloat16).cuda()
    Bt = torch.tensor(Bf).to(torch.bfloat16).cuda()
    Ct = torch.zeros(P.m, P.n, device="cuda")
    for _ in range(3):
        gm.run(At, Bt, Ct)
        gm.check()
    tr = gm.trace[: 4 * grid.total_tiles].view(-1, 4).cpu().numpy()
    peers = sk.fixup_peers_of(a)
    for t, lst in enumerate(peers):
        started = bool(lst) and tbl[lst[0], 0] <= t * grid.iters_per_tile
        if started:
            assert tr[t, 0] == lst[0] and tr[t, 1] == lst[-1] and tr[t, 3] == len(lst) - 1, t
        else:
            assert tr[t, 0] == -1, t
