"""The persistent sequence every CTA walks (SegmentIter, sk_kernel_common.cuh),
checked on the host through sk_persistent_order against the reference's
decomposition (decompose.cpp) -- CPU only, no device needed:

* coverage: over all CTAs, the segments are exactly the executor's segments of
  every nonempty range (executor.hpp:149-185), each unit on one CTA, its
  segments contiguous and ascending;
* order: balanced / fixed-split units run in descending id per CTA
  (executor.hpp:187-193);
* deadlock freedom of the owner-fold protocol: a step-by-step simulation in
  which an owner segment completes only after all of its tile's peers
  (fixup_peers_of, decompose.cpp:123-136) have emitted their partials, with
  every CTA co-resident, always runs to completion.
"""
import itertools

import numpy as np

import pytest


def segments_of(a):
    ipt = a.grid.iters_per_tile
    out = []
    for r in a.ranges:
        it = r.iter_begin
        while it < r.iter_end:
            tile = it // ipt
            lb = it - tile * ipt
            le = min(r.iter_end, (tile + 1) * ipt) - tile * ipt
            out.append((r.cta_id, tile, lb, le))
            it = (tile + 1) * ipt
    return out


def simulate(seqs, peers, ipt):
    """Owner segments (lb == 0 on a tile with more than one contributor) wait
    for every peer's partial; everything else completes when reached."""
    done_partials = set()
    pos = [0] * len(seqs)
    progressed = True
    while progressed:
        progressed = False
        for c, seq in enumerate(seqs):
            while pos[c] < len(seq):
                u, tile, lb, le = (int(x) for x in seq[pos[c]])
                plist = peers[tile]
                if lb == 0 and len(plist) > 1 and plist[0] == u:
                    if not all((p, tile) in done_partials for p in plist[1:]):
                        break
                elif lb != 0:
                    done_partials.add((u, tile))
                pos[c] += 1
                progressed = True
    return all(pos[c] == len(s) for c, s in enumerate(seqs))


CASES = [
    ((384, 384, 128), (128, 256, 64)),
    ((8192, 8192, 8192), (256, 256, 64)),
    ((1024, 1024, 32768), (256, 256, 64)),
    ((1280, 3840, 4096), (256, 256, 64)),
    ((1000, 1000, 520), (128, 256, 64)),
    ((129, 257, 65), (256, 256, 64)),
    ((3000, 700, 2000), (128, 256, 64)),
]


@pytest.mark.parametrize("shape,blk", CASES)
@pytest.mark.parametrize("p", [74, 148, 5])
def test_persistent_order_covers_and_never_deadlocks(sk, shape, blk, p):
    problem = sk.GemmProblem(*shape)
    b = sk.BlockingFactors(*blk)
    variant = sk.Variant.TwoSM if blk[0] == 256 else sk.Variant.OneSM
    assignments = [sk.data_parallel(problem, b), sk.fixed_split(problem, b, 3),
                   sk.stream_k(problem, b, p), sk.stream_k(problem, b, max(1, p // 3)),
                   sk.hybrid(problem, b, p, sk.HybridVariant.DpOneTileSk),
                   sk.hybrid(problem, b, p, sk.HybridVariant.TwoTileSkDp)]
    for a in assignments:
        num_ctas = min(a.grid_size, p)
        seqs = sk.persistent_order(a, num_ctas, variant=variant)
        got = sorted(tuple(int(x) for x in r) for s in seqs for r in s)
        assert got == sorted(segments_of(a)), (a.strategy, a.param)
        unit_cta = {}
        for c, s in enumerate(seqs):
            for r in s:
                assert unit_cta.setdefault(int(r[0]), c) == c  # a unit never splits across CTAs
            units = [int(u) for u, _ in itertools.groupby(int(r[0]) for r in s)]
            assert len(units) == len(set(units))  # each unit's segments are contiguous
            balanced = [u for u in units if not _dp_unit(sk, a, u)]
            assert balanced == sorted(balanced, reverse=True)
        assert simulate(seqs, sk.fixup_peers_of(a), a.grid.iters_per_tile), (a.strategy, a.param)


def _dp_unit(sk, a, u):
    """Data-parallel ids: all of data_parallel, and the hybrids' DP regions
    (decompose.cpp:92-119); balanced and fixed-split ids are the rest."""
    if a.strategy == sk.Strategy.DataParallel:
        return True
    if a.strategy not in (sk.Strategy.DpOneTileSk, sk.Strategy.TwoTileSkDp):
        return False
    t, p = a.grid.total_tiles, a.param
    w, r = divmod(t, p)
    if r == 0:  # degenerates to data-parallel
        return True
    if a.strategy == sk.Strategy.DpOneTileSk:  # DP ids [0, w*p), SK ids after
        return u < w * p
    return u >= p  # TwoTileSkDp: SK ids [0, p), DP ids [p, p + d)


@pytest.mark.parametrize("shape,blk", CASES + [((8192, 8192, 64), (256, 256, 64)),
                                               ((4000, 300, 777), (128, 256, 64))])
def test_tile_blocks_bijection(sk, shape, blk):
    """The default tile id -> block of C map is the reference's row-major one
    (executor.hpp:69-70, 173-174) on every kernel; the opt-in grouped layout
    (sk_gemm_desc.tile_group = G or -1) still denotes every block exactly once."""
    problem = sk.GemmProblem(*shape)
    b = sk.BlockingFactors(*blk)
    variant = sk.Variant.TwoSM if blk[0] == 256 else sk.Variant.OneSM
    a = sk.stream_k(problem, b, 74)
    tm, tn = a.grid.tiles_m, a.grid.tiles_n
    row_major = np.array([(t // tn, t % tn) for t in range(tm * tn)])
    assert np.array_equal(sk.tile_blocks(a, variant=variant), row_major)
    for g in (-1, 3, 10 ** 6):  # raster height, explicit, clamped to tiles_m
        blocks = sk.tile_blocks(a, variant=variant, tile_group=g)
        assert sorted(map(tuple, blocks.tolist())) == sorted(map(tuple, row_major.tolist()))
    b64 = sk.kernel_blocking(sk.DType.Float64)
    a64 = sk.stream_k(problem, b64, 296)
    t64 = a64.grid.tiles_n
    want = np.array([(t // t64, t % t64) for t in range(a64.grid.total_tiles)])
    assert np.array_equal(sk.tile_blocks(a64, sk.DType.Float64, sk.Variant.Auto, tile_group=-1), want)
