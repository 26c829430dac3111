"""Grid-size model (csrc/costmodel.cpp): the reference's formula for one wave
(costmodel.cpp:13-48), its argmin/tie rule, and NNLS recovery of planted
constants (acceptance.cpp criterion 3(b) restated)."""
import math

import pytest


def grid(sk, m, n, k, b=(128, 128, 32)):
    return sk.tile_grid(sk.GemmProblem(m, n, k), sk.BlockingFactors(*b))


def params(sk, **kw):
    p = sk.CostParams()
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def test_one_wave_formula_matches_reference(sk):
    """For g <= p and e = s = 0 the model is the reference's predict_time."""
    g = grid(sk, 256, 3584, 8192)  # t = 56, ipt = 256, total = 14336
    c = params(sk, a=1.0, b=5.0, c=1.0, d=10.0)
    for gs in (1, 8, 64, 108):
        ipc = math.ceil(14336 / gs)
        peers = math.ceil(256 / ipc)
        want = 1.0 + (5.0 if peers > 1 else 0.0) + ipc + 10.0 * (peers - 1)
        assert sk.predict_time(c, g, gs, 108) == pytest.approx(want)
    # iters_per_cta(wide, 108) == 133 (acceptance.cpp:52-53)
    assert math.ceil(g.total_iters / 108) == 133


def test_waves_and_segments(sk):
    g = grid(sk, 1024, 1024, 1024)  # t = 64 tiles, ipt = 32
    c = params(sk, e=2.0, a=1.0, c=0.5, s=3.0)
    # data-parallel g = t = 64 with p = 16: 4 waves of (a + c*ipt + s*1)
    assert sk.predict_time(c, g, 64, 16) == pytest.approx(2.0 + 4 * (1.0 + 0.5 * 32 + 3.0))


def test_select_prefers_dp_within_margin(sk):
    g = grid(sk, 1024, 1024, 1024)
    c = params(sk, a=1.0, c=1.0, margin=0.0)
    gsel = sk.select_grid_size(c, g, 108)
    assert gsel in range(1, 109) or gsel == 64
    c.margin = 0.99  # nothing beats DP by 99%
    assert sk.select_grid_size(c, g, 108) == g.total_tiles


def test_select_deep_k_picks_small_grid(sk):
    """Reduction-heavy constants give a small-g optimum on one deep-k tile
    (acceptance.cpp:104-106: 128x128x16384 -> g = 8)."""
    g = grid(sk, 128, 128, 16384)
    c = params(sk, a=1.0, b=1.0, c=1.0, d=8.0)
    assert sk.select_grid_size(c, g, 108) == 8


def test_calibrate_recovers_planted(sk):
    planted = params(sk, e=3.0, a=1.5, b=2.0, c=0.25, d=1.0, s=4.0)
    samples = []
    for shape in ((256, 3584, 8192), (1024, 1024, 1024), (128, 128, 16384), (4096, 4096, 512),
                  (2048, 512, 4096)):
        g = grid(sk, *shape)
        for gs in sorted({1, 2, 8, 32, 64, 74, g.total_tiles}):
            samples.append((g, gs, sk.predict_time(planted, g, gs, 74)))
    fit = sk.calibrate(samples, 74, margin=0.1)
    assert fit.fit_residual < 1e-9
    for f in ("e", "a", "b", "c", "d", "s"):
        assert getattr(fit, f) == pytest.approx(getattr(planted, f), rel=1e-6, abs=1e-9), f
    assert fit.margin == pytest.approx(0.1)


def test_auto_stream_k(sk):
    blk = sk.kernel_blocking(sk.DType.BFloat16, sk.Variant.TwoSM)
    p = sk.default_cost_params(sk.DType.BFloat16, sk.Variant.TwoSM)
    p.cluster_min_iters = 0.0  # the model alone (the cluster rule needs a device)
    # deep-k, few tiles: Stream-K
    a = sk.auto_stream_k(sk.GemmProblem(1024, 1024, 32768), blk, 74, p)
    assert a.strategy == sk.Strategy.StreamK and a.grid_size <= 74
    # small k, many tiles: data-parallel
    a = sk.auto_stream_k(sk.GemmProblem(4096, 4096, 256), blk, 74, p)
    assert a.strategy == sk.Strategy.DataParallel


def test_cluster_rule_constants(sk):
    """The cluster-fixup rule's per-kernel constants: 1-SM chunks >= 8
    iterations, 2-SM pairs >= 16, off on the wide tile and FP64."""
    one = sk.default_cost_params(sk.DType.BFloat16, sk.Variant.OneSM)
    two = sk.default_cost_params(sk.DType.Float16, sk.Variant.TwoSM)
    wide = sk.default_cost_params(sk.DType.BFloat16, sk.Variant.TwoSMWide)
    f64 = sk.default_cost_params(sk.DType.Float64, sk.Variant.Auto)
    assert (one.cluster_min_iters, one.cluster_kernel) == (8.0, 1.0)
    assert (two.cluster_min_iters, two.cluster_kernel) == (16.0, 2.0)
    assert wide.cluster_min_iters == 0.0 and f64.cluster_min_iters == 0.0
    # without a device the rule has no capacity to check and the model decides
    import torch

    if not torch.cuda.is_available():
        blk = sk.kernel_blocking(sk.DType.BFloat16, sk.Variant.OneSM)
        a = sk.auto_stream_k(sk.GemmProblem(128, 8192, 8192), blk, 148)
        assert a.strategy != sk.Strategy.FixedSplit
