"""The C-ABI library loads on a GPU-less host, exports every symbol include/skb200.h
declares, and its host-side validation mirrors the reference's error behaviour
(no device calls here)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "skb200.h")).read()
    return sorted(set(re.findall(r"\b(sk_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(sk):
    lib = C.CDLL(sk.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 16
    for s in syms:
        assert hasattr(lib, s), s


def test_only_sk_symbols_exported(sk):
    import subprocess

    out = subprocess.run(["nm", "-D", "--defined-only", sk.LIB_PATH], capture_output=True,
                         text=True).stdout
    names = [l.split()[-1] for l in out.splitlines() if l.strip()]
    assert names and all(n.startswith("sk_") for n in names), names[:10]


def test_sass_is_tcgen05_and_tma(sk):
    """The shipped kernels are Blackwell-native: UTC*MMA (tcgen05.mma), LDTM
    (tcgen05.ld), UTMALDG/UTMASTG (TMA) in the sm_100a cubin."""
    import shutil
    import subprocess

    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump missing")
    sass = subprocess.run([exe, "-sass", sk.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in sass
    for mnem in ("UTCHMMA", "LDTM", "UTMALDG", "UTMASTG"):
        assert mnem in sass, mnem
    assert "HMMA" not in sass.replace("UTCHMMA", "")  # no legacy mma.sync path for 16-bit


def test_status_strings_and_version(sk):
    lib = sk.lib()
    assert lib.sk_abi_version() == 5  # v2 SK_EXPLICIT, v3 tile_group, v4 2SM_WIDE, v5 cluster fixup
    for code in range(7):
        assert lib.sk_status_string(code)


def test_kernel_blocking_per_precision(sk):
    b = sk.kernel_blocking(sk.DType.BFloat16)  # AUTO -> 2-SM
    assert (b.blk_m, b.blk_n, b.blk_k) == (256, 256, 64)
    b = sk.kernel_blocking(sk.DType.Float16, sk.Variant.OneSM)
    assert (b.blk_m, b.blk_n, b.blk_k) == (128, 256, 64)
    b = sk.kernel_blocking(sk.DType.Float64)
    assert (b.blk_m, b.blk_n, b.blk_k) == (64, 64, 16)
    b = sk.kernel_blocking(sk.DType.BFloat16, sk.Variant.TwoSMWide)
    assert (b.blk_m, b.blk_n, b.blk_k) == (256, 512, 64)
    # AUTO with an explicit 1-SM blocking resolves to the 1-SM kernel
    d = _desc(sk, 512, 512, 512, (128, 256, 64), strategy=0, param=1)
    n = C.c_size_t()
    assert sk.lib().sk_workspace_size(C.byref(d), C.byref(n)) == 0


def test_wide_variant_workspace(sk):
    """SK_VARIANT_2SM_WIDE (256x512x64): AUTO resolves it from the blocking, each
    Stream-K unit's slab is 2 ranks x 128 x 512 fp32, and a 256x256 blocking
    under the wide variant is refused (the tile names the kernel)."""
    lib = sk.lib()
    n = C.c_size_t()
    d = _desc(sk, 8192, 8192, 8192, (256, 512, 64), strategy=2, param=74)
    assert lib.sk_workspace_size(C.byref(d), C.byref(n)) == 0  # AUTO -> wide
    assert n.value >= 74 * 2 * 128 * 512 * 4
    d.variant = int(sk.Variant.TwoSMWide)
    assert lib.sk_workspace_size(C.byref(d), C.byref(n)) == 0
    d = _desc(sk, 8192, 8192, 8192, (256, 256, 64), strategy=2, param=74)
    d.variant = int(sk.Variant.TwoSMWide)
    assert lib.sk_workspace_size(C.byref(d), C.byref(n)) == sk.SK_EUNSUPPORTED


def _desc(sk, m, n, k, blk, strategy=2, param=148, ab=3):
    d = sk.sk_gemm_desc()
    d.problem = sk.sk_problem(m, n, k, 1.0, 0.0)
    d.blocking = sk.sk_blocking(*blk)
    d.strategy = strategy
    d.param = param
    d.ab_type = ab
    d.lda, d.ldb, d.ldc = k, n, n
    return d


def test_workspace_size(sk):
    lib = sk.lib()
    n = C.c_size_t()
    d = _desc(sk, 8192, 8192, 8192, (128, 256, 64), strategy=2, param=148)
    assert lib.sk_workspace_size(C.byref(d), C.byref(n)) == 0
    assert n.value >= 148 * 128 * 256 * 4  # one fp32 slab per SK unit
    d = _desc(sk, 8192, 8192, 8192, (128, 256, 64), strategy=0, param=1)
    assert lib.sk_workspace_size(C.byref(d), C.byref(n)) == 0
    assert n.value < 4096  # data-parallel: no partials


def test_unsupported_and_invalid(sk):
    lib = sk.lib()
    n = C.c_size_t()
    d = _desc(sk, 256, 256, 256, (128, 128, 64))
    assert lib.sk_workspace_size(C.byref(d), C.byref(n)) == sk.SK_EUNSUPPORTED
    assert b"blocking" in lib.sk_last_error()
    d = _desc(sk, 0, 256, 256, (128, 256, 64))
    assert lib.sk_workspace_size(C.byref(d), C.byref(n)) == sk.SK_EINVAL
    d = _desc(sk, 256, 256, 256, (128, 256, 64), strategy=9)
    assert lib.sk_workspace_size(C.byref(d), C.byref(n)) == sk.SK_EINVAL
    d = _desc(sk, 256, 256, 256, (128, 256, 64), ab=0)  # int64 has no device kernel
    assert lib.sk_workspace_size(C.byref(d), C.byref(n)) == sk.SK_EUNSUPPORTED
    # sk_gemm rejects misaligned leading dimensions before touching the device
    d = _desc(sk, 256, 250, 256, (128, 256, 64))
    d.A = d.B = d.C = 1 << 20
    ws = C.c_size_t(1 << 30)
    assert lib.sk_gemm(C.byref(d), C.c_void_p(1 << 21), ws, None) == sk.SK_EUNSUPPORTED


def test_execute_shape_check(sk):
    a = sk.stream_k(sk.GemmProblem(8, 8, 8), sk.kernel_blocking(), 2)
    with pytest.raises(ValueError):
        sk.execute(a, np.zeros((8, 7), np.float32), np.zeros((8, 8), np.float32))
