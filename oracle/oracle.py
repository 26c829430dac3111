"""ctypes front end for the parity checkers -- TEST INFRASTRUCTURE ONLY.

Two checkers with the same Python surface:

* ``Oracle("port")``       -> oracle/libskoracle.so, our C restatement
  (oracle/skoracle.c, each function cites the reference file:line it follows);
* ``Oracle("reference")``  -> oracle/_ref/libstreamk_ref.so, the reference's own
  sources compiled by oracle/Makefile plus oracle/ref_driver.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this
module.  The product (paper_2301_03598_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "libskoracle.so")
REF_SO = os.path.join(HERE, "_ref", "libstreamk_ref.so")
REF_ACCEPTANCE = os.path.join(HERE, "_ref", "acceptance")
REF_SRC = "/root/reference/proj"

STRATEGIES = {
    "data_parallel": 0,
    "fixed_split": 1,
    "stream_k": 2,
    "dp_one_tile_sk": 3,
    "two_tile_sk_dp": 4,
}

_i64 = C.c_int64
_p64 = C.POINTER(C.c_int64)


def build(with_ref: bool | None = None) -> None:
    """Build the checkers (make -C oracle).  The reference build needs
    /root/reference, which only exists in the dev container."""
    if with_ref is None:
        with_ref = os.path.isdir(REF_SRC)
    targets = ["oracle"] + (["ref"] if with_ref else [])
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def have_reference() -> bool:
    return os.path.exists(REF_SO)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: status {code}")
        self.code = code


class Oracle:
    """Uniform numpy API over either checker library."""

    def __init__(self, kind: str = "port"):
        self.kind = kind
        if kind == "port":
            if not os.path.exists(PORT_SO):
                build(with_ref=False)
            self.lib = C.CDLL(PORT_SO)
            self.pre = "skor_"
        elif kind == "reference":
            if not os.path.exists(REF_SO):
                build(with_ref=True)
            self.lib = C.CDLL(REF_SO)
            self.pre = "ref_"
        else:
            raise ValueError(kind)

    def _f(self, name):
        return getattr(self.lib, self.pre + name)

    # ---- schedule -----------------------------------------------------------
    def tile_grid(self, m, n, k, bm, bn, bk):
        out = np.zeros(5, np.int64)
        st = self._f("tile_grid")(_i64(m), _i64(n), _i64(k), _i64(bm), _i64(bn), _i64(bk), _ptr(out))
        if st:
            raise OracleError(st, "tile_grid")
        return tuple(int(x) for x in out)

    def iter_to_coords(self, m, n, k, bm, bn, bk, i):
        tile, local = _i64(), _i64()
        if self.kind == "port":
            grid = np.array(self.tile_grid(m, n, k, bm, bn, bk), np.int64)
            st = self.lib.skor_iter_to_coords(_ptr(grid), _i64(i), C.byref(tile), C.byref(local))
        else:
            st = self.lib.ref_iter_to_coords(_i64(m), _i64(n), _i64(k), _i64(bm), _i64(bn),
                                             _i64(bk), _i64(i), C.byref(tile), C.byref(local))
        if st:
            raise OracleError(st, "iter_to_coords")
        return tile.value, local.value

    def schedule(self, strategy, m, n, k, bm, bn, bk, param=1) -> np.ndarray:
        """[g][2] int64 (begin, end) table; row index == cta_id."""
        s = STRATEGIES[strategy] if isinstance(strategy, str) else int(strategy)
        g = _i64()
        f = self._f("schedule")
        args = [C.c_int(s), _i64(m), _i64(n), _i64(k), _i64(bm), _i64(bn), _i64(bk), _i64(param)]
        st = f(*args, C.byref(g), C.c_void_p(), _i64(0))
        if st:
            raise OracleError(st, "schedule")
        out = np.zeros((g.value, 2), np.int64)
        st = f(*args, C.byref(g), _ptr(out), _i64(g.value))
        if st:
            raise OracleError(st, "schedule")
        return out

    def fixup_peers(self, strategy, m, n, k, bm, bn, bk, param=1):
        """CSR (offsets[t+1], ids[nnz]) of fixup_peers_of."""
        t = self.tile_grid(m, n, k, bm, bn, bk)[2]
        offsets = np.zeros(t + 1, np.int64)
        nnz = _i64()
        if self.kind == "port":
            ranges = self.schedule(strategy, m, n, k, bm, bn, bk, param)
            ipt = self.tile_grid(m, n, k, bm, bn, bk)[3]
            g = ranges.shape[0]
            st = self.lib.skor_fixup_peers(_ptr(ranges), _i64(g), _i64(ipt), _i64(t), _ptr(offsets),
                                           C.c_void_p(), _i64(0), C.byref(nnz))
            ids = np.zeros(max(nnz.value, 1), np.int64)
            st = st or self.lib.skor_fixup_peers(_ptr(ranges), _i64(g), _i64(ipt), _i64(t),
                                                 _ptr(offsets), _ptr(ids), _i64(ids.size), C.byref(nnz))
        else:
            s = STRATEGIES[strategy] if isinstance(strategy, str) else int(strategy)
            args = [C.c_int(s), _i64(m), _i64(n), _i64(k), _i64(bm), _i64(bn), _i64(bk), _i64(param)]
            st = self.lib.ref_fixup_peers(*args, _ptr(offsets), C.c_void_p(), _i64(0), C.byref(nnz))
            ids = np.zeros(max(nnz.value, 1), np.int64)
            st = st or self.lib.ref_fixup_peers(*args, _ptr(offsets), _ptr(ids), _i64(ids.size),
                                                C.byref(nnz))
        if st:
            raise OracleError(st, "fixup_peers")
        return offsets, ids[: nnz.value]

    def quantization_efficiency(self, t, p) -> float:
        out = C.c_double()
        st = self._f("quantization_efficiency")(_i64(t), _i64(p), C.byref(out))
        if st:
            raise OracleError(st, "quantization_efficiency")
        return out.value

    # ---- data ---------------------------------------------------------------
    def random_matrix(self, rows, cols, seed, dtype="float32") -> np.ndarray:
        suf, npdt = {"int64": ("i64", np.int64), "float32": ("f32", np.float32),
                     "float64": ("f64", np.float64)}[dtype]
        out = np.empty((rows, cols), npdt)
        self._f("random_matrix_" + suf)(_i64(rows), _i64(cols), C.c_uint64(seed & (2**64 - 1)),
                                        _ptr(out))
        return out

    def gemm_reference(self, A: np.ndarray, B: np.ndarray, bm, bn, bk) -> np.ndarray:
        suf = {np.dtype(np.int64): "i64", np.dtype(np.float32): "f32",
               np.dtype(np.float64): "f64"}[A.dtype]
        m, k = A.shape
        n = B.shape[1]
        A = np.ascontiguousarray(A)
        B = np.ascontiguousarray(B)
        Cm = np.empty((m, n), A.dtype)
        st = self._f("gemm_reference_" + suf)(_i64(m), _i64(n), _i64(k), _i64(bm), _i64(bn), _i64(bk),
                                              _ptr(A), _ptr(B), _ptr(Cm))
        if st:
            raise OracleError(st, "gemm_reference")
        return Cm

    def execute(self, strategy, param, A: np.ndarray, B: np.ndarray, bm, bn, bk,
                threads: int = 1) -> np.ndarray:
        """C = execute(strategy(problem, blocking, param), A, B) of the checker."""
        suf = {np.dtype(np.int64): "i64", np.dtype(np.float32): "f32",
               np.dtype(np.float64): "f64"}[A.dtype]
        m, k = A.shape
        n = B.shape[1]
        A = np.ascontiguousarray(A)
        B = np.ascontiguousarray(B)
        Cm = np.empty((m, n), A.dtype)
        if self.kind == "port":
            ranges = self.schedule(strategy, m, n, k, bm, bn, bk, param)
            st = getattr(self.lib, "skor_execute_" + suf)(
                _ptr(ranges), _i64(ranges.shape[0]), _i64(m), _i64(n), _i64(k), _i64(bm), _i64(bn),
                _i64(bk), _ptr(A), _ptr(B), _ptr(Cm))
        else:
            s = STRATEGIES[strategy] if isinstance(strategy, str) else int(strategy)
            st = getattr(self.lib, "ref_execute_" + suf)(
                C.c_int(s), _i64(param), _i64(m), _i64(n), _i64(k), _i64(bm), _i64(bn), _i64(bk),
                _ptr(A), _ptr(B), _ptr(Cm), C.c_int(threads))
        if st:
            raise OracleError(st, "execute")
        return Cm

    def execute_ranges(self, ranges: np.ndarray, A: np.ndarray, B: np.ndarray, bm, bn, bk,
                       threads: int = 1) -> np.ndarray:
        """C = execute(assignment with this [g][2] range table, A, B) of the checker
        (the reference parses it with its own from_text).  threads = 1 keeps the
        reference's descending dispatch sequential: safe whenever every fixup wait
        points to a higher id."""
        suf = {np.dtype(np.int64): "i64", np.dtype(np.float32): "f32",
               np.dtype(np.float64): "f64"}[A.dtype]
        m, k = A.shape
        n = B.shape[1]
        A = np.ascontiguousarray(A)
        B = np.ascontiguousarray(B)
        ranges = np.ascontiguousarray(ranges, dtype=np.int64).reshape(-1, 2)
        Cm = np.empty((m, n), A.dtype)
        fn = ("skor_execute_" if self.kind == "port" else "ref_execute_ranges_") + suf
        args = [_ptr(ranges), _i64(ranges.shape[0]), _i64(m), _i64(n), _i64(k), _i64(bm), _i64(bn),
                _i64(bk), _ptr(A), _ptr(B), _ptr(Cm)]
        if self.kind != "port":
            args.append(C.c_int(threads))
        st = getattr(self.lib, fn)(*args)
        if st:
            raise OracleError(st, "execute_ranges")
        return Cm

    # ---- reference-only text form -----------------------------------------
    def to_text(self, strategy, m, n, k, bm, bn, bk, param=1) -> str:
        if self.kind != "reference":
            raise NotImplementedError("to_text lives in the reference driver only")
        s = STRATEGIES[strategy] if isinstance(strategy, str) else int(strategy)
        n_ = _i64()
        args = [C.c_int(s), _i64(m), _i64(n), _i64(k), _i64(bm), _i64(bn), _i64(bk), _i64(param)]
        st = self.lib.ref_to_text(*args, C.c_void_p(), _i64(0), C.byref(n_))
        buf = C.create_string_buffer(n_.value + 1)
        st = st or self.lib.ref_to_text(*args, buf, _i64(n_.value + 1), C.byref(n_))
        if st:
            raise OracleError(st, "to_text")
        return buf.value.decode()


def verify(Cm: np.ndarray, Cref: np.ndarray, k: int, eps: float | None = None):
    """executor.hpp:217-239 semantics (see skoracle.c skor_verify).
    eps=None -> exact (int64 rule).  Returns (pass, max_abs, max_rel)."""
    lib = C.CDLL(PORT_SO) if os.path.exists(PORT_SO) else (build(False) or C.CDLL(PORT_SO))
    c = np.ascontiguousarray(Cm, dtype=np.float64).ravel()
    r = np.ascontiguousarray(Cref, dtype=np.float64).ravel()
    if c.size != r.size:
        raise ValueError("verify: shape mismatch")
    ma, mr = C.c_double(), C.c_double()
    ok = lib.skor_verify(_ptr(c), _ptr(r), _i64(c.size), _i64(k), C.c_double(eps or 0.0),
                         C.c_int(1 if eps is None else 0), C.byref(ma), C.byref(mr))
    return bool(ok), ma.value, mr.value


def corpus(seed: int, count: int, lo: int = 128, hi: int = 8192) -> np.ndarray:
    """[count][4] uint64 (m, n, k, matrix_seed) in run_sweep order (sweep.cpp:79-86)."""
    lib = C.CDLL(PORT_SO) if os.path.exists(PORT_SO) else (build(False) or C.CDLL(PORT_SO))
    out = np.zeros((count, 4), np.uint64)
    lib.skor_corpus(C.c_uint64(seed), _i64(count), _i64(lo), _i64(hi), _ptr(out))
    return out


def ref_run_sweep(seed: int, count: int, lo: int, hi: int, strategies, p: int, split: int,
                  blk) -> str:
    """The reference's run_sweep CSV text (sweep.cpp:75-112), unmeasured."""
    lib = C.CDLL(REF_SO)
    codes = np.array([STRATEGIES[s] if isinstance(s, str) else int(s) for s in strategies], np.int32)
    n = _i64()
    args = [C.c_uint64(seed), _i64(count), _i64(lo), _i64(hi), _ptr(codes), C.c_int(codes.size),
            _i64(p), _i64(split), _i64(blk[0]), _i64(blk[1]), _i64(blk[2])]
    st = lib.ref_run_sweep(*args, C.c_void_p(), _i64(0), C.byref(n))
    buf = C.create_string_buffer(n.value + 1)
    st = st or lib.ref_run_sweep(*args, buf, _i64(n.value + 1), C.byref(n))
    if st:
        raise OracleError(st, "ref_run_sweep")
    return buf.value.decode()


def ref_simulate(strategy, param, m, n, k, bm, bn, bk, p, params=None):
    """(makespan, utilization) of the reference's simulate (simulate.cpp:23-80)."""
    lib = C.CDLL(REF_SO)
    s = STRATEGIES[strategy] if isinstance(strategy, str) else int(strategy)
    a, b, c, d = (params if params is not None else (0.0, 0.0, 1.0, 0.0))
    ms, ut = C.c_double(), C.c_double()
    st = lib.ref_simulate(C.c_int(s), _i64(param), _i64(m), _i64(n), _i64(k), _i64(bm), _i64(bn),
                          _i64(bk), _i64(p), C.c_int(params is not None), C.c_double(a),
                          C.c_double(b), C.c_double(c), C.c_double(d), C.byref(ms), C.byref(ut))
    if st:
        raise OracleError(st, "ref_simulate")
    return ms.value, ut.value


def ref_corpus_dims(seed: int, count: int, lo: int = 128, hi: int = 8192) -> np.ndarray:
    lib = C.CDLL(REF_SO)
    out = np.zeros((count, 3), np.int64)
    st = lib.ref_corpus_dims(C.c_uint64(seed), _i64(count), _i64(lo), _i64(hi), _ptr(out))
    if st:
        raise OracleError(st, "ref_corpus_dims")
    return out
