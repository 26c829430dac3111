"""paper_2301_03598_b200 -- B200-native Stream-K GEMM behind the reference's API.

Python mirror of the reference core's public surface (/root/reference/proj,
core/include/streamk/*.hpp), implemented entirely by the C-ABI library
``_lib/libskb200.so`` (include/skb200.h): schedules are computed by its C++
closed forms, GEMMs run in its hand-written sm_100a kernels.  There is no
Python or CPU fallback: if the library is missing every entry point raises.

    reference                               here
    ---------------------------------------------------------------------------
    GemmProblem / BlockingFactors            GemmProblem / BlockingFactors
    tile_grid / iter_to_coords               tile_grid / iter_to_coords
    data_parallel / fixed_split /            data_parallel / fixed_split /
      stream_k / hybrid                        stream_k / hybrid
    fixup_peers_of / quantization_efficiency fixup_peers_of / quantization_efficiency
    to_text / from_text                      to_text / from_text
    execute<T>(a, A, B, threads)             execute(a, A, B)  (host arrays in/out)
                                             Gemm(a, ...).run(A, B, C) (device tensors)

Exceptions follow the reference: std::invalid_argument -> ValueError,
std::out_of_range -> IndexError, std::logic_error (double signal) ->
ProtocolError (a RuntimeError).
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SKB200_LIB: load an alternative build of the library (kernel experiments)
LIB_PATH = os.environ.get("SKB200_LIB") or os.path.join(_HERE, "_lib", "libskb200.so")

__all__ = [
    "DType", "Strategy", "HybridVariant", "Variant", "GemmProblem", "BlockingFactors", "TileGrid",
    "TileCoords", "CtaRange", "WorkAssignment", "tile_grid", "iter_to_coords", "data_parallel",
    "fixed_split", "stream_k", "hybrid", "fixup_peers_of", "quantization_efficiency", "to_text",
    "from_text", "kernel_blocking", "execute", "Gemm", "ProtocolError", "UnsupportedError",
    "CudaError", "lib", "corpus", "simulate", "random_matrix_device", "reload_env",
]


# ----------------------------------------------------------------------------- errors
class ProtocolError(RuntimeError):
    """std::logic_error in the reference: a fixup flag signalled twice (or the
    device wait watchdog fired)."""


class UnsupportedError(RuntimeError):
    """Valid for the reference, not for this device kernel (tile config, alignment)."""


class CudaError(RuntimeError):
    pass


SK_OK, SK_EINVAL, SK_EUNSUPPORTED, SK_ECUDA, SK_EPROTOCOL, SK_ERANGE, SK_ECAPACITY = range(7)


# ----------------------------------------------------------------------------- C ABI
class sk_problem(C.Structure):
    _fields_ = [("m", C.c_int64), ("n", C.c_int64), ("k", C.c_int64), ("alpha", C.c_double),
                ("beta", C.c_double)]


class sk_blocking(C.Structure):
    _fields_ = [("blk_m", C.c_int64), ("blk_n", C.c_int64), ("blk_k", C.c_int64)]


class sk_tile_grid_t(C.Structure):
    _fields_ = [("tiles_m", C.c_int64), ("tiles_n", C.c_int64), ("total_tiles", C.c_int64),
                ("iters_per_tile", C.c_int64), ("total_iters", C.c_int64)]


class sk_gemm_desc(C.Structure):
    _fields_ = [
        ("problem", sk_problem), ("blocking", sk_blocking), ("strategy", C.c_int32),
        ("ab_type", C.c_int32), ("param", C.c_int64), ("variant", C.c_int32),
        ("num_ctas", C.c_int32), ("A", C.c_void_p), ("lda", C.c_int64), ("B", C.c_void_p),
        ("ldb", C.c_int64), ("C", C.c_void_p), ("ldc", C.c_int64),
        ("trace", C.c_void_p), ("cta_clocks", C.c_void_p), ("events", C.c_void_p),
        ("ranges", C.c_void_p), ("num_ranges", C.c_int64),
        ("tile_group", C.c_int32), ("reserved0", C.c_int32),
    ]


class sk_sim_params(C.Structure):
    _fields_ = [("a", C.c_double), ("b", C.c_double), ("c", C.c_double), ("d", C.c_double)]


SK_EXPLICIT = 5  # sk_strategy for an arbitrary range table (skb200.h)


_P = C.POINTER
_lib: Optional[C.CDLL] = None

_SIGS = {
    "sk_status_string": (C.c_char_p, [C.c_int]),
    "sk_last_error": (C.c_char_p, []),
    "sk_abi_version": (C.c_int, []),
    "sk_tile_grid": (C.c_int, [_P(sk_problem), _P(sk_blocking), _P(sk_tile_grid_t)]),
    "sk_iter_to_coords": (C.c_int, [_P(sk_tile_grid_t), C.c_int64, _P(C.c_int64), _P(C.c_int64)]),
    "sk_schedule": (C.c_int, [_P(sk_problem), _P(sk_blocking), C.c_int, C.c_int64, _P(C.c_int64),
                              C.c_void_p, C.c_int64]),
    "sk_fixup_peers": (C.c_int, [_P(sk_problem), _P(sk_blocking), C.c_int, C.c_int64, C.c_void_p,
                                 C.c_void_p, C.c_int64, _P(C.c_int64)]),
    "sk_quantization_efficiency": (C.c_int, [C.c_int64, C.c_int64, _P(C.c_double)]),
    "sk_kernel_blocking": (C.c_int, [C.c_int, C.c_int, _P(sk_blocking)]),
    "sk_workspace_size": (C.c_int, [_P(sk_gemm_desc), _P(C.c_size_t)]),
    "sk_workspace_init": (C.c_int, [C.c_void_p, C.c_size_t, C.c_void_p]),
    "sk_workspace_check": (C.c_int, [C.c_void_p, C.c_void_p]),
    "sk_trace_size": (C.c_int, [_P(sk_gemm_desc), _P(C.c_int64)]),
    "sk_timeline_size": (C.c_int, [_P(sk_gemm_desc), _P(C.c_int64), _P(C.c_int64)]),
    "sk_gemm": (C.c_int, [_P(sk_gemm_desc), C.c_void_p, C.c_size_t, C.c_void_p]),
    "sk_device_topology": (C.c_int, [C.c_int, C.c_void_p, C.c_int32, _P(C.c_int32), _P(C.c_int32)]),
    "sk_persistent_order": (C.c_int, [_P(sk_gemm_desc), C.c_int64, C.c_int64, C.c_void_p, C.c_int64,
                                      _P(C.c_int64)]),
    "sk_tile_block": (C.c_int, [_P(sk_gemm_desc), C.c_int64, _P(C.c_int64), _P(C.c_int64)]),
    "sk_execute": (C.c_int, [_P(sk_problem), _P(sk_blocking), C.c_int, C.c_int64, C.c_int, C.c_int,
                             C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32]),
    "sk_execute_ranges": (C.c_int, [_P(sk_problem), _P(sk_blocking), C.c_void_p, C.c_int64, C.c_int,
                                    C.c_int, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_int32]),
    "sk_fixup_peers_ranges": (C.c_int, [_P(sk_problem), _P(sk_blocking), C.c_void_p, C.c_int64,
                                        C.c_void_p, C.c_void_p, C.c_int64, _P(C.c_int64)]),
    "sk_execute_release": (None, []),
    "sk_corpus": (C.c_int, [C.c_uint64, C.c_int64, C.c_int64, C.c_int64, C.c_void_p]),
    "sk_default_cost_params": (C.c_int, [C.c_int, C.c_int, C.c_void_p]),
    "sk_predict_time": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, _P(C.c_double)]),
    "sk_select_grid_size": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, _P(C.c_int64)]),
    "sk_calibrate": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p]),
    "sk_predict_schedule": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.c_int64,
                                      _P(C.c_double)]),
    "sk_select_schedule": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, _P(C.c_int32),
                                     _P(C.c_int64)]),
    "sk_save_matrix": (C.c_int, [C.c_char_p, C.c_int, C.c_int64, C.c_int64, C.c_void_p]),
    "sk_load_matrix_header": (C.c_int, [C.c_char_p, _P(C.c_int), _P(C.c_int64), _P(C.c_int64)]),
    "sk_load_matrix": (C.c_int, [C.c_char_p, C.c_int, C.c_int64, C.c_int64, C.c_void_p]),
    "sk_io_error": (C.c_char_p, []),
    "sk_random_matrix": (C.c_int, [C.c_int, C.c_int32, C.c_uint64, C.c_int64, C.c_int64, C.c_int,
                                   C.c_void_p, C.c_int64, C.c_void_p]),
    "sk_simulate": (C.c_int, [_P(sk_problem), _P(sk_blocking), C.c_int, C.c_int64, C.c_void_p,
                              C.c_int64, C.c_int64, C.c_void_p, _P(C.c_double), _P(C.c_double),
                              C.c_void_p, C.c_int64, _P(C.c_int64)]),
    "sk_reload_env": (None, []),
    "sk_persistent_capacity": (C.c_int, [C.c_int, C.c_int, C.c_int32, _P(C.c_int32)]),
    "sk_cluster_capacity": (C.c_int, [C.c_int, C.c_int32, C.c_int32, _P(C.c_int32)]),
}


def lib() -> C.CDLL:
    """Load libskb200.so (built by paper_2301_03598_b200.build / __graft_entry__.build)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2301_03598_b200.build`"
                              " (there is no CPU fallback)")
        h = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            if os.environ.get("SKB200_LIB") and not hasattr(h, name):
                continue  # an older experimental build may lack newer entry points
            f = getattr(h, name)
            f.restype = res
            f.argtypes = args
        _lib = h
    return _lib


def _check(st: int, what: str = "") -> None:
    if st == SK_OK:
        return
    detail = lib().sk_last_error().decode()
    msg = f"{what}: {detail}" if what else detail
    if st == SK_EINVAL:
        raise ValueError(msg)
    if st == SK_ERANGE:
        raise IndexError(msg)
    if st == SK_EPROTOCOL:
        raise ProtocolError(msg)
    if st == SK_EUNSUPPORTED:
        raise UnsupportedError(msg)
    if st == SK_ECUDA:
        raise CudaError(msg)
    raise RuntimeError(f"{msg} (status {st})")


# ----------------------------------------------------------------------------- domain (types.hpp)
class DType(enum.IntEnum):
    Int64 = 0
    Float32 = 1
    Float64 = 2
    BFloat16 = 3
    Float16 = 4


class Strategy(enum.IntEnum):  # types.hpp:70
    DataParallel = 0
    FixedSplit = 1
    StreamK = 2
    DpOneTileSk = 3
    TwoTileSkDp = 4


class HybridVariant(enum.IntEnum):  # decompose.hpp:9
    DpOneTileSk = 3
    TwoTileSkDp = 4


class Variant(enum.IntEnum):
    Auto = 0
    OneSM = 1
    TwoSM = 2
    TwoSMWide = 3  # 256x512x64 (two N=256 MMAs per k step), see skb200.h


_STRATEGY_NAMES = {
    Strategy.DataParallel: "data_parallel", Strategy.FixedSplit: "fixed_split",
    Strategy.StreamK: "stream_k", Strategy.DpOneTileSk: "dp_one_tile_sk",
    Strategy.TwoTileSkDp: "two_tile_sk_dp",
}


def strategy_name(s: Strategy) -> str:  # types.cpp:64-73
    return _STRATEGY_NAMES[Strategy(s)]


@dataclass(frozen=True)
class GemmProblem:  # types.hpp:20-27
    m: int = 1
    n: int = 1
    k: int = 1
    alpha: float = 1.0
    beta: float = 0.0
    dtype: DType = DType.Float32

    def _c(self) -> sk_problem:
        return sk_problem(self.m, self.n, self.k, self.alpha, self.beta)


@dataclass(frozen=True)
class BlockingFactors:  # types.hpp:30-34
    blk_m: int = 1
    blk_n: int = 1
    blk_k: int = 1

    def _c(self) -> sk_blocking:
        return sk_blocking(self.blk_m, self.blk_n, self.blk_k)


@dataclass(frozen=True)
class TileGrid:  # types.hpp:41-47
    tiles_m: int = 0
    tiles_n: int = 0
    total_tiles: int = 0
    iters_per_tile: int = 0
    total_iters: int = 0

    def _c(self) -> sk_tile_grid_t:
        return sk_tile_grid_t(self.tiles_m, self.tiles_n, self.total_tiles, self.iters_per_tile,
                              self.total_iters)


@dataclass(frozen=True)
class TileCoords:
    tile_idx: int
    local_iter: int


@dataclass(frozen=True)
class CtaRange:  # types.hpp:61-68
    cta_id: int
    iter_begin: int
    iter_end: int

    def length(self) -> int:
        return self.iter_end - self.iter_begin

    def empty(self) -> bool:
        return self.iter_end == self.iter_begin


@dataclass
class WorkAssignment:  # types.hpp:76-84
    strategy: Strategy = Strategy.DataParallel
    grid_size: int = 0
    split: int = 1
    problem: GemmProblem = field(default_factory=GemmProblem)
    blocking: BlockingFactors = field(default_factory=BlockingFactors)
    grid: TileGrid = field(default_factory=TileGrid)
    ranges: List[CtaRange] = field(default_factory=list)
    # The decomposition knob the closed-form device scheduler needs (s, g or p).
    param: int = 1

    def range_table(self) -> np.ndarray:
        return np.array([[r.iter_begin, r.iter_end] for r in self.ranges], np.int64).reshape(-1, 2)


def tile_grid(problem: GemmProblem, blocking: BlockingFactors) -> TileGrid:  # types.cpp:45-55
    out = sk_tile_grid_t()
    _check(lib().sk_tile_grid(C.byref(problem._c()), C.byref(blocking._c()), C.byref(out)),
           "tile_grid")
    return TileGrid(out.tiles_m, out.tiles_n, out.total_tiles, out.iters_per_tile, out.total_iters)


def iter_to_coords(grid: TileGrid, i: int) -> TileCoords:  # types.cpp:57-62
    t, l = C.c_int64(), C.c_int64()
    _check(lib().sk_iter_to_coords(C.byref(grid._c()), i, C.byref(t), C.byref(l)),
           "iter_to_coords")
    return TileCoords(t.value, l.value)


def _schedule_table(problem, blocking, strategy: Strategy, param: int) -> np.ndarray:
    g = C.c_int64()
    p, b = problem._c(), blocking._c()
    _check(lib().sk_schedule(C.byref(p), C.byref(b), int(strategy), param, C.byref(g), None, 0),
           strategy_name(strategy))
    tbl = np.zeros((g.value, 2), np.int64)
    _check(lib().sk_schedule(C.byref(p), C.byref(b), int(strategy), param, C.byref(g),
                             tbl.ctypes.data_as(C.c_void_p), g.value), strategy_name(strategy))
    return tbl


def _assignment(strategy: Strategy, problem: GemmProblem, blocking: BlockingFactors,
                param: int) -> WorkAssignment:
    tbl = _schedule_table(problem, blocking, strategy, param)
    return WorkAssignment(
        strategy=strategy, grid_size=tbl.shape[0],
        split=param if strategy == Strategy.FixedSplit else 1, problem=problem, blocking=blocking,
        grid=tile_grid(problem, blocking),
        ranges=[CtaRange(i, int(b), int(e)) for i, (b, e) in enumerate(tbl)], param=param)


def data_parallel(problem: GemmProblem, blocking: BlockingFactors) -> WorkAssignment:
    return _assignment(Strategy.DataParallel, problem, blocking, 1)  # decompose.cpp:38-48


def fixed_split(problem: GemmProblem, blocking: BlockingFactors, s: int) -> WorkAssignment:
    return _assignment(Strategy.FixedSplit, problem, blocking, s)  # decompose.cpp:50-69


def stream_k(problem: GemmProblem, blocking: BlockingFactors, g: int) -> WorkAssignment:
    return _assignment(Strategy.StreamK, problem, blocking, g)  # decompose.cpp:71-79


def hybrid(problem: GemmProblem, blocking: BlockingFactors, p: int,
           variant: HybridVariant) -> WorkAssignment:  # decompose.cpp:81-121
    return _assignment(Strategy(int(variant)), problem, blocking, p)


def fixup_peers_of(a: WorkAssignment) -> List[List[int]]:  # decompose.cpp:123-136
    off, ids = _peers_csr(a)
    return [ids[off[t]:off[t + 1]].tolist() for t in range(a.grid.total_tiles)]


def _explicit_table(a: WorkAssignment) -> np.ndarray:
    """The [g][2] range table of an assignment the closed forms do not produce
    (param == 0), for SK_EXPLICIT.  execute<T> indexes ranges by position while
    fixup_peers_of keys peers by cta_id (executor.hpp:148, decompose.cpp:130),
    so a table whose ids differ from their positions has no consistent meaning."""
    if any(r.cta_id != i for i, r in enumerate(a.ranges)) or len(a.ranges) != a.grid_size:
        raise ValueError("execute: range table cta_ids must be 0..g-1 in order")
    return np.ascontiguousarray(a.range_table(), dtype=np.int64)


def _peers_csr(a: WorkAssignment):
    p, b = a.problem._c(), a.blocking._c()
    off = np.zeros(a.grid.total_tiles + 1, np.int64)
    nnz = C.c_int64()
    if a.param == 0:  # explicit table
        tbl = _explicit_table(a)
        tp = tbl.ctypes.data_as(C.c_void_p)
        _check(lib().sk_fixup_peers_ranges(C.byref(p), C.byref(b), tp, tbl.shape[0],
                                           off.ctypes.data_as(C.c_void_p), None, 0, C.byref(nnz)),
               "fixup_peers_of")
        ids = np.zeros(max(nnz.value, 1), np.int64)
        _check(lib().sk_fixup_peers_ranges(C.byref(p), C.byref(b), tp, tbl.shape[0],
                                           off.ctypes.data_as(C.c_void_p),
                                           ids.ctypes.data_as(C.c_void_p), ids.size, C.byref(nnz)),
               "fixup_peers_of")
        return off, ids[: nnz.value]
    _check(lib().sk_fixup_peers(C.byref(p), C.byref(b), int(a.strategy), a.param,
                                off.ctypes.data_as(C.c_void_p), None, 0, C.byref(nnz)),
           "fixup_peers_of")
    ids = np.zeros(max(nnz.value, 1), np.int64)
    _check(lib().sk_fixup_peers(C.byref(p), C.byref(b), int(a.strategy), a.param,
                                off.ctypes.data_as(C.c_void_p), ids.ctypes.data_as(C.c_void_p),
                                ids.size, C.byref(nnz)), "fixup_peers_of")
    return off, ids[: nnz.value]


def quantization_efficiency(t: int, p: int) -> float:  # decompose.cpp:138-141
    out = C.c_double()
    _check(lib().sk_quantization_efficiency(t, p, C.byref(out)), "quantization_efficiency")
    return out.value


# ----------------------------------------------------------------------------- text form
def to_text(a: WorkAssignment) -> str:  # types.cpp:96-107
    lines = [f"{a.problem.m} {a.problem.n} {a.problem.k}",
             f"{a.blocking.blk_m} {a.blocking.blk_n} {a.blocking.blk_k}"]
    tok = strategy_name(a.strategy)
    if a.strategy == Strategy.FixedSplit:
        tok += f":{a.split}"
    lines.append(f"{tok} {a.grid_size}")
    lines += [f"{r.cta_id} {r.iter_begin} {r.iter_end}" for r in a.ranges]
    return "\n".join(lines) + "\n"


def from_text(text: str) -> WorkAssignment:  # types.cpp:109-128
    toks = text.split()
    try:
        m, n, k = (int(x) for x in toks[0:3])
        bm, bn, bk = (int(x) for x in toks[3:6])
        tok, g = toks[6], int(toks[7])
    except (IndexError, ValueError) as e:
        raise ValueError("assignment text: bad header") from e
    split = 1
    if tok.startswith("fixed_split:"):
        split = int(tok[len("fixed_split:"):])
        strategy = Strategy.FixedSplit
    else:
        inv = {v: k_ for k_, v in _STRATEGY_NAMES.items()}
        if tok not in inv:
            raise ValueError("unknown strategy token: " + tok)
        strategy = inv[tok]
    rest = toks[8:]
    ranges = [CtaRange(int(rest[i]), int(rest[i + 1]), int(rest[i + 2]))
              for i in range(0, len(rest) - len(rest) % 3, 3)]
    if len(ranges) != g:
        raise ValueError("assignment text: range count != grid size")
    problem, blocking = GemmProblem(m, n, k), BlockingFactors(bm, bn, bk)
    a = WorkAssignment(strategy=strategy, grid_size=g, split=split, problem=problem,
                       blocking=blocking, grid=tile_grid(problem, blocking), ranges=ranges)
    a.param = _infer_param(a)
    return a


def _infer_param(a: WorkAssignment) -> int:
    """Recover the closed-form knob (s, g or p) of a parsed assignment; 0 when
    the range table is not one the device scheduler can reproduce."""
    want = a.range_table()
    if a.strategy == Strategy.DataParallel:
        cands = [1]
    elif a.strategy == Strategy.FixedSplit:
        cands = [a.split]
    elif a.strategy == Strategy.StreamK:
        cands = [a.grid_size]
    else:
        cands = range(1, a.grid_size + 1)
    for c in cands:
        try:
            tbl = _schedule_table(a.problem, a.blocking, a.strategy, c)
        except ValueError:
            continue
        if tbl.shape == want.shape and np.array_equal(tbl, want):
            return c
    return 0


class CostParams(C.Structure):
    """costmodel.hpp:15-21 CostParams plus B200 terms (csrc/costmodel.cpp):
    time(g) = e + ceil(g/p)*(a + b[peers>1] + c*ipc + d*(peers-1) + s*segs);
    `margin` = minimum predicted gain before leaving data-parallel."""
    _fields_ = [("e", C.c_double), ("a", C.c_double), ("b", C.c_double), ("c", C.c_double),
                ("d", C.c_double), ("s", C.c_double), ("margin", C.c_double),
                ("fit_residual", C.c_double), ("coop_peers", C.c_double),
                ("cluster_min_iters", C.c_double), ("cluster_kernel", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


def default_cost_params(ab_type: "DType" = None, variant: "Variant" = None) -> CostParams:
    ab_type = DType.BFloat16 if ab_type is None else ab_type
    variant = Variant.TwoSM if variant is None else variant
    out = CostParams()
    _check(lib().sk_default_cost_params(int(ab_type), int(variant), C.byref(out)), "cost params")
    return out


def predict_time(params: CostParams, grid: "TileGrid", g: int, p: int) -> float:
    out = C.c_double()
    _check(lib().sk_predict_time(C.byref(params), C.byref(grid._c()), g, p, C.byref(out)),
           "predict_time")
    return out.value


def select_grid_size(params: CostParams, grid: "TileGrid", p: int) -> int:
    """costmodel.cpp:30-48 argmin over g in {1..p} U {t}; g == t means data-parallel."""
    out = C.c_int64()
    _check(lib().sk_select_grid_size(C.byref(params), C.byref(grid._c()), p, C.byref(out)),
           "select_grid_size")
    return out.value


def calibrate(samples, p: int, margin: float = 0.15, coop_peers: float = 0.0) -> CostParams:
    """NNLS fit from [(TileGrid, g, time_us), ...] (costmodel.cpp:142-225);
    coop_peers > 0 models the kernel's cooperative fixup (see sk_cost_params)."""
    n = len(samples)
    grids = (sk_tile_grid_t * n)(*[s[0]._c() for s in samples])
    gs = np.array([s[1] for s in samples], np.int64)
    ts = np.array([s[2] for s in samples], np.float64)
    out = CostParams()
    out.margin = margin
    out.coop_peers = coop_peers
    _check(lib().sk_calibrate(grids, gs.ctypes.data_as(C.c_void_p), ts.ctypes.data_as(C.c_void_p),
                              n, p, C.byref(out)), "calibrate")
    return out


def predict_schedule(params: CostParams, grid: "TileGrid", strategy: "Strategy", param: int,
                     p: int) -> float:
    out = C.c_double()
    _check(lib().sk_predict_schedule(C.byref(params), C.byref(grid._c()), int(strategy), param, p,
                                     C.byref(out)), "predict_schedule")
    return out.value


def auto_stream_k(problem: "GemmProblem", blocking: "BlockingFactors", p: int,
                  params: Optional[CostParams] = None) -> "WorkAssignment":
    """The Stream-K policy (sk_select_schedule): the model's argmin over
    data_parallel, stream_k(g <= p) and two_tile_sk_dp(p), keeping
    data-parallel unless another schedule is predicted to win by > margin; on
    the 1-SM kernel fixed_split(S) with the DSMEM cluster fixup when it applies.
    Default constants follow the blocking's kernel."""
    if params is None:
        v = Variant.OneSM if (blocking.blk_m, blocking.blk_n) == (128, 256) else Variant.TwoSM
        params = default_cost_params(variant=v)
    grid = tile_grid(problem, blocking)
    s, prm = C.c_int32(), C.c_int64()
    _check(lib().sk_select_schedule(C.byref(params), C.byref(grid._c()), p, C.byref(s),
                                    C.byref(prm)), "select_schedule")
    return _assignment(Strategy(s.value), problem, blocking, prm.value)


class MatrixFileError(RuntimeError):
    """std::runtime_error of the reference's SKMX reader (matrix.cpp:37-61)."""


_NP_OF = {DType.Int64: np.int64, DType.Float32: np.float32, DType.Float64: np.float64,
          DType.BFloat16: np.uint16, DType.Float16: np.float16}


def save_matrix(path: str, a: np.ndarray, dtype: Optional[DType] = None) -> None:
    """SKMX writer (matrix.hpp:78-84); uint16 arrays are stored as bfloat16."""
    if dtype is None:
        dtype = {np.dtype(v): k for k, v in _NP_OF.items()}[a.dtype]
    a = np.ascontiguousarray(a, dtype=_NP_OF[dtype])
    rows, cols = a.shape
    st = lib().sk_save_matrix(os.fsencode(path), int(dtype), rows, cols, a.ctypes.data_as(C.c_void_p))
    if st == 7:
        raise MatrixFileError(lib().sk_io_error().decode())
    _check(st, "save_matrix")


def load_matrix(path: str, dtype: DType) -> np.ndarray:
    """SKMX reader (matrix.hpp:86-93): the file's dtype tag must equal `dtype`."""
    t, r, c = C.c_int(), C.c_int64(), C.c_int64()
    st = lib().sk_load_matrix_header(os.fsencode(path), C.byref(t), C.byref(r), C.byref(c))
    if st == 7:
        raise MatrixFileError(lib().sk_io_error().decode())
    _check(st, "load_matrix")
    out = np.empty((r.value, c.value), _NP_OF[DType(dtype)])
    st = lib().sk_load_matrix(os.fsencode(path), int(dtype), r.value, c.value,
                              out.ctypes.data_as(C.c_void_p))
    if st == 7:
        raise MatrixFileError(lib().sk_io_error().decode())
    _check(st, "load_matrix")
    return out


def cluster_capacity(cluster: int, variant: "Variant" = None, device: int = -1) -> int:
    """Units (1-SM: CTAs, 2-SM: CTA pairs) co-resident as clusters of `cluster`
    units (2 to 8): fixed_split(S) runs the DSMEM cluster fixup when t * S fits."""
    variant = Variant.TwoSM if variant is None else variant
    out = C.c_int32()
    _check(lib().sk_cluster_capacity(int(variant), cluster, device, C.byref(out)), "cluster_capacity")
    return out.value


def persistent_capacity(ab_type: DType = DType.BFloat16, variant: Variant = Variant.TwoSM,
                        device: int = -1) -> int:
    """Co-resident CTAs (CTA pairs for 2-SM) of the persistent kernel on a device:
    the cap of every launch's persistent grid."""
    out = C.c_int32()
    _check(lib().sk_persistent_capacity(int(ab_type), int(variant), device, C.byref(out)),
           "persistent_capacity")
    return out.value


def reload_env() -> None:
    """Re-read the SKB200_* tuning overrides (the library reads them once)."""
    lib().sk_reload_env()


def simulate(a: WorkAssignment, p: int, params=None, events: bool = False):
    """The reference simulator (simulate.cpp:23-80) on this library's schedules:
    returns (makespan, utilization) or, with events=True, a timeline.Timeline.
    params: None (unit cost) or an object/dict with a, b, c, d (reference
    CostParams semantics; e.g. fitted from device timelines)."""
    from . import timeline as tlm

    prm = None
    if params is not None:
        get = (lambda k: params[k]) if isinstance(params, dict) else (lambda k: getattr(params, k))
        prm = sk_sim_params(get("a"), get("b"), get("c"), get("d"))
    strategy, table = int(a.strategy), None
    if a.param == 0:
        table = _explicit_table(a)
        strategy = SK_EXPLICIT
    args = [C.byref(a.problem._c()), C.byref(a.blocking._c()), strategy, a.param,
            table.ctypes.data_as(C.c_void_p) if table is not None else None,
            0 if table is None else table.shape[0], p, C.byref(prm) if prm is not None else None]
    ms, ut, n = C.c_double(), C.c_double(), C.c_int64()
    st = lib().sk_simulate(*args, C.byref(ms), C.byref(ut), None, 0, C.byref(n))
    if st not in (SK_OK,):
        _check(st, "simulate")
    if not events:
        return ms.value, ut.value
    ev = np.zeros((max(n.value, 1), 6), np.float64)
    _check(lib().sk_simulate(*args, C.byref(ms), C.byref(ut), ev.ctypes.data_as(C.c_void_p), n.value,
                             C.byref(n)), "simulate")
    kinds = {0: "mac", 1: "fixup_wait", 2: "fixup_reduce"}
    evs = [tlm.Event(int(r[0]), int(r[1]), kinds[int(r[2])], float(r[3]), float(r[4]), int(r[5]))
           for r in ev[:n.value]]
    return tlm.Timeline(p, evs, ms.value)


_GEN = {DType.Int64: 0, DType.Float32: 1, DType.Float64: 2}


def random_matrix_device(rows: int, cols: int, seed: int, gen: DType = DType.Float32,
                         out: DType = DType.BFloat16, shift: int = 0, ld: Optional[int] = None,
                         stream=None):
    """random_matrix<gen>(rows, cols, seed) of the reference (matrix.hpp:39-68),
    generated on the current CUDA device and rounded into `out` (a torch
    tensor, rows x ld, viewed as rows x cols).  Int64 values may be shifted
    right (arithmetic) by `shift`."""
    import torch

    tdt = {DType.BFloat16: torch.bfloat16, DType.Float16: torch.float16, DType.Float32: torch.float32,
           DType.Float64: torch.float64}[DType(out)]
    es = torch.tensor([], dtype=tdt).element_size()
    al = 16 // es
    ld = ld or -(-cols // al) * al
    buf = torch.empty(rows, ld, dtype=tdt, device="cuda")
    s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    _check(lib().sk_random_matrix(_GEN[DType(gen)], shift, seed & (2**64 - 1), rows, cols, int(out),
                                  C.c_void_p(buf.data_ptr()), ld, C.c_void_p(s)), "random_matrix")
    return buf[:, :cols]


def corpus(seed: int = 0, count: int = 32824, lo: int = 128, hi: int = 8192) -> np.ndarray:
    """The paper's log-sampled geometry corpus in run_sweep order
    (sweep.cpp:79-86): [count][4] uint64 rows of (m, n, k, matrix_seed)."""
    out = np.zeros((count, 4), np.uint64)
    _check(lib().sk_corpus(seed, count, lo, hi, out.ctypes.data_as(C.c_void_p)), "corpus")
    return out


# ----------------------------------------------------------------------------- device GEMM
def kernel_blocking(ab_type: DType = DType.BFloat16, variant: Variant = Variant.Auto) -> BlockingFactors:
    """The single tile configuration per precision the device kernel uses."""
    out = sk_blocking()
    _check(lib().sk_kernel_blocking(int(ab_type), int(variant), C.byref(out)), "kernel_blocking")
    return BlockingFactors(out.blk_m, out.blk_n, out.blk_k)


def device_topology(device: int = 0) -> Optional[np.ndarray]:
    """Die of each SM (0/1) as probed by the library for the die-aware
    data-parallel phase, or None when the device shows no clean two-die split."""
    die = np.zeros(256, np.int32)
    sms, ok = C.c_int32(0), C.c_int32(0)
    _check(lib().sk_device_topology(device, die.ctypes.data_as(C.c_void_p), 256, C.byref(sms),
                                    C.byref(ok)), "device_topology")
    return die[:sms.value].copy() if ok.value else None


def _launch_desc(a: WorkAssignment, ab_type: DType, variant: Variant, tile_group: int = 0):
    d = sk_gemm_desc()
    d.tile_group = tile_group
    d.problem, d.blocking = a.problem._c(), a.blocking._c()
    d.strategy, d.param = int(a.strategy), a.param
    table = _explicit_table(a) if a.param == 0 else None
    if table is not None:
        d.strategy, d.ranges, d.num_ranges = SK_EXPLICIT, table.ctypes.data, table.shape[0]
    d.ab_type, d.variant = int(ab_type), int(variant)
    d.lda, d.ldb, d.ldc = a.problem.k, a.problem.n, a.problem.n
    return d, table


def persistent_order(a: WorkAssignment, num_ctas: int, ab_type: DType = DType.BFloat16,
                     variant: Variant = Variant.TwoSM) -> List[np.ndarray]:
    """Per persistent CTA (pair), the [n][4] int64 records {unit, tile,
    local_begin, local_end} its producer / MMA issuer / epilogue walk in a
    `num_ctas`-CTA launch (host-side, sk_persistent_order)."""
    d, _table = _launch_desc(a, ab_type, variant)
    out = []
    for cta in range(num_ctas):
        n = C.c_int64()
        _check(lib().sk_persistent_order(C.byref(d), num_ctas, cta, None, 0, C.byref(n)),
               "persistent_order")
        rec = np.zeros((max(n.value, 1), 4), np.int64)
        _check(lib().sk_persistent_order(C.byref(d), num_ctas, cta, rec.ctypes.data_as(C.c_void_p),
                                         n.value, C.byref(n)), "persistent_order")
        out.append(rec[:n.value])
    return out


def tile_blocks(a: WorkAssignment, ab_type: DType = DType.BFloat16,
                variant: Variant = Variant.TwoSM, tile_group: int = 0) -> np.ndarray:
    """[t][2] (tile row, tile column) of C each tile id denotes on the device
    (sk_tile_block): the reference's row-major map unless tile_group asks for
    the grouped layout (sk_gemm_desc.tile_group)."""
    d, _table = _launch_desc(a, ab_type, variant, tile_group)
    out = np.zeros((a.grid.total_tiles, 2), np.int64)
    r, c = C.c_int64(), C.c_int64()
    for t in range(a.grid.total_tiles):
        _check(lib().sk_tile_block(C.byref(d), t, C.byref(r), C.byref(c)), "tile_block")
        out[t] = (r.value, c.value)
    return out


def _host_type(arr: np.ndarray) -> DType:
    if arr.dtype == np.float32:
        return DType.Float32
    if arr.dtype == np.float64:
        return DType.Float64
    if arr.dtype == np.float16:
        return DType.Float16
    if arr.dtype == np.uint16:  # raw bfloat16 bits
        return DType.BFloat16
    if arr.dtype == np.int64:
        return DType.Int64
    raise ValueError(f"unsupported host dtype {arr.dtype}")


def execute(a: WorkAssignment, A: np.ndarray, B: np.ndarray, compute: DType = DType.BFloat16,
            variant: Variant = Variant.Auto, device: int = -1,
            out: Optional[np.ndarray] = None) -> np.ndarray:
    """Drop-in of streamk::execute<T> (executor.hpp:130-207): host A (m x k),
    B (k x n) in, new host C (m x n) out, synchronous.
    compute BFloat16/Float16: A/B float32 (rounded on the device), float16 or
    uint16 (bfloat16 bits); C float32.
    compute Float64 (DMMA): A/B float64, float32 (execute<float>, widened
    exactly, C float32) or int64 (execute<int64_t>, exact, C int64; refused
    unless max|A| max|B| k < 2^53).  The blocking must be the kernel tile of
    `compute` (kernel_blocking).  `out`: optional C-contiguous m x n array of
    the C type to write into.  When A, B and out all live in pinned (page-locked)
    memory and need no conversion, the library overlaps the copies with the
    kernel (row blocks of A in, finished rows of C out)."""
    p = a.problem
    if A.shape != (p.m, p.k) or B.shape != (p.k, p.n):
        raise ValueError("execute: matrix shapes do not match assignment")
    tbl = _explicit_table(a) if a.param == 0 else None  # no closed form: SK_EXPLICIT
    ht = _host_type(A)
    if _host_type(B) != ht:
        raise ValueError("execute: A and B host dtypes differ")
    A = np.ascontiguousarray(A)
    B = np.ascontiguousarray(B)
    if compute == DType.Float64:  # C in the caller's type: execute<double|float|int64_t>
        cdt = {DType.Float64: np.float64, DType.Float32: np.float32, DType.Int64: np.int64}[ht]
    else:
        cdt = np.float32
    if out is not None:
        if out.shape != (p.m, p.n) or out.dtype != cdt or not out.flags.c_contiguous:
            raise ValueError(f"execute: out must be a C-contiguous {p.m}x{p.n} {np.dtype(cdt)} array")
        Cm = out
    else:
        Cm = np.empty((p.m, p.n), cdt)
    if tbl is not None:
        _check(lib().sk_execute_ranges(C.byref(p._c()), C.byref(a.blocking._c()),
                                       tbl.ctypes.data_as(C.c_void_p), tbl.shape[0], int(ht),
                                       int(compute), int(variant), A.ctypes.data_as(C.c_void_p),
                                       B.ctypes.data_as(C.c_void_p), Cm.ctypes.data_as(C.c_void_p),
                                       device), "execute")
        return Cm
    _check(lib().sk_execute(C.byref(p._c()), C.byref(a.blocking._c()), int(a.strategy), a.param,
                            int(ht), int(compute), int(variant), A.ctypes.data_as(C.c_void_p),
                            B.ctypes.data_as(C.c_void_p), Cm.ctypes.data_as(C.c_void_p), device),
           "execute")
    return Cm


class Gemm:
    """A planned device GEMM (stream-ordered, device pointers): the
    sk_gemm_desc plus its self-cleaning fixup workspace.

    Tensors are torch CUDA tensors (torch is device-memory plumbing here, not
    compute): A (m x k) and B (k x n) in bf16/fp16, C (m x n) fp32, each
    row-major with a 16-byte-multiple leading dimension.
    """

    def __init__(self, a: WorkAssignment, ab_type: DType = DType.BFloat16,
                 variant: Variant = Variant.Auto, num_ctas: int = 0, trace: bool = False,
                 timeline: bool = False, tile_group: int = 0):
        import torch  # device memory only

        self.a = a
        self.ab_type = ab_type
        d = sk_gemm_desc()
        d.problem = a.problem._c()
        d.blocking = a.blocking._c()
        d.strategy = int(a.strategy)
        # a range table no closed form reproduces runs as SK_EXPLICIT
        self.table = _explicit_table(a) if a.param == 0 else None
        if self.table is not None:
            d.strategy = SK_EXPLICIT
            d.ranges = self.table.ctypes.data
            d.num_ranges = self.table.shape[0]
        d.ab_type = int(ab_type)
        d.param = a.param
        d.variant = int(variant)
        d.num_ctas = num_ctas
        d.tile_group = tile_group  # 0: the reference's row-major tile -> C map
        d.lda, d.ldb, d.ldc = a.problem.k, a.problem.n, a.problem.n
        self.desc = d
        ws = C.c_size_t()
        _check(lib().sk_workspace_size(C.byref(d), C.byref(ws)), "workspace_size")
        self.ws_bytes = ws.value
        self.workspace = torch.empty(max(self.ws_bytes, 256), dtype=torch.uint8, device="cuda")
        stream = torch.cuda.current_stream().cuda_stream
        _check(lib().sk_workspace_init(C.c_void_p(self.workspace.data_ptr()), self.ws_bytes,
                                       C.c_void_p(stream)), "workspace_init")
        self.trace = None
        if trace:
            n = C.c_int64()
            _check(lib().sk_trace_size(C.byref(d), C.byref(n)), "trace_size")
            # [4t tile records | g partial counts | t C-block storers]; -1 = unwritten
            T = a.grid.total_tiles
            self.trace = torch.full((n.value,), -1, dtype=torch.int32, device="cuda")
            self.trace[4 * T:n.value - T] = 0
        # per-CTA {clock64, globaltimer} stamps at start/end (clock_mhz())
        self.cta_clocks = torch.zeros(4 * 2 * 512, dtype=torch.int64, device="cuda") if trace else None
        self.events = None
        if timeline:
            n, stride = C.c_int64(), C.c_int64()
            _check(lib().sk_timeline_size(C.byref(d), C.byref(n), C.byref(stride)), "timeline_size")
            self.events = torch.zeros(8 * max(n.value, 1), dtype=torch.int64, device="cuda")

    def block_storers(self) -> np.ndarray:
        """[tiles_m][tiles_n] unit that stored each block of C in the last traced
        launch (trace section 3; -1 = never stored)."""
        T = self.a.grid.total_tiles
        t = self.trace.cpu().numpy()
        return t[t.size - T:].reshape(self.a.grid.tiles_m, self.a.grid.tiles_n)

    def timeline(self) -> np.ndarray:
        """Device-measured events of the last launch (timeline=True), one row per
        tile segment: [unit, tile, core, kind, t_mac_start, t_mac_end, t_wait_end,
        t_done] (globaltimer ns); see paper_2301_03598_b200.timeline."""
        ev = self.events.view(-1, 8).cpu().numpy()
        return ev[ev[:, 7] > 0]

    def clock_mhz(self) -> float:
        """Effective SM clock of the last traced launch: median over CTAs of
        d(clock64) / d(globaltimer)."""
        c = self.cta_clocks.view(-1, 4).cpu().numpy()
        c = c[(c[:, 3] > c[:, 1]) & (c[:, 2] > c[:, 0])]
        return float(np.median((c[:, 2] - c[:, 0]) / (c[:, 3] - c[:, 1]) * 1e3)) if len(c) else 0.0

    def run(self, A, B, Cout, stream=None) -> None:
        import torch

        d = self.desc
        for t, name in ((A, "A"), (B, "B"), (Cout, "C")):
            if not t.is_cuda or t.stride(1) != 1:
                raise ValueError(f"{name} must be a row-major CUDA tensor")
        d.A, d.lda = A.data_ptr(), A.stride(0)
        d.B, d.ldb = B.data_ptr(), B.stride(0)
        d.C, d.ldc = Cout.data_ptr(), Cout.stride(0)
        d.trace = self.trace.data_ptr() if self.trace is not None else None
        d.cta_clocks = self.cta_clocks.data_ptr() if self.cta_clocks is not None else None
        d.events = self.events.data_ptr() if self.events is not None else None
        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        _check(lib().sk_gemm(C.byref(d), C.c_void_p(self.workspace.data_ptr()), self.ws_bytes,
                             C.c_void_p(s)), "sk_gemm")

    def check(self, stream=None) -> None:
        """Synchronise and raise ProtocolError if the fixup protocol misbehaved."""
        import torch

        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        _check(lib().sk_workspace_check(C.c_void_p(self.workspace.data_ptr()), C.c_void_p(s)),
               "workspace_check")
