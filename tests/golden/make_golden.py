"""Generate the committed golden fixtures from the REFERENCE ITSELF.

Runs the reference's own sources, compiled here by oracle/Makefile into
oracle/_ref/libstreamk_ref.so (it needs /root/reference, so it only runs in the
dev container).  Outputs (committed, small):

  tests/golden/schedules.json.gz  to_text / range tables / fixup_peers_of of every
                                BASELINE config at the kernel tile configs, the
                                reference tests' own golden instances, and
                                seeded random instances
  tests/golden/executor.npz     random_matrix streams, execute<T> outputs for
                                int64 / float32 / float64 instances, corpus dims

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import gzip
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle  # noqa: E402

NAMES = ["data_parallel", "fixed_split", "stream_k", "dp_one_tile_sk", "two_tile_sk_dp"]


def sched_entry(R, strat, m, n, k, bm, bn, bk, param, text=False):
    tbl = R.schedule(strat, m, n, k, bm, bn, bk, param)
    off, ids = R.fixup_peers(strat, m, n, k, bm, bn, bk, param)
    e = {"strategy": strat, "m": m, "n": n, "k": k, "bm": bm, "bn": bn, "bk": bk, "param": param,
         "grid": list(R.tile_grid(m, n, k, bm, bn, bk)), "ranges": tbl.ravel().tolist(),
         "peer_offsets": off.tolist(), "peer_ids": ids.tolist()}
    if text:
        e["text"] = R.to_text(strat, m, n, k, bm, bn, bk, param)
    return e


def main():
    oracle.build(with_ref=True)
    R = oracle.Oracle("reference")
    out = {"source": "reference streamk-lab core (oracle/_ref/libstreamk_ref.so)", "entries": []}
    E = out["entries"]
    # -- goldens of the reference's own tests (test_domain/test_decompose/acceptance)
    E.append(sched_entry(R, "stream_k", 384, 384, 128, 128, 128, 4, 4, text=True))
    E.append(sched_entry(R, "stream_k", 256, 3584, 8192, 128, 128, 32, 108))
    E.append(sched_entry(R, "stream_k", 128, 128, 16384, 128, 128, 32, 8, text=True))
    E.append(sched_entry(R, "stream_k", 4, 4, 4, 4, 4, 4, 7, text=True))
    E.append(sched_entry(R, "dp_one_tile_sk", 896, 384, 128, 128, 128, 128, 4, text=True))
    E.append(sched_entry(R, "two_tile_sk_dp", 896, 384, 128, 128, 128, 128, 4, text=True))
    E.append(sched_entry(R, "fixed_split", 32, 32, 5, 32, 32, 1, 2, text=True))
    E.append(sched_entry(R, "fixed_split", 384, 384, 128, 128, 128, 64, 2, text=True))
    E.append(sched_entry(R, "fixed_split", 64, 64, 64, 32, 32, 16, 3, text=True))
    E.append(sched_entry(R, "data_parallel", 384, 384, 128, 128, 128, 128, 1, text=True))
    # -- BASELINE configs at the kernel tile configs
    cfgs = [
        (384, 384, 128, 128, 128, 128, 4), (384, 384, 128, 128, 128, 4, 4),
        (384, 384, 128, 128, 128, 16, 4),
        (8192, 8192, 8192, 128, 256, 64, 148), (8192, 8192, 8192, 256, 256, 64, 74),
        (1024, 1024, 32768, 128, 256, 64, 148), (1024, 1024, 32768, 256, 256, 64, 74),
        (1280, 3840, 4096, 128, 256, 64, 148), (1280, 3840, 8192, 128, 256, 64, 148),
        (1280, 3840, 4096, 256, 256, 64, 74), (1024, 4864, 4096, 128, 256, 64, 148),
        (2048, 2048, 2048, 64, 64, 16, 148), (1024, 1024, 1024, 64, 64, 16, 148),
    ]
    for (m, n, k, bm, bn, bk, p) in cfgs:
        for strat in NAMES:
            param = {"data_parallel": 1, "fixed_split": 2}.get(strat, p)
            E.append(sched_entry(R, strat, m, n, k, bm, bn, bk, param))
    # -- seeded random instances (acceptance c6 ranges: dims <= 300, blk <= 40)
    rng = np.random.default_rng(0x5eed)
    for _ in range(150):
        m, n, k = (int(x) for x in rng.integers(1, 301, 3))
        bm, bn, bk = (int(x) for x in rng.integers(1, 41, 3))
        strat = NAMES[int(rng.integers(0, 5))]
        param = {"data_parallel": 1, "fixed_split": int(rng.integers(1, 10))}.get(
            strat, int(rng.integers(1, 161)))
        E.append(sched_entry(R, strat, m, n, k, bm, bn, bk, param))
    with gzip.open(os.path.join(HERE, "schedules.json.gz"), "wt") as f:
        json.dump(out, f, separators=(",", ":"))

    # -- executor / generator fixtures
    arr = {}
    arr["rm_f64_16x16_s99"] = R.random_matrix(16, 16, 99, "float64")
    arr["rm_f32_7x9_s123"] = R.random_matrix(7, 9, 123, "float32")
    arr["rm_i64_32x32_s5"] = R.random_matrix(32, 32, 5, "int64")
    # execute int64 (test_executor.cpp:85-108 instances); |C| < 2^31 so stored as int32
    A = R.random_matrix(384, 128, 31, "int64")
    B = R.random_matrix(128, 384, 32, "int64")
    arr["x_i64_sk4_C"] = R.execute("stream_k", 4, A, B, 128, 128, 4, threads=4).astype(np.int32)
    A = R.random_matrix(128, 96, 41, "int64")
    B = R.random_matrix(96, 128, 42, "int64")
    arr["x_i64_fs3_C"] = R.execute("fixed_split", 3, A, B, 128, 128, 32, threads=3).astype(np.int32)
    # float32 stream_k g=6 96x96x512 (test_executor.cpp:157-165)
    A = R.random_matrix(96, 512, 71, "float32")
    B = R.random_matrix(512, 96, 72, "float32")
    arr["x_f32_sk6_C"] = R.execute("stream_k", 6, A, B, 32, 32, 16, threads=4)
    arr["x_f32_ref_C"] = R.gemm_reference(A, B, 32, 32, 16)
    # float64 two_tile_sk_dp p=5 on 200x150x300 blk 32x32x16
    A = R.random_matrix(200, 300, 81, "float64")
    B = R.random_matrix(300, 150, 82, "float64")
    arr["x_f64_2t5_C"] = R.execute("two_tile_sk_dp", 5, A, B, 32, 32, 16, threads=4)
    # kernel-tile instance: stream_k g=7 on 384x768x1000 int64 (the smoke() case)
    A = R.random_matrix(384, 1000, 31, "int64")
    B = R.random_matrix(1000, 768, 32, "int64")
    Cs = R.execute("stream_k", 7, A, B, 128, 256, 64, threads=8)
    arr["x_i64_smoke_rowsum"], arr["x_i64_smoke_colsum"] = Cs.sum(1), Cs.sum(0)
    arr["x_i64_smoke_C_rows0_8"] = Cs[:8].astype(np.int32)
    arr["corpus_dims_s0"] = oracle.ref_corpus_dims(0, 256)
    np.savez_compressed(os.path.join(HERE, "executor.npz"), **arr)
    print("wrote", len(E), "schedule entries and", len(arr), "arrays")


if __name__ == "__main__":
    main()
