"""Rows f2 / f4 of SURVEY.md section 8(f) on the CPU:

* the sweep CSV keeps the reference's `# schema=1` header and its first nine
  columns byte-identical to run_sweep's (sweep.cpp:75-112) for the same corpus,
  strategies, p and blocking (acceptance.cpp:269-283 checks the reference's
  own byte-determinism the same way);
* sk_simulate (the library's restatement of simulate.cpp:23-80) gives the
  reference simulator's makespan and utilization bit-for-bit, unit cost and
  with CostParams.
"""
import numpy as np
import pytest

NAMES = ["data_parallel", "stream_k", "two_tile_sk_dp", "dp_one_tile_sk", "fixed_split"]


@pytest.mark.parametrize("p,blk", [(74, (256, 256, 64)), (148, (128, 256, 64)), (8, (128, 128, 32))])
def test_sweep_reference_columns_byte_identical(sk, ref, p, blk):
    import oracle
    from paper_2301_03598_b200 import sweep as sw

    count = 150
    text = oracle.ref_run_sweep(0, count, 128, 8192, NAMES, p, 2, blk)
    lines = text.splitlines()
    assert lines[0] == sw.SCHEMA
    assert lines[1] == ",".join(sw.REF_COLUMNS)
    b = sk.BlockingFactors(*blk)
    ours = []
    for m, n, k, _seed in sk.corpus(0, count, 128, 8192).tolist():
        for a in sw.strategies_for(sk.GemmProblem(int(m), int(n), int(k)), b, p, NAMES):
            # unmeasured reference rows end with an empty measured_time field
            ours.append(",".join(str(x) for x in sw.ref_columns(a, p)) + ",")
    assert ours == lines[2:]


def test_csv_line_layout(sk):
    """A measured row: the reference's ten columns, then the GPU columns."""
    from paper_2301_03598_b200 import sweep as sw

    a = sk.stream_k(sk.GemmProblem(1024, 1024, 4096), sk.BlockingFactors(256, 256, 64), 74)
    r = {"ref": sw.ref_columns(a, 74), "time_us": 12.5, "strategy": "stream_k", "param": 74,
         "variant": "2sm", "dtype": "bf16", "copies": 16, "l2_cold": 0, "tflops": 687.2,
         "gbps": 1000.0, "int_exact": 1, "float_check": "full", "max_rel_err": 1e-7,
         "verified": "pass", "cpu_time_s": 0.5, "cpu_threads": 16, "cpu_model": "reference:x"}
    fields = sw.csv_line(r).split(",")
    assert len(fields) == len(sw.COLUMNS)
    assert fields[9] == "1.25e-05"  # measured_time, seconds, %.9g
    assert fields[sw.COLUMNS.index("verified")] == "pass"


def test_simulate_matches_reference(sk, ref):
    import oracle

    rng = np.random.default_rng(7)
    for trial in range(60):
        m, n, k = (int(x) for x in rng.integers(1, 3000, 3))
        bm, bn, bk = (int(x) for x in rng.choice([16, 32, 64, 128, 256], 3))
        strat = int(rng.integers(0, 5))
        param = int(rng.integers(1, 200))
        p = int(rng.integers(1, 160))
        b = sk.BlockingFactors(bm, bn, bk)
        a = sk._assignment(sk.Strategy(strat), sk.GemmProblem(m, n, k), b, param)
        for params in (None, (3.0, 1.5, 0.7, 2.25)):
            want = oracle.ref_simulate(strat, param, m, n, k, bm, bn, bk, p, params)
            got = sk.simulate(a, p, None if params is None else dict(zip("abcd", params)))
            assert got == want, (trial, strat, param, p, params)


def test_simulate_events_and_errors(sk):
    """Event records follow simulate.cpp's dispatch: one mac event per unit (empty
    ranges included), a fixup_reduce after every owner with peers when costed."""
    b = sk.BlockingFactors(128, 128, 4)
    a = sk.stream_k(sk.GemmProblem(384, 384, 128), b, 4)  # acceptance c1: 4 x 72
    tl = sk.simulate(a, 4, events=True)
    assert tl.makespan == 72.0 and len(tl.events) == 4
    assert sk.simulate(a, 4) == (72.0, 1.0)
    tl = sk.simulate(a, 4, {"a": 1.0, "b": 2.0, "c": 1.0, "d": 5.0}, events=True)
    reduce = [e for e in tl.events if e.kind == "fixup_reduce"]
    peers = sk.fixup_peers_of(a)
    assert len(reduce) == len({p[0] for p in peers if len(p) > 1})
    with pytest.raises(ValueError):
        sk.simulate(a, 0)
