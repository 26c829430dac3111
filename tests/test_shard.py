"""Multi-process sharding on CPU (gloo, world size 2): the column-block split
covers C exactly, each rank's schedule is the reference decomposition of its
sub-problem, and the blocks computed independently (oracle executor, no data
exchange) reassemble to the full product.  The corpus split is a partition."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    import oracle

    import paper_2301_03598_b200 as sk
    from paper_2301_03598_b200 import shard

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        port_ = oracle.Oracle("port")
        m, n, k = 300, 1000, 520
        blk = sk.BlockingFactors(128, 256, 64)
        A = port_.random_matrix(m, k, 5, "int64")
        B = port_.random_matrix(k, n, 6, "int64")
        sub, n0, n1 = shard.shard_problem(sk.GemmProblem(m, n, k), rank, world, blk)
        # per-rank schedule == reference decomposition of the sub-problem
        a = sk.stream_k(sub, blk, 7)
        assert np.array_equal(a.range_table(),
                              port_.schedule("stream_k", sub.m, sub.n, sub.k, 128, 256, 64, 7))
        Cblk = port_.execute("stream_k", 7, A, np.ascontiguousarray(B[:, n0:n1]), 128, 256, 64)
        # control-plane gather for verification only
        blocks = [None] * world
        dist.all_gather_object(blocks, (n0, Cblk.astype(np.float64)))
        if rank == 0:
            full = np.concatenate([b for _, b in sorted(blocks, key=lambda x: x[0])], axis=1)
            q.put(bool(np.array_equal(full, (A @ B).astype(np.float64))))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_column_blocks_partition(sk):
    from paper_2301_03598_b200 import shard

    for n, world, bn in ((8192, 8, 256), (1000, 3, 256), (100, 4, 256), (5000, 2, 128)):
        blocks = shard.column_blocks(n, world, bn)
        assert blocks[0][0] == 0 and blocks[-1][1] == n
        for (a0, a1), (b0, b1) in zip(blocks, blocks[1:]):
            assert a1 == b0
        for n0, n1 in blocks:
            assert n1 == n0 or n0 % bn == 0  # whole tile columns per (nonempty) rank
    with pytest.raises(ValueError):
        shard.column_blocks(0, 2, 256)


def test_corpus_assignment_partition(sk):
    from paper_2301_03598_b200 import shard

    shapes = [tuple(int(x) for x in r[:3]) for r in sk.corpus(0, 500)]
    for policy in ("round_robin", "lpt"):
        parts = shard.assign_corpus(shapes, 4, policy)
        flat = sorted(i for p in parts for i in p)
        assert flat == list(range(500))
    rr = shard.assign_corpus(shapes, 4, "round_robin")
    assert rr[1][:3] == [1, 5, 9]


def test_gloo_world2_column_shards_reassemble():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, q), nprocs=2, start_method="spawn", join=True)
    assert q.get(timeout=60) is True


def _gpu_worker(rank, world, port, q):
    """One rank of a world-2 job on ONE GPU: the CUDA kernel computes this
    rank's column block on views of the full tensors; the blocks travel over
    gloo only for verification (control plane)."""
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    import oracle

    import paper_2301_03598_b200 as sk
    from paper_2301_03598_b200 import shard

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        port_ = oracle.Oracle("port")
        m, n, k = 1000, 2944, 1504  # 16-byte rows (TMA)
        V = sk.Variant.TwoSM
        blk = sk.kernel_blocking(sk.DType.BFloat16, V)
        Ai = port_.random_matrix(m, k, 15, "int64")
        Bi = port_.random_matrix(k, n, 16, "int64")
        A = torch.from_numpy(Ai.astype(np.float32)).cuda().to(torch.bfloat16)
        B = torch.from_numpy(Bi.astype(np.float32)).cuda().to(torch.bfloat16)
        C = torch.full((m, n), float("nan"), device="cuda")
        ok = True
        for make in (lambda p: sk.stream_k(p, blk, 74), lambda p: sk.hybrid(p, blk, 74, sk.HybridVariant.TwoTileSkDp),
                     lambda p: sk.data_parallel(p, blk)):
            g = shard.run_column_shard(lambda sub: sk.Gemm(make(sub), variant=V), A, B, C, rank, world, blk)
            g.check()
            sub, n0, n1 = shard.shard_problem(sk.GemmProblem(m, n, k), rank, world, blk)
            # this rank's schedule == the reference decomposition of its sub-problem
            a = make(sub)
            ok &= bool(np.array_equal(a.range_table(), port_.schedule(
                int(a.strategy), sub.m, sub.n, sub.k, blk.blk_m, blk.blk_n, blk.blk_k, a.param)))
            blocks = [None] * world
            dist.all_gather_object(blocks, (n0, C[:, n0:n1].double().cpu().numpy()))
            if rank == 0:
                full = np.concatenate([b for _, b in sorted(blocks, key=lambda x: x[0])], axis=1)
                want = port_.execute("data_parallel", 1, Ai, Bi, blk.blk_m, blk.blk_n, blk.blk_k)
                ok &= bool(np.array_equal(full, want.astype(np.float64)))
        if rank == 0:
            q.put(ok)
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_gpu_world2_column_shards_bit_exact(torch_cuda):
    """shard.run_column_shard at world size 2 (gloo, one GPU): each rank's CUDA
    launch on its N-column block reassembles to a C bit-exact with the oracle's
    int64 executor; no data-path collective."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    mp.start_processes(_gpu_worker, args=(2, port, q), nprocs=2, start_method="spawn", join=True)
    assert q.get(timeout=120) is True
