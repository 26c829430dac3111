"""Multi-GPU sharding with no data-path collective.

* A large GEMM is split by N-column blocks that are whole tile columns: rank j
  computes C[:, n_j:n_{j+1}] = A . B[:, n_j:n_{j+1}].  Each rank's schedule is
  the reference decomposition of GemmProblem{m, n_{j+1} - n_j, k}, so
  per-device schedule parity is the reference's own decompose().
* The geometry corpus is split one problem per GPU (shape i -> rank i % world,
  or LPT on FLOPs), merged back in input order.

The only inter-process traffic is control plane (barriers, timing, gathering
results for verification); the GEMM data path never crosses GPUs.
"""
from __future__ import annotations

import heapq
from typing import List, Sequence, Tuple

import paper_2301_03598_b200 as sk


def column_blocks(n: int, world: int, blk_n: int) -> List[Tuple[int, int]]:
    """Balanced split of the tile columns of an n-wide C over `world` ranks:
    the first (tiles_n % world) ranks get one extra tile column.  Returns
    [(n0, n1)] per rank; a rank may get an empty block when tiles_n < world."""
    if n < 1 or world < 1 or blk_n < 1:
        raise ValueError("column_blocks: n, world, blk_n >= 1")
    tiles_n = -(-n // blk_n)
    q, r = divmod(tiles_n, world)
    out, col = [], 0
    for j in range(world):
        cols = q + (1 if j < r else 0)
        n0 = min(n, col * blk_n)
        n1 = min(n, (col + cols) * blk_n)
        out.append((n0, n1))
        col += cols
    return out


def shard_problem(problem: "sk.GemmProblem", rank: int, world: int,
                  blocking: "sk.BlockingFactors") -> Tuple["sk.GemmProblem", int, int]:
    """This rank's sub-problem and its column range [n0, n1)."""
    n0, n1 = column_blocks(problem.n, world, blocking.blk_n)[rank]
    if n1 <= n0:
        return None, n0, n1
    return sk.GemmProblem(problem.m, n1 - n0, problem.k, problem.alpha, problem.beta), n0, n1


def assign_corpus(shapes: Sequence[Tuple[int, int, int]], world: int,
                  policy: str = "round_robin") -> List[List[int]]:
    """Shape indices per rank: round robin (i % world) or LPT on 2mnk."""
    if policy == "round_robin":
        return [list(range(j, len(shapes), world)) for j in range(world)]
    if policy == "lpt":
        heap = [(0.0, j) for j in range(world)]
        out: List[List[int]] = [[] for _ in range(world)]
        order = sorted(range(len(shapes)), key=lambda i: -2.0 * shapes[i][0] * shapes[i][1] * shapes[i][2])
        for i in order:
            load, j = heapq.heappop(heap)
            out[j].append(i)
            heapq.heappush(heap, (load + 2.0 * shapes[i][0] * shapes[i][1] * shapes[i][2], j))
        return [sorted(x) for x in out]
    raise ValueError(policy)


def run_column_shard(gemm_factory, A, B, C, rank: int, world: int, blocking, stream=None):
    """Device path: run this rank's column block through `gemm_factory(sub_problem)`
    (returns an sk.Gemm) on views of the caller's tensors; no collective."""
    problem = sk.GemmProblem(A.shape[0], B.shape[1], A.shape[1])
    sub, n0, n1 = shard_problem(problem, rank, world, blocking)
    if sub is None:
        return None
    g = gemm_factory(sub)
    g.run(A, B[:, n0:n1], C[:, n0:n1], stream)
    return g
