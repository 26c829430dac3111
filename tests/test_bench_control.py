"""bench.py's multi-rank control plane on CPU: two ranks over gloo (the only
inter-rank traffic of the bench -- barrier and max-over-ranks; no NCCL), and
the reference arm's JSON contract on a tiny row sample."""
import json
import os
import socket
import subprocess
import sys

import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port), LOCAL_RANK=str(rank))
    import bench

    cp = bench.ControlPlane(world)
    cp.barrier()
    got = cp.max(1.5 + rank)
    backend = cp.dist.get_backend()
    cp.close()
    q.put((rank, got, backend))


def test_control_plane_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_rank, args=(2, _free_port(), q), nprocs=2, start_method="spawn", join=True)
    res = sorted(q.get(timeout=60) for _ in range(2))
    assert [r[1] for r in res] == [2.5, 2.5]  # max over ranks seen by both
    assert all(r[2] == "gloo" for r in res)


def test_bench_has_no_nccl():
    src = open(os.path.join(ROOT, "bench.py")).read()
    assert '"nccl"' not in src and "'nccl'" not in src


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "0", "--cpu-rows", "8"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "TFLOP/s"
    assert line["cpu_baseline"]["kind"] in ("reference", "port") and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["value"] > 0
