"""Multi-rank host logic of bench.py on CPU (gloo, world_size 2): the N>1
path shards independent fields across ranks (weak scaling, no data-path
collective), times on each rank, and reports the max over ranks."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, ws, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import bench

    w, r, local = bench.dist_init(backend="gloo")
    ms = 2.0 + 3.0 * r  # this rank's device time
    bench.barrier(w)
    m = bench.max_over_ranks(ms, w, device="cpu")
    q.put((r, local, bench.field_seed(r), m, bench.aggregate_gbs(w, 1e9, m)))
    import torch.distributed as dist

    dist.destroy_process_group()


def test_two_rank_max_and_aggregate():
    ws = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(ws))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    seeds = [o[2] for o in out]
    assert seeds == [0, 1]  # distinct fields: weak scaling over independent units
    for r, local, seed, m, agg in out:
        assert m == 5.0  # max over ranks, identical on every rank
        assert agg == pytest.approx(2 * 1e9 / 5e-3 / 1e9)


def test_reference_arm_nonzero_rank_exits_without_work():
    sys.path.insert(0, ROOT)
    import bench

    class A:
        steps = 1
        warmup = 0
        warmup_ref = 0
        ref_threads = 1

    assert bench.run_reference(A(), 2, 1) is None


def test_self_launch_two_ranks():
    """`bench.py --gpus 2` outside torchrun spawns 2 ranks itself (gloo
    plumbing check): one JSON line from rank 0 with n_gpus 2, max over ranks."""
    import json
    import subprocess

    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dist-selftest"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [json.loads(x) for x in p.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, p.stdout
    assert lines[0]["n_gpus"] == 2 and lines[0]["ms_per_step"] == 2.0
    assert p.stderr.count("[bench] rank ") == 2
