"""Host-side DSO logic (chunk planning, bucketing) and multi-GPU request
sharding, including a world_size-2 gloo run of the sharding plumbing."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_2509_22681_b200 as fb
from paper_2509_22681_b200.orchestrator import ProfileSet, bucket_of, plan_chunks
from paper_2509_22681_b200.sharding import assign_requests

PRODUCTION_SHAPES = ProfileSet(shapes=(128, 256, 512, 1024), executors_per_shape=1)


def test_plan_kats():
    # reference tests/test_orchestrator.py:41-61
    got = lambda n: [(c.shape, c.real_count, c.pad_count) for c in plan_chunks(n, PRODUCTION_SHAPES).chunks]
    assert got(640) == [(512, 512, 0), (128, 128, 0)]
    assert got(100) == [(128, 100, 28)]
    assert got(1700) == [(1024, 1024, 0), (512, 512, 0), (128, 128, 0), (128, 36, 92)]


def test_plan_invariants_exhaustive():
    profiles = ProfileSet(shapes=(4, 8, 16, 32), executors_per_shape=1)
    for batch in range(1, 4 * 32 + 1):
        plan = plan_chunks(batch, profiles)
        shapes = [c.shape for c in plan.chunks]
        assert all(s in profiles.shapes for s in shapes)
        assert shapes == sorted(shapes, reverse=True)
        assert all(c.real_count + c.pad_count == c.shape for c in plan.chunks)
        assert sum(c.real_count for c in plan.chunks) == batch == plan.total_real
        assert all(c.pad_count == 0 for c in plan.chunks[:-1])


def test_profile_set_validation():
    for kw in (dict(shapes=()), dict(shapes=(8, 8)), dict(shapes=(8, 4)),
               dict(shapes=(4,), executors_per_shape=0)):
        with pytest.raises(ValueError):
            ProfileSet(**kw)
    with pytest.raises(ValueError):
        plan_chunks(0, PRODUCTION_SHAPES)


def test_bucket_of_powers_of_two():
    cfg = fb.ModelConfig(256, 64, 4, 1, 1024, 2, 1024, 2048)
    assert bucket_of(1024, 256, cfg) == (256, 256)
    assert bucket_of(1000, 17, cfg) == (256, 32)
    assert bucket_of(0, 3, cfg) == (0, 16)
    assert bucket_of(4, 2048, cfg) == (1, 2048)


def test_assign_requests_balanced_and_complete():
    rng = np.random.default_rng(0)
    shapes = [(1024, int(c)) for c in 16 + rng.integers(0, 2033, 200)]
    for ws in (1, 2, 4, 8):
        parts = assign_requests(shapes, ws, num_blocks=4)
        flat = sorted(i for p in parts for i in p)
        assert flat == list(range(len(shapes)))
        loads = [sum(4 * shapes[i][1] + shapes[i][0] for i in p) for p in parts]
        assert max(loads) - min(loads) <= 4 * 2048 + 1024


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    from paper_2509_22681_b200.sharding import Dist, assign_requests

    d = Dist(backend="gloo")
    shapes = [(64, c) for c in (5, 100, 7, 64, 3, 33)]
    mine = assign_requests(shapes, world, num_blocks=2)[rank]
    d.barrier()
    tmax = d.max(1.0 + rank)
    total = d.sum(float(sum(shapes[i][1] for i in mine)))
    out[rank] = (tuple(mine), tmax, total)
    d.close()


def test_sharding_gloo_world2():
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    a, b = out[0], out[1]
    assert set(a[0]).isdisjoint(b[0]) and sorted(a[0] + b[0]) == list(range(6))
    assert a[1] == b[1] == 2.0  # max over ranks
    assert a[2] == b[2] == 212.0  # every candidate scored exactly once


def test_candidate_buckets():
    from paper_2509_22681_b200.orchestrator import cand_bucket

    assert [cand_bucket(c) for c in (1, 16, 17, 100, 129, 257, 300, 384, 385, 600, 768, 769, 1100, 1536, 1537)] == \
        [16, 16, 32, 128, 256, 384, 384, 384, 512, 768, 768, 1024, 1536, 1536, 2048]
    for c in range(1, 2049):
        b = cand_bucket(c)
        assert b >= c and (b < 128 or b % 128 == 0)


def test_vectorised_plan_matches_scalar_buckets():
    """The vectorised plan (large batches) groups exactly like bucket_of."""
    from paper_2509_22681_b200.orchestrator import BucketScheduler

    cfg = fb.ModelConfig(256, 64, 4, 1, 1024, 2, 1024, 2048)

    class Eng:
        config = cfg

    sched = BucketScheduler.__new__(BucketScheduler)
    sched.engine, sched.target_rows, sched.max_slots = Eng(), 4096, 64
    rng = np.random.default_rng(3)
    shapes = [(4 * int(h), int(c)) for h, c in zip(rng.integers(0, 257, 500), rng.integers(1, 2049, 500))]
    plan = sched.plan(shapes)
    seen = sorted(i for _, idx in plan for i in idx)
    assert seen == list(range(500))
    for key, idx in plan:
        assert len(idx) <= sched.slots_for(key[1])
        assert all(bucket_of(*shapes[i], cfg) == key for i in idx)
        assert idx == sorted(idx)


def test_bench_reference_arm_under_torchrun_gloo(tmp_path):
    """The driver's launch of the reference arm at N = 2 (torchrun, one process per
    rank): rank 0 alone times the CPU reference and prints one JSON line with the
    reference-arm keys, the other rank exits 0."""
    import json
    import subprocess
    import sys

    env = dict(os.environ, FLAME_BENCH_CPU_PROCS="2", OMP_NUM_THREADS="1")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--impl", "reference",
           "--gpus", "2", "--workload", "cfg1", "--steps", "1", "--warmup", "3"]
    out = subprocess.run(cmd, cwd=str(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    # "reference" when the unmodified reference is installed in baseline/_ref, else the oracle port
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] in ("reference", "port")
