"""DSO on the device: the reference orchestrator tests
(tests/test_orchestrator.py) re-run against B200 executors."""

import threading

import numpy as np
import pytest

import paper_2509_22681_b200 as fb
from paper_2509_22681_b200.orchestrator import (BucketScheduler, ImplicitShapeRunner, PoolClosedError,
                                                ProfileSet, build_pool, execute_request)

pytestmark = pytest.mark.gpu


def small_model():
    cfg = fb.ModelConfig(8, 4, 2, 1, 12, 2, 16, 256, seed=21)
    return cfg, fb.init_params(cfg)


def test_chunked_scores_match_unchunked(gpu):
    cfg, params = small_model()
    pool = build_pool(ProfileSet(shapes=(4, 8, 16), executors_per_shape=2), params, cfg)
    rng = np.random.default_rng(5)
    history = rng.normal(size=(8, 8))
    for batch in (1, 3, 4, 16, 21, 37):
        cand = rng.normal(size=(batch, 8))
        chunked = execute_request(history, cand, pool)
        direct = fb.model_forward(history, cand, params, cfg)
        np.testing.assert_array_equal(chunked, direct)
    pool.shutdown()


def test_pool_mechanics_and_zero_steady_state_allocations(gpu):
    cfg, params = small_model()
    pool = build_pool(ProfileSet(shapes=(4, 8), executors_per_shape=3), params, cfg)
    assert pool.executor_count == 6 and pool.queue_size(4) == 3
    rng = np.random.default_rng(8)
    history = rng.normal(size=(8, 8))
    for batch in (3, 8, 17, 25):
        res = pool.execute(history, rng.normal(size=(batch, 8)))
        assert res.scores.shape == (batch, 2) and res.compute_s > 0
    assert pool.steady_state_allocations == 0
    ex = pool.acquire(4)
    pool.release(ex)
    with pytest.raises(RuntimeError):
        pool.release(ex)
    pool.shutdown()
    with pytest.raises(PoolClosedError):
        pool.execute(history, rng.normal(size=(2, 8)))


def test_concurrent_requests_all_exact(gpu):
    cfg, params = small_model()
    pool = build_pool(ProfileSet(shapes=(4, 8), executors_per_shape=2), params, cfg)
    rng = np.random.default_rng(11)
    history = rng.normal(size=(8, 8))
    batches = [rng.normal(size=(int(n), 8)) for n in rng.integers(1, 20, 12)]
    expected = [fb.model_forward(history, c, params, cfg) for c in batches]
    results = [None] * len(batches)

    def worker(i):
        results[i] = execute_request(history, batches[i], pool)

    threads = [threading.Thread(target=worker, args=(i,)) for i in range(len(batches))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for got, want in zip(results, expected):
        np.testing.assert_array_equal(got, want)
    pool.shutdown()


def test_implicit_runner(gpu):
    cfg, params = small_model()
    runner = ImplicitShapeRunner(params, cfg)
    rng = np.random.default_rng(10)
    history = rng.normal(size=(8, 8))
    cand = rng.normal(size=(7, 8))
    assert runner.steady_state_allocations == 0
    res = runner.execute(history, cand)
    assert runner.steady_state_allocations > 0
    np.testing.assert_array_equal(res.scores, fb.model_forward(history, cand, params, cfg))


def test_bucket_scheduler_zipf_candidates(gpu):
    """cfg4-style traffic: C = 16 + Zipf rank; buckets batch many requests per replay."""
    cfg = fb.ModelConfig(64, 16, 4, 1, 256, 2, 256, 2048, seed=2)
    params = fb.init_params(cfg)
    eng = fb.get_engine(params, cfg, "bf16")
    sched = BucketScheduler(eng, target_rows=2048)
    rng = np.random.default_rng(2509)
    w = 1.0 / np.arange(1, 2034)
    cdf = np.cumsum(w / w.sum())
    counts = 16 + np.searchsorted(cdf, rng.random(40))
    reqs = [(rng.uniform(-1, 1, (256, 64)), rng.uniform(-1, 1, (int(c), 64))) for c in counts]
    got = sched.score(reqs)
    for (h, c), s in zip(reqs[:10], got[:10]):
        np.testing.assert_array_equal(s, fb.model_forward(h, c, params, cfg))
    assert all(s.shape == (len(c), 2) for (_, c), s in zip(reqs, got))


def test_bucket_scheduler_ring_and_ids(gpu):
    """Many groups per bucket (small target_rows) wrap each bucket's executor ring:
    async submit/collect must still return every request's exact scores; the id
    path (device PDA) must equal embedding-path scoring of the same rows."""
    from paper_2509_22681_b200.pda import build_item_table

    cfg = fb.ModelConfig(64, 16, 4, 1, 256, 2, 256, 256, seed=3)
    params = fb.init_params(cfg)
    eng = fb.FlameEngine(params, cfg, "bf16")
    table = build_item_table(500, 64)
    eng.set_table(table, dtype="fp32")
    sched = BucketScheduler(eng, target_rows=64, with_ids=True, executors_per_bucket=2)
    rng = np.random.default_rng(7)
    counts = rng.integers(1, 200, 30)
    reqs = [(rng.integers(0, 500, 256), rng.integers(0, 500, int(c))) for c in counts]
    plan = sched.plan([(256, int(c)) for c in counts])
    assert max(sum(1 for k, _ in plan if k == key) for key, _ in plan) > 2  # ring wraps
    got = sched.score(reqs, ids=True)
    assert len(sched.last_latencies) == len(reqs) and min(sched.last_latencies) > 0
    emb = BucketScheduler(eng, target_rows=64)
    want = emb.score([(table[h], table[c]) for h, c in reqs])
    for g, w, c in zip(got, want, counts):
        assert g.shape == (int(c), 2)
        np.testing.assert_array_equal(g, w)


def test_score_stream_matches_score(gpu):
    """Streaming several batches (next batch submitted before the previous is
    collected) returns, per batch and in order, exactly what score() returns."""
    cfg = fb.ModelConfig(32, 8, 2, 1, 64, 2, 64, 128, seed=9)
    params = fb.init_params(cfg)
    eng = fb.FlameEngine(params, cfg, "bf16")
    sched = BucketScheduler(eng, target_rows=256, executors_per_bucket=2)
    rng = np.random.default_rng(4)
    batches = []
    for _ in range(4):
        counts = rng.integers(1, 129, int(rng.integers(3, 9)))
        batches.append([(rng.uniform(-1, 1, (64, 32)), rng.uniform(-1, 1, (int(c), 32))) for c in counts])
    streamed = list(sched.score_stream(batches))
    assert len(streamed) == len(batches)
    for batch, got in zip(batches, streamed):
        want = sched.score(batch)
        for g, w in zip(got, want):
            np.testing.assert_array_equal(g, w)
