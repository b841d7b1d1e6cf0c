"""The device service with the reference's feature-cache semantics over the HBM
item table (§8(f)2, feature_cache.DeviceFeatureCache): the reference service
tests that depend on the cache (tests/test_service.py:53-62 cold async cache ->
zero embeddings) and the freshness rules of cache.py:170-357, on the device."""

import numpy as np
import pytest

import paper_2509_22681_b200 as fb
from oracle import flame_oracle as orc
from paper_2509_22681_b200.feature_cache import CacheConfig, CacheMode
from paper_2509_22681_b200.pda import item_embedding
from paper_2509_22681_b200.service import DeviceService, ScoreRequest

pytestmark = pytest.mark.gpu

CFG = fb.ModelConfig(32, 8, 2, 1, 64, 2, 64, 32, seed=5)
NUM_ITEMS = 400
TOL = 1e-4  # fp32 verification mode


class Clock:
    def __init__(self):
        self.now = 0.0

    def __call__(self):
        return self.now


def request_of(hist, cand):
    return ScoreRequest(user_id=1, history_item_ids=np.asarray(list(hist), dtype=np.int64),
                        candidate_item_ids=np.asarray(list(cand), dtype=np.int64))


def rows(ids, versions=None):
    versions = versions or {}
    return np.asarray([item_embedding(1234, int(i), versions.get(int(i), 0), CFG.hidden_dim) for i in ids]
                      ).reshape(len(ids), CFG.hidden_dim)


def service(mode, clock=None, **kw):
    return DeviceService(CFG, num_items=NUM_ITEMS, target_rows=256, precision="fp32",
                         cache=CacheConfig(mode=mode, ttl_s=5.0, **kw), clock=clock or Clock())


def test_cold_async_cache_scores_zero_embeddings_then_refreshed_rows(gpu):
    svc = service(CacheMode.ASYNC)
    try:
        req = request_of(range(8), range(300, 303))
        resp = svc.handle_request(req)  # every lookup is EMPTY: zero rows (reference test_service.py:53-62)
        want0 = orc.model_forward(np.zeros((8, 32)), np.zeros((3, 32)), svc.params, CFG)
        assert np.abs(resp.scores - want0).max() <= TOL
        svc.feature_cache.drain_refreshes()  # the background refreshes land
        resp = svc.handle_request(req)
        want = orc.model_forward(rows(range(8)), rows(range(300, 303)), svc.params, CFG)
        assert np.abs(resp.scores - want).max() <= TOL
        c = svc.metrics_snapshot()["cache"]
        assert (c["misses"], c["hits_fresh"], c["remote_queries"]) == (11, 11, 11)
    finally:
        svc.close()


def test_sync_cache_fresh_values_and_ttl(gpu):
    clock = Clock()
    svc = service(CacheMode.SYNC, clock)
    try:
        req = request_of(range(16), range(200, 221))
        base = orc.model_forward(rows(range(16)), rows(range(200, 221)), svc.params, CFG)
        assert np.abs(svc.handle_request(req).scores - base).max() <= TOL
        svc.mutate([205])  # store version advances; the cached row stays until the TTL expires
        assert np.abs(svc.handle_request(req).scores - base).max() <= TOL
        clock.now += 5.1
        new = orc.model_forward(rows(range(16)), rows(range(200, 221), {205: 1}), svc.params, CFG)
        got = svc.handle_request(req).scores
        assert np.abs(got - new).max() <= TOL
        assert np.abs(got[5] - base[5]).max() > 1e-6  # candidate 205 changed
    finally:
        svc.close()


def test_lru_eviction_reads_as_empty(gpu):
    # a capacity-1 single-bucket sync cache: each lookup evicts the previous key;
    # a later request for an evicted key misses and is fetched again
    svc = service(CacheMode.SYNC, bucket_count=1, capacity_per_bucket=1)
    try:
        req = request_of([], [7])
        want = orc.model_forward(np.zeros((0, 32)), rows([7]), svc.params, CFG)
        assert np.abs(svc.handle_request(req).scores - want).max() <= TOL
        svc.handle_request(request_of([], [9]))  # evicts 7
        assert svc.feature_cache.bucket_keys(0) == [9]
        # 7 again: a miss, fetched and written again before the batch runs
        assert np.abs(svc.handle_request(req).scores - want).max() <= TOL
        assert svc.metrics_snapshot()["cache"]["misses"] == 3
    finally:
        svc.close()


def test_concurrent_callers_with_async_refreshes(gpu):
    # 8 threads scoring while background refreshes land: no request fails, every
    # score is finite, and once the refreshes have drained the same requests score
    # exactly what a resident (always-fresh) table scores
    import threading

    svc = DeviceService(CFG, num_items=NUM_ITEMS, target_rows=256, precision="fp32",
                        cache=CacheConfig(mode=CacheMode.ASYNC, ttl_s=1e9))
    ref = DeviceService(CFG, num_items=NUM_ITEMS, target_rows=256, precision="fp32")
    rng = np.random.default_rng(3)
    reqs = [request_of(rng.integers(0, NUM_ITEMS, 2 * int(rng.integers(0, 33))),
                       rng.integers(0, NUM_ITEMS, int(rng.integers(1, 33)))) for _ in range(64)]
    errors = []

    def worker(k):
        try:
            for req in reqs[k::8]:
                out = svc.handle_request(req).scores
                assert np.isfinite(out).all()
        except BaseException as exc:  # noqa: BLE001
            errors.append(exc)

    try:
        threads = [threading.Thread(target=worker, args=(k,)) for k in range(8)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        assert not errors, errors[0]
        svc.feature_cache.drain_refreshes()
        for req in reqs:
            svc.handle_request(req)  # lookups after the drain: every key fresh, rows written
        for req in reqs:
            np.testing.assert_allclose(svc.handle_request(req).scores, ref.handle_request(req).scores,
                                       rtol=0, atol=1e-6)
    finally:
        svc.close()
        ref.close()


def test_pushed_values_fill_the_cache(gpu):
    # refresh_values behind the cache is a cache fill (reference FeatureCache.put):
    # the next lookup of the key is a fresh hit on the pushed value
    svc = service(CacheMode.SYNC)
    try:
        req = request_of(range(4), [50, 51])
        base = svc.handle_request(req).scores
        new = rows([51], {51: 3})[0]
        svc.refresh_values([51], [new.astype("<f8").tobytes() + b"\0" * 64])
        got = svc.handle_request(req).scores
        want = orc.model_forward(rows(range(4)), np.stack([rows([50])[0], new]), svc.params, CFG)
        assert np.abs(got - want).max() <= TOL
        assert np.abs(got[1] - base[1]).max() > 1e-6
        assert svc.metrics_snapshot()["cache"]["misses"] == 6  # the pushed key was not fetched
    finally:
        svc.close()
