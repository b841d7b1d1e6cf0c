"""The feature cache in front of the HBM table (§8(f)2) against the reference's
cache acceptance suite (tests/test_acceptance.py:155-272, criterion C4):
single-flight async refresh, non-blocking async under a slow store, sync
freshness after a store mutation, and LRU trace equivalence with a single-list
reference over 1e5 operations per bucket configuration.  Host-only: the device
side of the cache is the queue of row writes, checked here too."""

import threading
import time
from collections import defaultdict

import numpy as np
import pytest

from paper_2509_22681_b200.feature_cache import (CacheConfig, CacheMode, DeviceFeatureCache, Freshness,
                                                 item_key_hash)
from paper_2509_22681_b200.pda import item_embedding


class Clock:
    def __init__(self):
        self.now = 0.0

    def __call__(self):
        return self.now


class Store:
    """Stand-in for SimulatedRemoteStore (store.py:81-127): versioned deterministic
    values in the wire format, fixed latency, fetch instrumentation."""

    def __init__(self, dim=4, latency_s=0.0, bytes_per_value=64, seed=1):
        self.dim, self.latency_s, self.bpv, self.seed = dim, latency_s, bytes_per_value, seed
        self.versions = defaultdict(int)
        self.lock = threading.Lock()
        self.fetch_calls = 0
        self.in_flight = defaultdict(int)
        self.max_concurrent = defaultdict(int)
        self.abort = threading.Event()

    def value_for(self, i):
        raw = item_embedding(self.seed, i, self.versions[i], self.dim).astype("<f8").tobytes()
        return raw + b"\0" * max(0, self.bpv - len(raw))

    def mutate(self, i):
        with self.lock:
            self.versions[i] += 1

    def fetch(self, i):
        with self.lock:
            self.fetch_calls += 1
            self.in_flight[i] += 1
            self.max_concurrent[i] = max(self.max_concurrent[i], self.in_flight[i])
        try:
            if self.latency_s > 0:
                self.abort.wait(self.latency_s)
            return self.value_for(i)
        finally:
            with self.lock:
                self.in_flight[i] -= 1

    def decode(self, v):
        if len(v) < 8 * self.dim:
            return np.zeros(self.dim)
        return np.frombuffer(v[: 8 * self.dim], dtype="<f8")


def make(store, clock=None, **kw):
    return DeviceFeatureCache(CacheConfig(**kw), store.fetch, store.decode, clock=clock or time.monotonic)


def test_single_flight_async_refresh():
    clock, store = Clock(), Store(latency_s=0.005)
    cache = make(store, clock, bucket_count=4, capacity_per_bucket=16, ttl_s=10.0, mode=CacheMode.ASYNC)
    cache.put(42, b"old")
    clock.now += 60.0
    threads = [threading.Thread(target=cache.get_async, args=(42,)) for _ in range(32)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    cache.drain_refreshes()
    assert store.fetch_calls == 1
    assert store.max_concurrent[42] <= 1
    cache.close()


def test_async_never_blocks_on_a_slow_store():
    store = Store(latency_s=10.0)
    cache = make(store, bucket_count=4, capacity_per_bucket=16, ttl_s=10.0, mode=CacheMode.ASYNC)
    t0 = time.perf_counter()
    out = cache.get_async(7)
    assert time.perf_counter() - t0 < 1.0
    assert out.status is Freshness.EMPTY and out.value == b""
    store.abort.set()
    cache.drain_refreshes()
    cache.close()


def test_sync_freshness_after_mutation():
    clock, store = Clock(), Store(seed=3)
    cache = make(store, clock, bucket_count=4, capacity_per_bucket=16, ttl_s=5.0, mode=CacheMode.SYNC)
    stale = cache.get_sync(11)
    store.mutate(11)
    clock.now += 5.1
    fresh = cache.get_sync(11)
    assert fresh != stale and fresh == store.value_for(11)
    cache.close()


@pytest.mark.parametrize("bucket_count,capacity", [(1, 8), (4, 16), (16, 32)])
def test_lru_trace_equivalence(bucket_count, capacity):
    rng = np.random.default_rng(bucket_count * 1000 + capacity)
    store = Store(dim=1, bytes_per_value=16, seed=4)
    cache = make(store, bucket_count=bucket_count, capacity_per_bucket=capacity, ttl_s=1e9, mode=CacheMode.SYNC)
    ref = {b: [] for b in range(bucket_count)}
    universe = bucket_count * capacity * 4
    ops = rng.integers(0, 2, 100_000)
    picks = rng.integers(0, universe, 100_000)
    for op, k in zip(ops.tolist(), picks.tolist()):
        lst = ref[cache.bucket_index(k)]
        if op == 0:
            cache.put(k, b"v")
            if k in lst:
                lst.remove(k)
            lst.append(k)
            if len(lst) > capacity:
                lst.pop(0)
        elif k in lst:
            cache.get_sync(k)
            lst.remove(k)
            lst.append(k)
    for b in range(bucket_count):
        assert cache.bucket_keys(b) == ref[b], f"bucket {b} diverged"
    cache.close()


def test_bucket_hash_is_the_reference_feature_key_hash():
    # FeatureKey(ITEM, 0).stable_hash() as the reference computes it (cache.py:43-75;
    # checked for ids 0..999 against the installed reference)
    assert item_key_hash(0) == 0xDF30F36F6B91D29C
    assert len({item_key_hash(i) % 64 for i in range(5000)}) == 64


def test_batch_rows_are_the_lookup_results():
    store = Store(dim=4)
    cache = make(store, bucket_count=1, capacity_per_bucket=2, ttl_s=100.0, mode=CacheMode.SYNC)
    ids, rows = cache.lookup_lists([np.array([5, 3, 5]), np.array([9])])  # per list: unique ascending
    got = dict(zip(ids.tolist(), rows))
    assert set(got) == {3, 5, 9}
    for k in (3, 5, 9):  # 3 is evicted by 9 afterwards, but this batch resolved its value
        np.testing.assert_allclose(got[k], store.decode(store.value_for(k)).astype(np.float32))
    assert cache.bucket_keys(0) == [5, 9]
    assert cache.lookup_lists([np.array([5, 9])]) is None  # fresh hits: rows already hold them
    st = cache.stats()
    assert (st.misses, st.hits_fresh, st.remote_queries, st.bytes_fetched) == (3, 2, 3, 3 * 64)
    ids, rows = cache.lookup_lists([np.array([3])])  # evicted: a miss, fetched again
    assert ids.tolist() == [3]
    cache.close()


def test_async_batch_reads_empty_until_a_later_lookup():
    store = Store(dim=4)
    cache = make(store, bucket_count=4, capacity_per_bucket=8, ttl_s=100.0, mode=CacheMode.ASYNC)
    assert cache.lookup_lists([np.array([1, 2])]) is None  # cold: EMPTY = the zero rows already there
    cache.drain_refreshes()
    ids, rows = cache.lookup_lists([np.array([1, 2])])  # refreshed: fresh hits, rows written now
    assert sorted(ids.tolist()) == [1, 2] and np.abs(rows).sum() > 0
    cache.close()


def test_write_plans_follow_the_order_they_are_applied_in():
    # two batches resolve an id to different values (a refresh landed in between);
    # whichever plan is applied last is what the row record says, so a later batch
    # that resolves the other value rewrites the row (the device service makes and
    # applies the plans under one lock)
    store = Store(dim=4)
    cache = make(store, bucket_count=1, capacity_per_bucket=8, ttl_s=100.0, mode=CacheMode.SYNC)
    seen_a = cache.resolve_lists([np.array([7])])
    cache.put(7, b"")  # the value changes (EMPTY) before the second batch resolves it
    seen_b = cache.resolve_lists([np.array([7])])
    assert seen_b[7] == b"" and seen_a[7] != b""
    assert cache.device_writes(seen_b) is None  # EMPTY = the zero row already there
    ids, rows = cache.device_writes(seen_a)  # applied last: the row now holds a's value
    assert ids.tolist() == [7] and np.abs(rows).sum() > 0
    ids, rows = cache.device_writes(cache.resolve_lists([np.array([7])]))  # EMPTY again: zero row written
    assert ids.tolist() == [7] and np.abs(rows).sum() == 0
    cache.close()
