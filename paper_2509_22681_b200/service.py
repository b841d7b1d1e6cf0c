"""Device-resident request path: the reference ``Service.handle_request``
(pkg/src/flameserve/service.py:127-171) with its feature path moved into HBM.

The reference resolves every request's item ids through a host feature cache
in front of a (simulated) remote store, packs the embeddings, and hands them to
the runner.  Here the store's embeddings live in a device item table (row =
item id, the store's value for version 0, ``store.py:59-78``), the id lists go
to the GPU in pinned staging buffers (only the slots in use), and the PDA
kernels deduplicate and gather the rows on the device before the forward pass
(``DeviceExecutor.score_ids``).  Requests are batched through the DSO
(``BucketScheduler``): ``handle_batch`` scores many requests with one graph
replay per shape group.

Names, validation and errors follow the reference: ``ScoreRequest`` /
``ScoreResponse``, ``RequestError(ValueError)`` (HTTP 400) for contract
violations (``service.py:115-125``), ``ServiceClosedError(RuntimeError)`` (503)
after ``close``.  The reference store resolves every id deterministically
(``item_embedding``, ``store.py:59-63``), so a request holding ids outside the
device table (negative, or >= ``num_items``) is resolved on the host with the
same store function and scored through the embedding path; its scores equal
what the reference serves for those ids.  ``mutate`` mirrors ``SimulatedRemoteStore.mutate``
(``store.py:104-108``): the key's version advances and its row is refreshed in
HBM at once (the incremental-refresh path of SURVEY §8f.2), so later requests
see the new features.

Concurrent callers are coalesced: while one thread's batch runs on the device,
requests arriving from other threads queue up, and the next free caller scores
the whole queue as one DSO batch (leader / follower, no extra thread).  The
reference's ablation toggles map onto the device path (``ServiceConfig``,
``config.py:53-99``): ``cache_enabled`` = features resident in the HBM item
table (off: the host resolves every id from its store copy and ships fp32 rows),
``mem_opt`` = pinned staging with async copies (off: pageable, synchronous),
``routing`` = ``explicit`` DSO buckets with graphs vs ``implicit`` exact-shape
executors built per request (reference ``ImplicitShapeRunner``).

Feature cache.  By default the HBM table is resident and
always fresh (every id reads the store's current value; ``mutate`` refreshes the
rows at once).  With ``cache=CacheConfig(...)`` the table becomes the value
store of the reference's feature cache (``feature_cache.DeviceFeatureCache``,
cache.py:170-357): it starts cold (zero rows = EMPTY values), every request's
ids go through the cache's sync single-flight or async stale-while-revalidate
lookups in the reference's order, fetched values and LRU evictions become row
writes applied before the batch is submitted, and ``mutate`` only advances the
store version, so changed features arrive when the TTL expires — the reference
service's semantics, cold-async zero embeddings included.

Out of scope (host harness without device arithmetic): simulated
store latency and the transfer cost model.
"""

from __future__ import annotations

import threading
import time
from dataclasses import dataclass, field, replace

import numpy as np

from .config import ModelConfig
from .engine import DeviceExecutor, FlameEngine
from .feature_cache import EMPTY_VALUE, CacheConfig, DeviceFeatureCache
from .orchestrator import BucketScheduler
from .params import ModelParams, init_params, load_params
from .pda import DEFAULT_STORE_SEED, build_item_table, item_embedding

ROUTINGS = ("explicit", "implicit")


class RequestError(ValueError):
    """The request violates the wire contract; maps to a 400-class response."""


class ServiceClosedError(RuntimeError):
    """The service is draining or shut down."""


@dataclass(frozen=True)
class ScoreRequest:
    user_id: int
    history_item_ids: np.ndarray
    candidate_item_ids: np.ndarray
    context: dict = field(default_factory=dict)


@dataclass(frozen=True)
class ScoreResponse:
    scores: np.ndarray  # (C, num_tasks)
    overall_latency_ms: float
    compute_latency_ms: float


@dataclass(frozen=True)
class ServiceConfig:
    """The device service's deployment knobs.  ``from_dict`` reads the
    reference's service JSON (``config.py:53-91``: ``model``, ``cache_enabled``,
    ``mem_opt``, ``orchestrator.routing`` / ``profile_shapes``, ``params_path``);
    keys of the reference's host harness (cache TTLs, store latency, bandwidth
    table, listen address) are accepted and ignored."""

    model: ModelConfig
    num_items: int = 100_000
    store_seed: int = DEFAULT_STORE_SEED
    cache_enabled: bool = True
    mem_opt: bool = True
    routing: str = "explicit"
    profile_shapes: tuple = ()  # candidate counts warmed at startup, at max_history_len
    params_path: str | None = None
    table_dtype: str = "fp32"
    precision: str = "bf16"
    target_rows: int = 16384
    max_batch: int = 256  # requests coalesced into one dispatch
    cache: CacheConfig | None = None  # reference feature-cache semantics over the table (None: resident)
    bytes_per_value: int = 512  # store value size (store.py:29), for the fetched-bytes counters

    def __post_init__(self) -> None:
        if self.routing not in ROUTINGS:
            raise ValueError(f"routing must be one of {ROUTINGS}, got {self.routing!r}")
        if self.num_items < 1 or self.max_batch < 1:
            raise ValueError("num_items and max_batch must be >= 1")

    @classmethod
    def from_dict(cls, d: dict) -> "ServiceConfig":
        model = d["model"]
        kw = {"model": model if isinstance(model, ModelConfig) else ModelConfig.from_dict(model)}
        orch = d.get("orchestrator", {})
        if "routing" in orch:
            kw["routing"] = str(orch["routing"])
        if "profile_shapes" in orch:
            kw["profile_shapes"] = tuple(int(x) for x in orch["profile_shapes"])
        for k in ("cache_enabled", "mem_opt"):
            if k in d:
                kw[k] = bool(d[k])
        if isinstance(d.get("cache"), CacheConfig):
            kw["cache"] = d["cache"]
        elif isinstance(d.get("cache"), dict) and d.get("cache_semantics", True):
            kw["cache"] = CacheConfig.from_dict(d["cache"])
        if "bytes_per_value" in d.get("remote_store", {}):
            kw["bytes_per_value"] = int(d["remote_store"]["bytes_per_value"])
        for k in ("num_items", "store_seed", "target_rows", "max_batch"):
            if k in d:
                kw[k] = int(d[k])
        for k in ("params_path", "table_dtype", "precision", "routing"):
            if k in d:
                kw[k] = d[k]
        return cls(**kw)

    def with_ablation(self, cache: bool, mem_opt: bool, routing: str) -> "ServiceConfig":
        return replace(self, cache_enabled=cache, mem_opt=mem_opt, routing=routing)


def _percentile(values, q: float) -> float:
    """Nearest-rank percentile (reference metrics.py:11-19)."""
    s = sorted(values)
    k = max(1, int(np.ceil(q * len(s))))
    return s[k - 1]


class _Ticket:
    """One queued request of the coalescing dispatcher."""

    __slots__ = ("hist", "cand", "scores", "lat", "error", "done")

    def __init__(self, hist, cand) -> None:
        self.hist, self.cand = hist, cand
        self.scores = None
        self.lat = 0.0
        self.error = None
        self.done = False


class DeviceService:
    """One model deployment on one B200: weights, item table, DSO executors."""

    def __init__(self, config: ModelConfig, params: ModelParams | None = None, *, num_items: int = 100_000,
                 store_seed: int = DEFAULT_STORE_SEED, table: np.ndarray | None = None,
                 table_dtype: str = "fp32", precision: str = "bf16", device=None,
                 target_rows: int = 16384, cache_enabled: bool = True, mem_opt: bool = True,
                 routing: str = "explicit", max_batch: int = 256, cache: CacheConfig | None = None,
                 bytes_per_value: int = 512, clock=time.monotonic) -> None:
        if routing not in ROUTINGS:
            raise ValueError(f"routing must be one of {ROUTINGS}, got {routing!r}")
        self.config = config
        self.params = params if params is not None else init_params(config)
        self.store_seed = store_seed
        self.cache_enabled, self.mem_opt, self.routing = cache_enabled, mem_opt, routing
        self.max_batch = max_batch
        self.engine = FlameEngine(self.params, config, precision=precision, device=device)
        if table is None:
            table = build_item_table(num_items, config.hidden_dim, store_seed)
        # the store's current values; the device table mirrors it (cache on) or
        # the host resolves requests from it (cache off)
        self._store = np.array(table, dtype=np.float32)
        self.num_items = self._store.shape[0]
        self._versions: dict[int, int] = {}
        self.bytes_per_value = bytes_per_value
        self.feature_cache = None
        if cache is not None:
            # the table is the cache's value store: cold = every row EMPTY (zeros)
            self.feature_cache = DeviceFeatureCache(cache, self._fetch_value, self._decode_value, clock=clock)
            self.engine.set_table(np.zeros_like(self._store), dtype=table_dtype)
        else:
            self.engine.set_table(self._store, dtype=table_dtype)
        self.scheduler = BucketScheduler(self.engine, target_rows=target_rows, with_ids=True, pinned=mem_opt)
        self._lock = threading.Lock()  # device work vs. table refresh
        self._closed = False
        self._inflight = 0
        self._drained = threading.Condition(threading.Lock())
        self._queue: list = []
        self._leader = False
        self._in_flight = 0  # batches taken by a leader and not yet completed
        self._on_device = 0  # of those, batches submitted to the GPU
        self.max_inflight = 2
        self._cv = threading.Condition(threading.Lock())
        self._overall_ms: list = []
        self._compute_ms: list = []
        self._stats_lock = threading.Lock()
        self.requests_total = 0
        self.pairs_processed = 0
        self.lookups = 0
        self.hits = 0
        self.feature_bytes = 0  # feature data moved host -> device (ids, rows, refreshes)
        self.dispatches = 0  # coalesced batches run
        self._implicit_allocs = 0
        self._alloc_base = 0

    @classmethod
    def from_config(cls, cfg: ServiceConfig, device=None) -> "DeviceService":
        params = None
        if cfg.params_path:
            file_cfg, params = load_params(cfg.params_path)
            if file_cfg != cfg.model:
                raise ValueError(f"{cfg.params_path} holds parameters of a different model config")
        svc = cls(cfg.model, params, num_items=cfg.num_items, store_seed=cfg.store_seed,
                  table_dtype=cfg.table_dtype, precision=cfg.precision, device=device,
                  target_rows=cfg.target_rows, cache_enabled=cfg.cache_enabled, mem_opt=cfg.mem_opt,
                  routing=cfg.routing, max_batch=cfg.max_batch, cache=cfg.cache,
                  bytes_per_value=cfg.bytes_per_value)
        if cfg.profile_shapes:
            svc.warm([(cfg.model.max_history_len, c) for c in cfg.profile_shapes])
        return svc

    def warm(self, shapes) -> None:
        """Build the executors of the buckets of ``shapes`` ((H, C) pairs) now;
        allocations after the last ``warm`` count as steady-state allocations."""
        if self.routing == "explicit":
            with self._lock:
                self.scheduler.warm(shapes)
                self._alloc_base = self.scheduler.allocations

    # -- request path ---------------------------------------------------------

    def _validate(self, req: ScoreRequest) -> None:
        """Reference Service._validate (service.py:115-125)."""
        model = self.config
        c = len(req.candidate_item_ids)
        h = len(req.history_item_ids)
        if c < 1:
            raise RequestError("candidates must be non-empty")
        if c > model.max_candidates:
            raise RequestError(f"candidate count {c} exceeds max {model.max_candidates}")
        if h > model.max_history_len:
            raise RequestError(f"history length {h} exceeds max {model.max_history_len}")
        if h % model.num_blocks != 0:
            raise RequestError(f"history length {h} must be a multiple of num_blocks {model.num_blocks}")

    def handle_request(self, req: ScoreRequest) -> ScoreResponse:
        return self.handle_batch([req])[0]

    def handle_batch(self, reqs) -> list[ScoreResponse]:
        """Score many requests at once; per-request compute latency runs from the
        dispatch of the request's batch to the collection of its group."""
        t0 = time.perf_counter()
        for r in reqs:
            self._validate(r)
        with self._drained:
            if self._closed:
                raise ServiceClosedError("service is shut down")
            self._inflight += 1
        try:
            tickets = [_Ticket(np.asarray(r.history_item_ids, dtype=np.int64),
                               np.asarray(r.candidate_item_ids, dtype=np.int64)) for r in reqs]
            self._dispatch(tickets)
            for t in tickets:
                if t.error is not None:
                    raise t.error
            t1 = time.perf_counter()
            out = [ScoreResponse(t.scores, (t1 - t0) * 1000.0, t.lat * 1000.0) for t in tickets]
            with self._stats_lock:
                for r, o in zip(reqs, out):
                    self._overall_ms.append(o.overall_latency_ms)
                    self._compute_ms.append(o.compute_latency_ms)
                    self.requests_total += 1
                    self.pairs_processed += len(r.candidate_item_ids)
            return out
        finally:
            with self._drained:
                self._inflight -= 1
                self._drained.notify_all()

    def _dispatch(self, tickets) -> None:
        """Leader / follower coalescing with up to ``max_inflight`` batches on the
        device: the tickets are queued; a caller that finds no submission in
        progress and a free in-flight slot takes up to ``max_batch`` queued
        tickets (anyone's), submits them, hands the leader role on, then waits
        for that batch and completes its tickets.  While one batch runs on the
        GPU the next one is staged and submitted, and requests that arrive
        meanwhile form the batch after it."""
        with self._cv:
            self._queue.extend(tickets)
        while True:
            with self._cv:
                self._cv.wait_for(lambda: all(t.done for t in tickets)
                                  or (self._queue and not self._leader and self._in_flight < self.max_inflight))
                if all(t.done for t in tickets):
                    return
                self._leader = True
            owned = []
            try:
                while True:  # submit while there is queued work and an in-flight slot
                    with self._cv:
                        if not self._queue or self._in_flight >= self.max_inflight:
                            break
                        self._in_flight += 1
                        batch, self._queue = self._queue[: self.max_batch], self._queue[self.max_batch:]
                    try:
                        owned.append((batch, self._submit(batch)))
                    except BaseException as exc:  # noqa: BLE001 - surfaced to each ticket's caller
                        for t in batch:
                            t.error = exc
                        owned.append((batch, None))
            finally:
                with self._cv:
                    self._leader = False
                    self._cv.notify_all()
            for batch, handle in owned:
                try:
                    if handle is not None:
                        self._complete(batch, handle)
                except BaseException as exc:  # noqa: BLE001
                    for t in batch:
                        t.error = exc
                finally:
                    with self._cv:
                        for t in batch:
                            t.done = True
                        self._in_flight -= 1
                        self._cv.notify_all()

    def _host_rows(self, ids: np.ndarray) -> np.ndarray:
        """The store's rows for ``ids``, resolved on the host: table ids from the
        store copy, any other id from the store function (store.py:59-63)."""
        rows = np.zeros((ids.size, self.config.hidden_dim), dtype=np.float32)
        ok = (ids >= 0) & (ids < self.num_items)
        rows[ok] = self._store[ids[ok]]
        for k in np.flatnonzero(~ok):
            rows[k] = self.embedding_of(int(ids[k]))
        return rows

    def _in_table(self, t) -> bool:
        n = self.num_items
        return bool((t.hist.size == 0 or (t.hist.min() >= 0 and t.hist.max() < n))
                    and (t.cand.min() >= 0 and t.cand.max() < n))

    def _submit(self, batch):
        """Resolve the batch's features and submit it (explicit routing), or run
        it to completion (implicit routing).  Returns what ``_complete`` needs.
        With the cache on, requests whose ids all lie in the device table go as
        id lists (PDA on the device); the others are resolved on the host."""
        d = self.config.hidden_dim
        n_ids = sum(t.hist.size + t.cand.size for t in batch)
        on_dev = [self.cache_enabled and self._in_table(t) for t in batch]
        id_work = [(t.hist, t.cand) for t, f in zip(batch, on_dev) if f]
        row_work = [(self._host_rows(t.hist), self._host_rows(t.cand)) for t, f in zip(batch, on_dev) if not f]
        hits = sum(t.hist.size + t.cand.size for t, f in zip(batch, on_dev) if f)
        nbytes = 8 * hits + 4 * d * (n_ids - hits)
        with self._stats_lock:
            self.dispatches += 1
            self.lookups += n_ids
            self.hits += hits
            self.feature_bytes += nbytes
        order = [i for i, f in enumerate(on_dev) if f] + [i for i, f in enumerate(on_dev) if not f]
        resolved = []
        if self.feature_cache is not None:
            # reference resolve order: per request, history then candidates
            # (service.py:136-137), outside the lock (sync mode may wait on the store)
            resolved = [self.feature_cache.resolve_lists((t.hist, t.cand)) for t, f in zip(batch, on_dev) if f]
        with self._lock:
            # the rows each lookup resolved are written before the batch runs; the
            # write plan is made under the same lock as the writes, so two batches'
            # plans cannot land on the device in the opposite order
            writes: dict = {}
            for seen in resolved:
                w = self.feature_cache.device_writes(seen)
                if w is not None:
                    writes.update(zip(w[0].tolist(), w[1]))
            if writes:
                self._write_rows(writes)
            if self.routing == "explicit":
                recs = []
                for work, ids in ((id_work, True), (row_work, False)):
                    if work:
                        recs.append(self.scheduler.submit_batch(work, ids=ids))
                        with self._cv:
                            self._on_device += 1
                return ("rec", (order, recs))
            out = [self._run_implicit(h, c, True) for h, c in id_work]
            out += [self._run_implicit(h, c, False) for h, c in row_work]
            return ("done", (order, out))

    def _complete(self, batch, handle) -> None:
        kind, (order, obj) = handle
        scores, lat = [], []
        if kind == "rec":
            err = None
            for rec in obj:
                try:
                    s_, l_ = self.scheduler.collect_batch(rec)
                    scores += s_
                    lat += l_
                except BaseException as exc:  # noqa: BLE001 - every rec is collected first
                    err = err or exc
                finally:
                    with self._cv:
                        self._on_device -= 1
                        self._cv.notify_all()
            if err is not None:
                raise err
        else:
            scores, lat = [s for s, _ in obj], [l for _, l in obj]
        for i, s_, l_ in zip(order, scores, lat):
            batch[i].scores, batch[i].lat = s_, l_

    def _quiesce(self) -> None:
        """Wait until the device has finished every submitted batch (caller holds
        ``_lock``, so no new batch can be submitted).  This waits on the DEVICE, not
        on the batches' collection: a leader thread may hold a submitted batch it
        will only collect after its next submission, which needs ``_lock``."""
        import torch

        torch.cuda.synchronize(self.engine.device)

    def _run_implicit(self, hist, cand, ids: bool):
        """Reference ImplicitShapeRunner (orchestrator.py:225-260): exact-shape
        buffers allocated for the request, eager launch, released afterwards."""
        ex = DeviceExecutor(self.engine, 1, len(hist) // self.config.num_blocks, len(cand),
                            with_ids=ids, pinned=self.mem_opt)
        self._implicit_allocs += ex.allocations
        try:
            t0 = time.perf_counter()
            if ids:
                s = ex.score_ids([(hist, cand)], graph=False)[0]
            else:
                s = ex.score([(hist, cand)], graph=False)[0]
            return s, time.perf_counter() - t0
        finally:
            ex.close()

    @property
    def steady_state_allocations(self) -> int:
        if self.routing == "implicit":
            return self._implicit_allocs
        return self.scheduler.allocations - self._alloc_base

    # -- feature path ---------------------------------------------------------

    def _fetch_value(self, item_id: int) -> bytes:
        """The store's value for an item (store.py:85-102 minus the latency model):
        the current embedding in the wire format, fp64 LE + filler."""
        raw = self.embedding_of(item_id).astype("<f8").tobytes()
        return raw + b"\x00" * max(0, self.bytes_per_value - len(raw))

    def _decode_value(self, value) -> np.ndarray:
        """store.py:74-78: values shorter than d float64s decode to zeros."""
        d = self.config.hidden_dim
        if len(value) < 8 * d:
            return np.zeros(d, dtype=np.float32)
        return np.frombuffer(value[: 8 * d], dtype="<f8").astype(np.float32)

    def _write_rows(self, writes: dict) -> None:
        """Write feature-cache rows {id: row} into the device table (caller holds
        ``_lock``; waits for the batches on the device first)."""
        ids = np.fromiter(writes.keys(), dtype=np.int64, count=len(writes))
        rows = np.stack(list(writes.values())).astype(np.float32, copy=False)
        self._quiesce()
        self.engine.update_rows(ids, rows)
        with self._stats_lock:
            self.feature_bytes += int(rows.size) * 4

    def cache_stats(self):
        """Reference Service.cache_stats (service.py:176-177); None without a cache."""
        return self.feature_cache.stats() if self.feature_cache is not None else None

    def embedding_of(self, item_id: int) -> np.ndarray:
        """The store's current embedding of an item (store.py:59-63, any id)."""
        return item_embedding(self.store_seed, int(item_id), self._versions.get(int(item_id), 0),
                              self.config.hidden_dim)

    def mutate(self, item_ids) -> None:
        """Advance the items' versions (reference store.mutate) and refresh their
        rows in the device table.  The version bump, the row computation and the
        device update happen under one lock, so concurrent mutates of one id
        cannot leave the table behind ``_versions``."""
        ids = [int(i) for i in np.atleast_1d(item_ids)]
        if not ids:
            return
        with self._lock:
            for i in ids:
                self._versions[i] = self._versions.get(i, 0) + 1
            if self.feature_cache is not None:
                # behind a feature cache the new values arrive through its refreshes
                return
            tab = sorted({i for i in ids if 0 <= i < self.num_items})
            if not tab:
                return
            rows = np.stack([self.embedding_of(i) for i in tab])
            self._quiesce()
            self._store[tab] = rows
            self.engine.update_rows(np.asarray(tab, dtype=np.int64), rows)
        with self._stats_lock:
            self.feature_bytes += rows.size * 4

    def refresh_values(self, item_ids, values) -> None:
        """Write raw store feature values (reference wire format, store.py:66-78:
        float64 LE embedding + filler; empty -> zero row) into the device table,
        decoded on the GPU — the path a store feed / cache refresh would use."""
        ids = np.asarray(item_ids, dtype=np.int64).reshape(-1)
        values = list(values)
        d = self.config.hidden_dim
        if self.feature_cache is not None:
            # behind the feature cache a pushed value is a cache fill (cache.py:321-325
            # put): the row is written when a lookup next resolves the key
            for i, v in zip(ids.tolist(), values):
                self.feature_cache.put(i, bytes(v))
            with self._stats_lock:
                self.feature_bytes += sum(len(v) for v in values)
            return
        with self._lock:
            self._quiesce()
            self.engine.update_values(ids, values)
            for i, v in zip(ids, values):
                if 0 <= i < self.num_items:
                    self._store[i] = np.frombuffer(v[: 8 * d], dtype="<f8") if len(v) >= 8 * d else 0.0
        with self._stats_lock:
            self.feature_bytes += sum(len(v) for v in values)

    # -- observability / lifecycle --------------------------------------------

    def metrics_snapshot(self) -> dict:
        """Reference /metrics fields (api.py:60-66): request counts, latency
        summaries, cache hit rate, feature bytes moved, steady-state allocations."""
        def summary(series):
            if not series:
                return {"count": 0}
            return {"count": len(series), "mean": sum(series) / len(series),
                    "p50": _percentile(series, 0.5), "p99": _percentile(series, 0.99)}

        cache = {"enabled": self.cache_enabled, "lookups": self.lookups,
                 "hit_rate": self.hits / self.lookups if self.lookups else 0.0}
        st = self.cache_stats()
        if st is not None:
            n = st.hits_fresh + st.hits_stale + st.misses
            cache.update(hits_fresh=st.hits_fresh, hits_stale=st.hits_stale, misses=st.misses,
                         remote_queries=st.remote_queries, bytes_fetched=st.bytes_fetched,
                         hit_rate=(st.hits_fresh + st.hits_stale) / n if n else 0.0)
        with self._stats_lock:
            return {"requests_total": self.requests_total, "pairs_processed": self.pairs_processed,
                    "overall_ms": summary(self._overall_ms), "compute_ms": summary(self._compute_ms),
                    "cache": cache,
                    "network_bytes": self.feature_bytes, "dispatches": self.dispatches,
                    "steady_state_allocs": self.steady_state_allocations}

    def close(self, drain_timeout_s: float = 30.0) -> None:
        """Stop accepting requests and wait for in-flight ones (service.py:222-233)."""
        with self._drained:
            self._closed = True
            deadline = time.monotonic() + drain_timeout_s
            while self._inflight > 0:
                remaining = deadline - time.monotonic()
                if remaining <= 0:
                    raise TimeoutError(f"{self._inflight} requests still in flight")
                self._drained.wait(timeout=remaining)
        if self.feature_cache is not None:
            self.feature_cache.close()
        self.scheduler.close()
        self.engine.close()
