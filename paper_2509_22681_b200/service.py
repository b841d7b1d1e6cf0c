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
after ``close``.  Unknown ids (outside the table) score as zero embeddings, as
an empty store value does in the reference (``decode_embedding``,
``store.py:74-78``).  ``mutate`` mirrors ``SimulatedRemoteStore.mutate``
(``store.py:104-108``): the key's version advances and its row is refreshed in
HBM at once (the incremental-refresh path of SURVEY §8f.2), so later requests
see the new features.

Out of scope (host harness without device arithmetic): the host
feature cache and its staleness modes, simulated store latency, the transfer
cost model, the HTTP layer.
"""

from __future__ import annotations

import threading
import time
from dataclasses import dataclass, field

import numpy as np

from .config import ModelConfig
from .engine import FlameEngine
from .orchestrator import BucketScheduler
from .params import ModelParams, init_params
from .pda import DEFAULT_STORE_SEED, build_item_table, item_embedding


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


def _percentile(values, q: float) -> float:
    """Nearest-rank percentile (reference metrics.py:11-19)."""
    s = sorted(values)
    k = max(1, int(np.ceil(q * len(s))))
    return s[k - 1]


class DeviceService:
    """One model deployment on one B200: weights, item table, DSO executors."""

    def __init__(self, config: ModelConfig, params: ModelParams | None = None, *, num_items: int = 100_000,
                 store_seed: int = DEFAULT_STORE_SEED, table: np.ndarray | None = None,
                 table_dtype: str = "fp32", precision: str = "bf16", device=None,
                 target_rows: int = 16384) -> None:
        self.config = config
        self.params = params if params is not None else init_params(config)
        self.store_seed = store_seed
        self.engine = FlameEngine(self.params, config, precision=precision, device=device)
        if table is None:
            table = build_item_table(num_items, config.hidden_dim, store_seed)
        self.engine.set_table(table, dtype=table_dtype)
        self.num_items = table.shape[0]
        self._versions: dict[int, int] = {}
        self.scheduler = BucketScheduler(self.engine, target_rows=target_rows, with_ids=True)
        self._lock = threading.Lock()  # scoring vs. table refresh
        self._closed = False
        self._inflight = 0
        self._drained = threading.Condition(threading.Lock())
        self._overall_ms: list = []
        self._compute_ms: list = []
        self.requests_total = 0
        self.pairs_processed = 0

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
        """Score many requests at once through the DSO; per-request latencies are
        from the call to the collection of the request's group."""
        t0 = time.perf_counter()
        for r in reqs:
            self._validate(r)
        with self._drained:
            if self._closed:
                raise ServiceClosedError("service is shut down")
            self._inflight += 1
        try:
            batch = [(np.asarray(r.history_item_ids, dtype=np.int64), np.asarray(r.candidate_item_ids, dtype=np.int64))
                     for r in reqs]
            with self._lock:
                t1 = time.perf_counter()
                scores = self.scheduler.score(batch, ids=True)
                lat = list(self.scheduler.last_latencies)
            out = []
            for r, s, l in zip(reqs, scores, lat):
                overall = (t1 - t0 + l) * 1000.0
                out.append(ScoreResponse(s, overall, l * 1000.0))
                self._overall_ms.append(overall)
                self._compute_ms.append(l * 1000.0)
                self.requests_total += 1
                self.pairs_processed += len(r.candidate_item_ids)
            return out
        finally:
            with self._drained:
                self._inflight -= 1
                self._drained.notify_all()

    # -- feature path ---------------------------------------------------------

    def embedding_of(self, item_id: int) -> np.ndarray:
        """The store's current embedding of an item (zeros outside the table)."""
        if not 0 <= item_id < self.num_items:
            return np.zeros(self.config.hidden_dim)
        return item_embedding(self.store_seed, int(item_id), self._versions.get(int(item_id), 0),
                              self.config.hidden_dim)

    def mutate(self, item_ids) -> None:
        """Advance the items' versions (reference store.mutate) and refresh their
        rows in the device table."""
        ids = [int(i) for i in np.atleast_1d(item_ids) if 0 <= int(i) < self.num_items]
        if not ids:
            return
        for i in ids:
            self._versions[i] = self._versions.get(i, 0) + 1
        rows = np.stack([self.embedding_of(i) for i in ids])
        with self._lock:
            self.engine.update_rows(np.asarray(ids, dtype=np.int64), rows)

    def refresh_values(self, item_ids, values) -> None:
        """Write raw store feature values (reference wire format, store.py:66-78:
        float64 LE embedding + filler; empty -> zero row) into the device table,
        decoded on the GPU — the path a store feed / cache refresh would use."""
        with self._lock:
            self.engine.update_values(np.asarray(item_ids, dtype=np.int64), list(values))

    # -- observability / lifecycle --------------------------------------------

    def metrics_snapshot(self) -> dict:
        def summary(series):
            if not series:
                return {"count": 0}
            return {"count": len(series), "mean": sum(series) / len(series),
                    "p50": _percentile(series, 0.5), "p99": _percentile(series, 0.99)}

        return {"requests_total": self.requests_total, "pairs_processed": self.pairs_processed,
                "overall_ms": summary(self._overall_ms), "compute_ms": summary(self._compute_ms),
                "steady_state_allocs": 0}

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
        self.scheduler.close()
        self.engine.close()
