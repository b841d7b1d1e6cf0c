"""Process-per-GPU request dispatcher: one request stream served by N B200s.

Requests are independent (reference model/forward.py:186-204), so a box of N
GPUs serves one stream by routing WHOLE requests to per-GPU worker processes —
no collective on the scoring path.  Each worker owns one GPU and one
``DeviceService`` (weights, HBM item table, DSO executors, its own request
coalescing); the front end, in the caller's process, routes every request to the
worker with the least outstanding work (the ``sharding.request_work`` rows of the
requests it holds that have not come back — the online form of
``assign_requests``), and completes each caller's future when that worker's
result arrives.  This is the multi-device counterpart of the reference's
``Service.handle_request`` concurrency (service.py:127-171: a semaphore of
in-flight requests over one runner; orchestrator.py:163-165: a thread pool of
chunks).

Transport: one duplex pipe per worker; a group of requests travels as one frame
(tags, per-request lengths, and the concatenated history / candidate ids as
int64 arrays), a scored batch comes back as one message (tags, row counts, the
concatenated score rows, compute times) — ids, not embeddings, cross the process
boundary (the feature rows are gathered on the worker's GPU).  Inside a worker, a reader thread queues arriving requests and
two handler threads drain the queue into ``handle_batch`` calls, so one batch
is staged while the previous one runs on the device.

``scorer_factory(rank)`` builds a worker's scorer (anything with
``handle_batch(list[ScoreRequest]) -> list[ScoreResponse]`` and ``close()``);
the default builds ``DeviceService.from_config(config, device=rank)``.
"""

from __future__ import annotations

import multiprocessing as mp
import queue
import threading
import time
from concurrent.futures import Future

import numpy as np

from .sharding import request_work

_STOP = "stop"


class DispatchError(RuntimeError):
    """A worker failed to start or died."""


class ServiceFactory:
    """Default worker scorer: a DeviceService on GPU ``devices[rank]`` (``rank``
    when no device map is given); picklable for spawn."""

    def __init__(self, config, devices=None) -> None:
        self.config = config
        self.devices = list(devices) if devices is not None else None

    def __call__(self, rank: int):
        from .service import DeviceService

        return DeviceService.from_config(self.config, device=self.devices[rank] if self.devices else rank)


def _worker_main(rank: int, conn, factory, max_batch: int, handlers: int) -> None:
    """Worker process: own GPU ``rank``; serve requests from ``conn`` until stopped."""
    from .service import ScoreRequest

    try:
        scorer = factory(rank)
    except BaseException as exc:  # noqa: BLE001 - reported to the front end
        conn.send(("error", repr(exc)))
        return
    conn.send(("ready", rank))
    inbox: queue.Queue = queue.Queue()
    send_lock = threading.Lock()

    def handle() -> None:
        while True:
            item = inbox.get()
            if item is None:
                return
            batch = [item]
            while len(batch) < max_batch:
                try:
                    nxt = inbox.get_nowait()
                except queue.Empty:
                    break
                if nxt is None:
                    inbox.put(None)
                    break
                batch.append(nxt)
            reqs = [ScoreRequest(user_id=0, history_item_ids=h, candidate_item_ids=c) for _, h, c in batch]
            try:
                out = scorer.handle_batch(reqs)
                # one message for the whole batch: tags, per-request row counts, all score rows
                msgs = [("oks", np.array([b[0] for b in batch], dtype=np.int64),
                         np.array([o.scores.shape[0] for o in out], dtype=np.int64),
                         np.concatenate([o.scores for o in out]),
                         np.array([o.compute_latency_ms for o in out]))]
            except BaseException as exc:  # noqa: BLE001 - every request of the batch gets it
                if len(batch) > 1:  # isolate the failing request(s): retry one by one
                    msgs = []
                    for tag, r in zip((b[0] for b in batch), reqs):
                        try:
                            o = scorer.handle_batch([r])[0]
                            msgs.append(("ok", tag, o.scores, o.compute_latency_ms))
                        except BaseException as e1:  # noqa: BLE001
                            msgs.append(("err", tag, type(e1).__name__, str(e1)))
                else:
                    msgs = [("err", batch[0][0], type(exc).__name__, str(exc))]
            with send_lock:
                for m in msgs:
                    conn.send(m)

    threads = [threading.Thread(target=handle, daemon=True) for _ in range(handlers)]
    for t in threads:
        t.start()
    try:
        while True:
            msg = conn.recv()
            if msg == _STOP:
                break
            if msg[0] == "frame":  # several requests in one message (submit_many)
                _, tags, hl, cl, hflat, cflat = msg
                hs = np.split(hflat, np.cumsum(hl)[:-1])
                cs = np.split(cflat, np.cumsum(cl)[:-1])
                for tag, h, c in zip(tags.tolist(), hs, cs):
                    inbox.put((tag, h, c))
            else:
                inbox.put(msg)
    except EOFError:
        pass
    for _ in threads:
        inbox.put(None)
    for t in threads:
        t.join()
    try:
        scorer.close()
    finally:
        with send_lock:
            conn.send(("closed", rank))
        conn.close()


class MultiDeviceService:
    """Front end of N per-GPU workers with least-outstanding-work routing."""

    def __init__(self, config=None, n_devices: int = 1, *, scorer_factory=None, max_batch: int = 256,
                 handlers: int = 2, start_timeout_s: float = 600.0, devices=None) -> None:
        """``devices``: the GPU of each worker (default: worker k on GPU k); two
        workers may share a GPU (tests on a one-GPU box)."""
        if n_devices < 1:
            raise ValueError("n_devices must be >= 1")
        if devices is not None and len(devices) != n_devices:
            raise ValueError("devices must name one GPU per worker")
        if scorer_factory is None:
            if config is None:
                raise ValueError("a ServiceConfig or a scorer_factory is required")
            scorer_factory = ServiceFactory(config, devices)
        self.num_blocks = config.model.num_blocks if config is not None else 1
        ctx = mp.get_context("spawn")
        self._conns, self._procs = [], []
        for rank in range(n_devices):
            a, b = ctx.Pipe(duplex=True)
            p = ctx.Process(target=_worker_main, args=(rank, b, scorer_factory, max_batch, handlers), daemon=True)
            p.start()
            b.close()
            self._conns.append(a)
            self._procs.append(p)
        for rank, c in enumerate(self._conns):
            if not c.poll(start_timeout_s):
                self._kill()
                raise DispatchError(f"worker {rank} did not start within {start_timeout_s:.0f}s")
            msg = c.recv()
            if msg[0] != "ready":
                self._kill()
                raise DispatchError(f"worker {rank} failed to start: {msg[1]}")
        self.n = n_devices
        self._alive = [True] * n_devices  # a worker that exited or died takes no more requests
        self._lock = threading.Lock()
        self._send_locks = [threading.Lock() for _ in range(n_devices)]
        self._outstanding = [0] * n_devices
        self._pending: dict = {}
        self._tag = 0
        self.routed = [0] * n_devices  # requests sent to each worker
        self._stats_lock = threading.Lock()
        self._overall_ms: list = []
        self._compute_ms: list = []
        self.pairs_processed = 0
        self._closed = False
        self._readers = [threading.Thread(target=self._read, args=(r,), daemon=True) for r in range(n_devices)]
        for t in self._readers:
            t.start()

    def _kill(self) -> None:
        for p in self._procs:
            if p.is_alive():
                p.kill()

    def _read(self, rank: int) -> None:
        conn = self._conns[rank]
        while True:
            try:
                msg = conn.recv()
            except (EOFError, OSError):
                msg = ("died", rank)
            if msg[0] in ("closed", "died"):
                with self._lock:
                    self._alive[rank] = False
                    dead = [t for t, (r, _, _, _) in self._pending.items() if r == rank]
                    for tag in dead:
                        _, fut, _, _ = self._pending.pop(tag)
                        fut.set_exception(DispatchError(f"worker {rank} exited with requests in flight"))
                return
            if msg[0] == "oks":
                _, tags, counts, flat, ms = msg
                now = time.perf_counter()
                rows = np.split(flat, np.cumsum(counts)[:-1])
                done = []
                with self._lock:
                    for tag in tags.tolist():
                        r, fut, work, t0 = self._pending.pop(tag)
                        self._outstanding[r] -= work
                        done.append((fut, t0))
                for (fut, t0), sc, m in zip(done, rows, ms.tolist()):
                    fut.set_result((sc, m, now - t0))
                continue
            tag = msg[1]
            with self._lock:
                r, fut, work, t0 = self._pending.pop(tag)
                self._outstanding[r] -= work
            if msg[0] == "ok":
                fut.set_result((msg[2], msg[3], time.perf_counter() - t0))
            else:
                from .service import RequestError

                exc_t = RequestError if msg[2] == "RequestError" else (ValueError if msg[2] == "ValueError"
                                                                       else RuntimeError)
                fut.set_exception(exc_t(msg[3]))

    def submit(self, history_item_ids, candidate_item_ids) -> Future:
        """Route one request; the future yields (scores (C, tasks), compute ms,
        end-to-end seconds from submit to result)."""
        return self.submit_many([(history_item_ids, candidate_item_ids)])[0]

    def submit_many(self, requests) -> list:
        """Route a group of requests, each to the worker with the least outstanding
        work at its turn, and send each worker its share as ONE message (ids
        concatenated); returns one future per request, in order."""
        hs = [np.ascontiguousarray(h, dtype=np.int64).reshape(-1) for h, _ in requests]
        cs = [np.ascontiguousarray(c, dtype=np.int64).reshape(-1) for _, c in requests]
        futs = [Future() for _ in requests]
        per: dict = {}
        t0 = time.perf_counter()
        with self._lock:
            if self._closed:
                from .service import ServiceClosedError

                raise ServiceClosedError("dispatcher is closed")
            live = [q for q in range(self.n) if self._alive[q]]
            if not live:
                raise DispatchError("no live workers")
            for k, (h, c) in enumerate(zip(hs, cs)):
                work = request_work(h.size, c.size, self.num_blocks)
                rank = min(live, key=lambda q: (self._outstanding[q], q))
                self._outstanding[rank] += work
                self._tag += 1
                self._pending[self._tag] = (rank, futs[k], work, t0)
                self.routed[rank] += 1
                per.setdefault(rank, []).append((self._tag, k))
        for rank, items in per.items():
            tags = np.array([t for t, _ in items], dtype=np.int64)
            idx = [k for _, k in items]
            msg = ("frame", tags, np.array([hs[k].size for k in idx], dtype=np.int64),
                   np.array([cs[k].size for k in idx], dtype=np.int64),
                   np.concatenate([hs[k] for k in idx]), np.concatenate([cs[k] for k in idx]))
            try:
                with self._send_locks[rank]:
                    self._conns[rank].send(msg)
            except (BrokenPipeError, EOFError, OSError) as exc:
                # the worker went away between routing and sending: fail its share
                # now (its reader may already have drained the pending table)
                with self._lock:
                    self._alive[rank] = False
                    lost = [self._pending.pop(int(t)) for t in tags if int(t) in self._pending]
                    for r, _, work, _ in lost:
                        self._outstanding[r] -= work
                for _, fut, _, _ in lost:
                    fut.set_exception(DispatchError(f"worker {rank} is gone: {exc!r}"))
        return futs

    def score(self, requests) -> list:
        """Score (history ids, candidate ids) pairs; results in request order."""
        futs = self.submit_many(list(requests))
        return [f.result()[0] for f in futs]

    # -- the DeviceService request interface (so api.create_app can serve N GPUs)
    def handle_batch(self, reqs) -> list:
        """Reference ``Service.handle_request`` semantics for a list of
        ``ScoreRequest``s, routed over the workers: ``ScoreResponse``s in order;
        contract violations raise the workers' ``RequestError``."""
        from .service import ScoreResponse

        t0 = time.perf_counter()
        futs = self.submit_many([(r.history_item_ids, r.candidate_item_ids) for r in reqs])
        out = []
        for f in futs:
            scores, compute_ms, _ = f.result()
            out.append(ScoreResponse(scores, (time.perf_counter() - t0) * 1000.0, compute_ms))
        with self._stats_lock:
            for o in out:
                self._overall_ms.append(o.overall_latency_ms)
                self._compute_ms.append(o.compute_latency_ms)
                self.pairs_processed += o.scores.shape[0]
        return out

    def handle_request(self, req):
        return self.handle_batch([req])[0]

    def metrics_snapshot(self) -> dict:
        """Front-end view: request counts, latency summaries (nearest rank), the
        requests routed to each GPU worker."""
        from .service import _percentile

        def summary(series):
            if not series:
                return {"count": 0}
            return {"count": len(series), "mean": sum(series) / len(series),
                    "p50": _percentile(series, 0.5), "p99": _percentile(series, 0.99)}

        with self._stats_lock:
            return {"requests_total": len(self._overall_ms), "pairs_processed": self.pairs_processed,
                    "overall_ms": summary(self._overall_ms), "compute_ms": summary(self._compute_ms),
                    "routed_per_worker": list(self.routed), "workers": self.n}

    def outstanding(self) -> list:
        with self._lock:
            return list(self._outstanding)

    def alive(self) -> list:
        """Which workers still take requests."""
        with self._lock:
            return list(self._alive)

    def close(self, timeout_s: float = 60.0) -> None:
        with self._lock:
            if self._closed:
                return
            self._closed = True
        for rank, c in enumerate(self._conns):
            with self._send_locks[rank]:
                try:
                    c.send(_STOP)
                except (BrokenPipeError, OSError):
                    pass
        for t in self._readers:
            t.join(timeout_s)
        for p in self._procs:
            p.join(timeout_s)
        self._kill()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
