"""Host logic of DeviceService without a GPU: the leader / follower coalescing
of concurrent callers (every ticket gets its own result, batches merge, at most
max_inflight batches are outstanding, errors reach their callers) and request
validation, with the device submit / complete replaced by stubs."""

import threading
import time

import numpy as np
import pytest

from paper_2509_22681_b200.config import ModelConfig
from paper_2509_22681_b200.service import DeviceService, RequestError, ScoreRequest, _Ticket

CFG = ModelConfig(32, 8, 2, 1, 64, 2, 64, 32, seed=5)


def stub_service(max_batch=8, max_inflight=2, fail_on=None, delay=0.002):
    svc = object.__new__(DeviceService)
    svc.config = CFG
    svc._queue, svc._leader, svc._in_flight, svc.max_inflight = [], False, 0, max_inflight
    svc._cv = threading.Condition(threading.Lock())
    svc.max_batch = max_batch
    svc.batches, svc.peak = [], 0

    def submit(batch):
        if fail_on is not None and any(int(t.cand[0]) == fail_on for t in batch):
            raise RuntimeError("device error")
        with svc._cv:
            svc.peak = max(svc.peak, svc._in_flight)
        svc.batches.append(len(batch))
        return [float(t.cand.sum()) for t in batch]

    def complete(batch, handle):
        time.sleep(delay)
        for t, v in zip(batch, handle):
            t.scores, t.lat = v, delay

    svc._submit, svc._complete = submit, complete
    return svc


def run_threads(svc, n_threads, per_thread):
    results, errors = {}, []

    def worker(k):
        for j in range(per_thread):
            key = k * 1000 + j
            t = _Ticket(np.zeros(0, np.int64), np.array([key, 1], np.int64))
            try:
                svc._dispatch([t])
                if t.error is not None:
                    raise t.error
                results[key] = t.scores
            except Exception as exc:  # noqa: BLE001
                errors.append((key, exc))

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(n_threads)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=60)
    assert not any(t.is_alive() for t in threads), "dispatcher deadlocked"
    return results, errors


def test_every_ticket_gets_its_own_result_and_batches_merge():
    svc = stub_service()
    results, errors = run_threads(svc, 16, 20)
    assert not errors
    assert len(results) == 16 * 20
    assert all(v == k + 1 for k, v in results.items())
    assert len(svc.batches) < 16 * 20          # concurrent callers were coalesced
    assert max(svc.batches) <= svc.max_batch
    assert svc.peak <= svc.max_inflight        # never more than max_inflight outstanding
    assert svc._in_flight == 0 and not svc._leader and not svc._queue


def test_errors_reach_only_their_batch():
    svc = stub_service(max_batch=1, fail_on=3005)
    results, errors = run_threads(svc, 4, 10)
    assert [k for k, _ in errors] == [3005]
    assert isinstance(errors[0][1], RuntimeError)
    assert len(results) == 4 * 10 - 1


def test_one_caller_many_tickets():
    svc = stub_service(max_batch=4)
    tickets = [_Ticket(np.zeros(0, np.int64), np.array([k, 0], np.int64)) for k in range(10)]
    svc._dispatch(tickets)
    assert [t.scores for t in tickets] == [float(k) for k in range(10)]
    assert svc.batches == [4, 4, 2]


def test_validation_matches_reference_messages():
    svc = stub_service()
    req = lambda h, c: ScoreRequest(1, np.zeros(h, np.int64), np.zeros(c, np.int64))  # noqa: E731
    for bad, msg in [(req(8, 0), "non-empty"), (req(8, 33), "exceeds max"), (req(66, 3), "history length"),
                     (req(7, 3), "multiple of num_blocks")]:
        with pytest.raises(RequestError, match=msg):
            svc._validate(bad)
    svc._validate(req(8, 32))
