"""Process-per-GPU dispatcher (§8(e), paper_2509_22681_b200.dispatch) on CPU:
two worker processes with a scoring stub in place of the per-GPU DeviceService
check the routing (least outstanding work, every worker used), the result
order under concurrency, error propagation, and shutdown."""

import threading
import time

import numpy as np
import pytest

from paper_2509_22681_b200.dispatch import MultiDeviceService


class StubScorer:
    """Scores = f(candidate ids, rank); sleeps in proportion to the work."""

    def __init__(self, rank):
        self.rank = rank

    def handle_batch(self, reqs):
        from paper_2509_22681_b200.service import RequestError, ScoreResponse

        out = []
        for r in reqs:
            if len(r.candidate_item_ids) == 0:
                raise RequestError("candidates must be non-empty")
            time.sleep(1e-5 * (len(r.history_item_ids) + len(r.candidate_item_ids)))
            s = np.stack([np.asarray(r.candidate_item_ids, dtype=np.float64) * 2.0 + len(r.history_item_ids),
                          np.full(len(r.candidate_item_ids), float(self.rank))], axis=1)
            out.append(ScoreResponse(s, 0.0, 0.01))
        return out

    def close(self):
        pass


class StubFactory:
    def __call__(self, rank):
        return StubScorer(rank)


@pytest.fixture(scope="module")
def svc():
    s = MultiDeviceService(n_devices=2, scorer_factory=StubFactory(), start_timeout_s=120)
    yield s
    s.close()


def test_stream_results_in_order_and_both_workers_used(svc):
    rng = np.random.default_rng(0)
    reqs = [(rng.integers(0, 1000, 2 * int(rng.integers(0, 300))), rng.integers(0, 1000, int(rng.integers(1, 200))))
            for _ in range(60)]
    out = svc.score(reqs)
    for (h, c), s in zip(reqs, out):
        np.testing.assert_array_equal(s[:, 0], c * 2.0 + len(h))
    ranks = {int(s[0, 1]) for s in out}
    assert ranks == {0, 1}
    assert min(svc.routed) > 0 and sum(svc.routed) >= 60
    assert svc.outstanding() == [0, 0]


def test_concurrent_callers(svc):
    results = {}

    def caller(k):
        h = np.arange(10 * k, dtype=np.int64)
        c = np.arange(k + 1, dtype=np.int64) + 100 * k
        results[k] = (h, c, svc.submit(h, c).result(timeout=60))

    threads = [threading.Thread(target=caller, args=(k,)) for k in range(16)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for k, (h, c, (scores, compute_ms, e2e_s)) in results.items():
        np.testing.assert_array_equal(scores[:, 0], c * 2.0 + len(h))
        assert e2e_s > 0


def test_least_outstanding_work_routing(svc):
    # one long request occupies a worker; the short ones that follow go to the other
    big = svc.submit(np.zeros(20000, dtype=np.int64), np.zeros(5000, dtype=np.int64))
    smalls = [svc.submit(np.zeros(2, dtype=np.int64), np.arange(3)) for _ in range(5)]
    big_rank = int(big.result(timeout=60)[0][0, 1])
    assert all(int(f.result(timeout=60)[0][0, 1]) != big_rank for f in smalls)


def test_errors_reach_the_caller(svc):
    from paper_2509_22681_b200.service import RequestError

    with pytest.raises(RequestError):
        svc.submit(np.zeros(4, dtype=np.int64), np.zeros(0, dtype=np.int64)).result(timeout=60)
    ok = svc.submit(np.zeros(4, dtype=np.int64), np.arange(2)).result(timeout=60)[0]
    assert ok.shape == (2, 2)


def test_closed_dispatcher_refuses():
    s = MultiDeviceService(n_devices=1, scorer_factory=StubFactory(), start_timeout_s=120)
    s.close()
    with pytest.raises(RuntimeError):
        s.submit(np.zeros(2, dtype=np.int64), np.arange(2))


def test_http_over_the_dispatcher(svc):
    # api.create_app serves the dispatcher like a DeviceService (N GPUs behind one HTTP front end)
    from fastapi.testclient import TestClient

    from paper_2509_22681_b200.api import create_app

    app = create_app(svc)
    client = TestClient(app)  # no context manager: the fixture owns the dispatcher's lifetime
    r = client.post("/score", json={"user_id": 1, "history": [1, 2, 3, 4], "candidates": [10, 11]})
    assert r.status_code == 200
    assert [row[0] for row in r.json()["scores"]] == [24.0, 26.0]
    assert client.post("/score", json={"user_id": 1, "history": [1], "candidates": []}).status_code == 400
    m = client.get("/metrics").json()
    assert m["requests_total"] >= 1 and m["workers"] == 2


def test_dead_worker_is_routed_around():
    # a worker that dies fails the requests it held and takes no new ones; the
    # stream continues on the survivors
    s = MultiDeviceService(n_devices=2, scorer_factory=StubFactory(), start_timeout_s=120)
    try:
        s._procs[0].kill()
        deadline = time.time() + 60
        while s.alive()[0] and time.time() < deadline:
            time.sleep(0.05)
        assert s.alive() == [False, True]
        out = s.score([(np.arange(4), np.arange(3)) for _ in range(6)])
        assert all(int(o[0, 1]) == 1 for o in out)
        s._procs[1].kill()
        while s.alive()[1] and time.time() < deadline:
            time.sleep(0.05)
        from paper_2509_22681_b200.dispatch import DispatchError

        with pytest.raises(DispatchError):
            s.submit(np.zeros(2, dtype=np.int64), np.arange(2))
    finally:
        s.close(timeout_s=5)
