"""Device request path (paper_2509_22681_b200.service): the reference service
tests (tests/test_service.py) re-run against the HBM item table + PDA + DSO."""

import numpy as np
import pytest

import paper_2509_22681_b200 as fb
from oracle import flame_oracle as orc
from paper_2509_22681_b200.pda import item_embedding
from paper_2509_22681_b200.service import (DeviceService, RequestError, ScoreRequest, ServiceClosedError)

pytestmark = pytest.mark.gpu

CFG = fb.ModelConfig(32, 8, 2, 1, 64, 2, 64, 32, seed=5)
NUM_ITEMS = 400


def request_of(hist, cand):
    return ScoreRequest(user_id=1, history_item_ids=np.asarray(list(hist), dtype=np.int64),
                        candidate_item_ids=np.asarray(list(cand), dtype=np.int64))


def resolve(ids, versions=None):
    """Reference resolve_embeddings (service.py:97-108) over the store function
    (store.py:59-63 resolves every id, in the table or not)."""
    versions = versions or {}
    rows = [item_embedding(1234, int(i), versions.get(int(i), 0), CFG.hidden_dim) for i in ids]
    return np.asarray(rows).reshape(len(ids), CFG.hidden_dim)


@pytest.fixture(scope="module")
def service(gpu):
    s = DeviceService(CFG, num_items=NUM_ITEMS, target_rows=256)
    yield s
    if not s._closed:
        s.close()


def test_pipeline_matches_reference_forward(service):
    # reference tests/test_service.py:42-51 (pipeline == direct forward)
    req = request_of(range(16), range(200, 221))
    resp = service.handle_request(req)
    want = orc.model_forward(resolve(req.history_item_ids), resolve(req.candidate_item_ids),
                             service.params, CFG)
    assert resp.scores.shape == (21, 2)
    assert np.abs(resp.scores - want).max() <= 2e-2
    assert resp.overall_latency_ms >= resp.compute_latency_ms > 0


def test_identical_requests_identical_scores(service):
    req = request_of(range(12), range(50, 57))
    np.testing.assert_array_equal(service.handle_request(req).scores, service.handle_request(req).scores)


def test_batch_equals_single_and_ids_outside_the_table_resolve_like_the_store(service):
    # ids < 0 or >= num_items: host-resolved with the store function
    rng = np.random.default_rng(3)
    reqs = [request_of(rng.integers(-5, NUM_ITEMS + 50, 2 * int(rng.integers(0, 33))),
                       rng.integers(-5, NUM_ITEMS + 50, int(rng.integers(1, 33)))) for _ in range(12)]
    batch = service.handle_batch(reqs)
    for r, b in zip(reqs, batch):
        np.testing.assert_array_equal(b.scores, service.handle_request(r).scores)
        want = orc.model_forward(resolve(r.history_item_ids), resolve(r.candidate_item_ids), service.params, CFG)
        assert np.abs(b.scores - want).max() <= 2e-2


def test_mutate_refreshes_device_rows(service):
    req = request_of(range(8), range(100, 104))
    before = service.handle_request(req).scores
    service.mutate([101, 3, NUM_ITEMS + 7])
    after = service.handle_request(req).scores
    assert not np.array_equal(before, after)
    versions = {101: 1, 3: 1, NUM_ITEMS + 7: 1}
    req2 = request_of(range(8), [NUM_ITEMS + 7])
    want2 = orc.model_forward(resolve(req2.history_item_ids, versions), resolve(req2.candidate_item_ids, versions),
                              service.params, CFG)
    assert np.abs(service.handle_request(req2).scores - want2).max() <= 2e-2
    want = orc.model_forward(resolve(req.history_item_ids, versions), resolve(req.candidate_item_ids, versions),
                             service.params, CFG)
    assert np.abs(after - want).max() <= 2e-2


def test_validation_metrics_and_close(service):
    for bad in (request_of(range(8), []), request_of(range(7), range(3)), request_of(range(8), range(33)),
                request_of(range(66), range(3))):
        with pytest.raises(RequestError):
            service.handle_request(bad)
    n0 = service.pairs_processed
    service.handle_batch([request_of(range(8), range(5)), request_of(range(8), range(16))])
    assert service.pairs_processed == n0 + 21
    snap = service.metrics_snapshot()
    assert snap["requests_total"] >= 2 and snap["overall_ms"]["count"] == snap["requests_total"]
    service.close()
    with pytest.raises(ServiceClosedError):
        service.handle_request(request_of(range(8), range(3)))


def test_refresh_from_store_wire_values(gpu):
    """Raw store values (float64 LE + filler, store.py:66-78) decoded on the device;
    an empty value gives a zero row, as decode_embedding does."""
    svc = DeviceService(CFG, num_items=NUM_ITEMS, target_rows=256)
    d = CFG.hidden_dim
    new_emb = np.linspace(-1, 1, d)
    values = [new_emb.astype("<f8").tobytes() + b"\x00" * (512 - 8 * d), b""]
    svc.refresh_values([7, 9], values)
    req = request_of(range(8), [7, 9, 11])
    got = svc.handle_request(req).scores
    hist = resolve(req.history_item_ids)
    hist[7] = new_emb
    cand = np.stack([new_emb, np.zeros(d), resolve([11])[0]])
    want = orc.model_forward(hist, cand, svc.params, CFG)
    assert np.abs(got - want).max() <= 2e-2
    svc.close()


def test_concurrent_handle_request_threads(gpu):
    """Requests from several threads (the reference service is thread-safe,
    service.py:127-171) score exactly as when issued one by one."""
    import threading

    svc = DeviceService(CFG, num_items=NUM_ITEMS, target_rows=256)
    rng = np.random.default_rng(12)
    reqs = [request_of(rng.integers(0, NUM_ITEMS, 2 * int(rng.integers(0, 33))), rng.integers(0, NUM_ITEMS, int(c)))
            for c in rng.integers(1, 33, 16)]
    want = [svc.handle_request(r).scores for r in reqs]
    got = [None] * len(reqs)

    def worker(k):
        for i in range(k, len(reqs), 4):
            got[i] = svc.handle_request(reqs[i]).scores

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for g, w in zip(got, want):
        np.testing.assert_array_equal(g, w)
    svc.close()


def test_bf16_table_refresh(gpu):
    """A bf16 device table takes the same row / value refreshes (rounded to bf16)."""
    svc = DeviceService(CFG, num_items=NUM_ITEMS, target_rows=256, table_dtype="bf16")
    req = request_of(range(8), [5, 6])
    base = svc.handle_request(req).scores
    svc.mutate([5])
    svc.refresh_values([6], [b""])
    after = svc.handle_request(req).scores
    assert not np.array_equal(base, after)
    cand = np.stack([svc.embedding_of(5), np.zeros(CFG.hidden_dim)])
    want = orc.model_forward(resolve(req.history_item_ids), cand, svc.params, CFG)
    assert np.abs(after - want).max() <= 2e-2
    svc.close()


@pytest.mark.timeout(180)
def test_mutate_while_callers_are_scoring(gpu):
    # a row refresh waits for the DEVICE (not for the in-flight batches'
    # collection, which the submitting leader does only after its next submit):
    # concurrent mutate + scoring must neither deadlock nor fail
    import threading

    svc = DeviceService(CFG, num_items=NUM_ITEMS, target_rows=256)
    rng = np.random.default_rng(8)
    reqs = [request_of(rng.integers(0, NUM_ITEMS, 2 * int(rng.integers(0, 33))),
                       rng.integers(0, NUM_ITEMS, int(rng.integers(1, 33)))) for _ in range(96)]
    errors = []
    stop = threading.Event()

    def caller(k):
        try:
            for req in reqs[k::6]:
                assert np.isfinite(svc.handle_request(req).scores).all()
        except BaseException as exc:  # noqa: BLE001
            errors.append(exc)

    def mutator():
        i = 0
        while not stop.is_set():
            svc.mutate([i % NUM_ITEMS])
            i += 7

    try:
        m = threading.Thread(target=mutator)
        m.start()
        threads = [threading.Thread(target=caller, args=(k,)) for k in range(6)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        stop.set()
        m.join()
        assert not errors, errors[0]
    finally:
        stop.set()
        svc.close()
