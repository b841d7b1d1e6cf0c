"""HTTP wire contract of paper_2509_22681_b200.api (reference api.py:19-73 and
its tests): request/response models, 400 / 503 mapping, /metrics, /healthz.
The CPU test drives a stand-in service; the GPU test serves a DeviceService."""

import numpy as np
import pytest
from fastapi.testclient import TestClient

from paper_2509_22681_b200.api import create_app
from paper_2509_22681_b200.service import RequestError, ScoreResponse, ServiceClosedError


class FakeService:
    def __init__(self):
        self.closed = False
        self.calls = 0

    def handle_request(self, req):
        if self.closed:
            raise ServiceClosedError("service is shut down")
        if len(req.candidate_item_ids) == 0:
            raise RequestError("candidates must be non-empty")
        self.calls += 1
        c = len(req.candidate_item_ids)
        return ScoreResponse(np.full((c, 2), 0.5), 1.5, 1.0)

    def metrics_snapshot(self):
        return {"requests_total": self.calls}

    def close(self):
        self.closed = True


def test_wire_contract_cpu():
    svc = FakeService()
    with TestClient(create_app(svc)) as client:
        r = client.post("/score", json={"user_id": 1, "history": [1, 2], "candidates": [3, 4, 5]})
        assert r.status_code == 200
        body = r.json()
        assert body["scores"] == [[0.5, 0.5]] * 3 and body["overall_latency_ms"] == 1.5
        assert client.post("/score", json={"user_id": 1, "history": [], "candidates": []}).status_code == 400
        assert client.post("/score", json={"user_id": 1}).status_code == 422  # candidates required
        assert client.get("/metrics").json() == {"requests_total": 1}
        assert client.get("/healthz").json() == {"status": "ok"}
        svc.closed = True
        assert client.post("/score", json={"user_id": 1, "candidates": [1]}).status_code == 503
    assert svc.closed


@pytest.mark.gpu
def test_score_over_http_gpu(gpu):
    import paper_2509_22681_b200 as fb
    from paper_2509_22681_b200.service import DeviceService, ScoreRequest

    cfg = fb.ModelConfig(32, 8, 2, 1, 64, 2, 64, 32, seed=5)
    svc = DeviceService(cfg, num_items=300, target_rows=256)
    want = svc.handle_request(ScoreRequest(1, np.arange(16), np.arange(40, 52))).scores
    with TestClient(create_app(svc)) as client:
        r = client.post("/score", json={"user_id": 1, "history": list(range(16)), "candidates": list(range(40, 52))})
        assert r.status_code == 200
        np.testing.assert_array_equal(np.asarray(r.json()["scores"]), want)
        bad = client.post("/score", json={"user_id": 1, "history": list(range(15)), "candidates": [1]})
        assert bad.status_code == 400
        assert client.get("/metrics").json()["requests_total"] >= 2
