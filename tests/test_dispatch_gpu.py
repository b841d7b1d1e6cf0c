"""The process-per-GPU dispatcher over real DeviceService workers (one per
visible GPU, or two sharing GPU 0): a routed request stream scores exactly what one
in-process DeviceService scores for the same requests (the kernels are batch-
composition invariant, so the coalescing of each worker does not change a bit)."""

import numpy as np
import pytest
import torch

import paper_2509_22681_b200 as fb
from paper_2509_22681_b200.dispatch import MultiDeviceService
from paper_2509_22681_b200.service import DeviceService, RequestError, ScoreRequest, ServiceConfig

pytestmark = pytest.mark.gpu


def test_dispatched_stream_equals_single_service(gpu):
    model = fb.ModelConfig(32, 8, 2, 1, 64, 2, 256, 128, seed=5)
    cfg = ServiceConfig(model=model, num_items=500, target_rows=1024)
    rng = np.random.default_rng(4)
    reqs = [(rng.integers(0, 500, 2 * int(rng.integers(0, 129))), rng.integers(0, 500, int(rng.integers(1, 129))))
            for _ in range(80)]
    # two worker processes: one per GPU, or both on GPU 0 of a one-GPU box
    devices = [0, 1] if torch.cuda.device_count() >= 2 else [0, 0]
    with MultiDeviceService(cfg, n_devices=2, devices=devices) as svc:
        got = svc.score(reqs)
        with pytest.raises(RequestError):
            svc.submit(np.zeros(3, dtype=np.int64), np.arange(2)).result(timeout=120)
        assert sum(svc.routed) == 81 and min(svc.routed) > 0  # both workers scored
    ref = DeviceService.from_config(cfg)
    try:
        want = [r.scores for r in ref.handle_batch(
            [ScoreRequest(0, h, c) for h, c in reqs])]
    finally:
        ref.close()
    for g, w in zip(got, want):
        np.testing.assert_array_equal(g, w)
