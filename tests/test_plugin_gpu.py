"""Drop-in at the plug-in point (§8(b)): the UNMODIFIED
reference ``flameserve.service.Service`` with its runner swapped for the B200
``ExecutorPool`` / ``ImplicitShapeRunner``, fed the reference's own
``ModelParams`` / ``ModelConfig`` objects, answers ``handle_request`` with the
scores of the reference's own runner (numpy ``model_forward``).

The reference is imported from ``baseline/_ref`` — the offline pip install of
/root/reference made by the build container (``python -m pip install
--no-index --no-build-isolation --no-deps --target baseline/_ref <copy of
/root/reference/pkg>``).  It is git-ignored but travels with the
repo snapshot to the GPU box; without it these tests skip.
"""

import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REF_PKG = Path(__file__).resolve().parent.parent / "baseline" / "_ref"


@pytest.fixture(scope="module")
def ref():
    if not (REF_PKG / "flameserve").is_dir():
        pytest.skip("reference not installed under baseline/_ref")
    if str(REF_PKG) not in sys.path:
        sys.path.insert(0, str(REF_PKG))
    import flameserve.config as rconfig
    import flameserve.orchestrator as rorch
    import flameserve.service as rservice

    return rconfig, rorch, rservice


def _request(rservice, cfg, seed, h, c):
    rng = np.random.default_rng(seed)
    return rservice.ScoreRequest(user_id=seed, history_item_ids=rng.integers(0, 50_000, h),
                                 candidate_item_ids=rng.integers(0, 50_000, c), context={"page": "home"})


@pytest.mark.parametrize("routing", ["explicit", "implicit"])
@pytest.mark.parametrize("prec,tol", [("fp32", 1e-4), ("bf16", 2e-2)])
def test_reference_service_with_b200_runner(gpu, ref, routing, prec, tol):
    from paper_2509_22681_b200 import orchestrator as orch

    rconfig, rorch, rservice = ref
    from flameserve.cache import CacheConfig, CacheMode
    from flameserve.store import RemoteStoreConfig

    # sync cache and no simulated latency: both services resolve identical rows
    cfg = rconfig.ServiceConfig(
        cache=CacheConfig(mode=CacheMode.SYNC), remote_store=RemoteStoreConfig(0.0, 0.0),
        orchestrator=rconfig.OrchestratorConfig(profile_shapes=(64, 256), executors_per_shape=2, routing=routing))
    baseline = rservice.Service(cfg)  # stock runner: numpy model_forward
    plugged = rservice.Service(cfg)
    assert type(plugged.params).__module__.startswith("flameserve.")  # the reference's own params object
    plugged.runner.shutdown()
    if routing == "explicit":
        profiles = orch.ProfileSet(cfg.orchestrator.profile_shapes, cfg.orchestrator.executors_per_shape)
        plugged.runner = orch.ExecutorPool(profiles, plugged.params, cfg.model, attn_impl=cfg.attention_impl,
                                           precision=prec)
    else:
        plugged.runner = orch.ImplicitShapeRunner(plugged.params, cfg.model, attn_impl=cfg.attention_impl,
                                                  precision=prec)
    try:
        for seed, h, c in ((1, 512, 300), (2, 0, 7), (3, 1024, 64), (4, 98, 1)):
            req = _request(rservice, cfg, seed, h, c)
            want = baseline.handle_request(req).scores
            got = plugged.handle_request(req)
            assert got.scores.shape == want.shape == (c, cfg.model.num_tasks)
            err = float(np.abs(got.scores - want).max())
            assert err <= tol, f"{routing}/{prec} request {seed}: max abs {err:.3e}"
            assert got.compute_latency_ms > 0
        with pytest.raises(rservice.RequestError):
            plugged.handle_request(_request(rservice, cfg, 5, 3, 4))  # not a multiple of num_blocks
        snap = plugged.metrics_snapshot()
        assert snap["requests_total"] == 4
        if routing == "explicit":
            assert snap["steady_state_allocs"] == 0
    finally:
        plugged.close()
        baseline.close()


def test_reference_loaded_params_drive_the_engine(gpu, ref, tmp_path):
    # a reference-written FLMP file (reference save_params) loaded by the
    # reference load_params: the B200 model_forward accepts those objects as is
    import flameserve.model as rmodel

    import paper_2509_22681_b200 as fb

    cfg = rmodel.ModelConfig(32, 8, 2, 2, 64, 3, 128, 64, seed=11)
    rmodel.save_params(rmodel.init_params(cfg), cfg, tmp_path / "m.flmp")
    rcfg, rparams = rmodel.load_params(tmp_path / "m.flmp")
    rng = np.random.default_rng(0)
    hist, cand = rng.uniform(-1, 1, (96, 32)), rng.uniform(-1, 1, (20, 32))
    want = rmodel.model_forward(hist, cand, rparams, rcfg)
    got = fb.model_forward(hist, cand, rparams, rcfg, precision="fp32")
    assert float(np.abs(got - want).max()) <= 1e-4
    eng = fb.FlameEngine.from_flmp((tmp_path / "m.flmp").read_bytes(), precision="fp32")
    try:
        ex = eng.executor(1, 64, 32)
        assert float(np.abs(ex.score([(hist, cand)])[0] - want).max()) <= 1e-4
    finally:
        eng.close()
