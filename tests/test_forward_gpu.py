"""Device parity of the SUMI-ranker forward pass (through the C ABI) against
the reference's golden outputs, plus the reference's own property tests
(tests/test_forward.py) re-run on the device.

Tolerances (north star): fp32 verification mode <= 1e-4, bf16 mode <= 2e-2
max-abs on the sigmoid scores.  Batch-invariance properties are bit-exact.
"""

import numpy as np
import pytest

import paper_2509_22681_b200 as fb
from conftest import FORWARD_CASES, SMALL_CASES, golden_forward

pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-4, "bf16": 2e-2}


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
@pytest.mark.parametrize("name", FORWARD_CASES)
def test_forward_matches_reference_golden(gpu, name, prec):
    cfg, params, hist, cand, blob = golden_forward(name)
    out = fb.model_forward(hist, cand, params, cfg, precision=prec)
    assert out.shape == blob["scores"].shape
    err = np.abs(out - blob["scores"]).max()
    assert err <= TOL[prec], f"{name}/{prec}: max abs {err:.3e}"


@pytest.mark.parametrize("name", SMALL_CASES)
def test_parallel_equals_sequential_golden(gpu, name):
    # reference test_forward.py:224-232: the one-pass result equals the
    # per-candidate oracle; on the device, per-candidate calls are bit-exact
    # rows of the batched call
    cfg, params, hist, cand, blob = golden_forward(name)
    full = fb.model_forward(hist, cand, params, cfg, precision="fp32")
    assert np.abs(full - blob["sequential"]).max() <= 1e-4
    for i in range(min(cand.shape[0], 6)):
        solo = fb.model_forward(hist, cand[i:i + 1], params, cfg, precision="fp32")
        np.testing.assert_array_equal(solo[0], full[i])


def small_config(**kw):
    base = dict(hidden_dim=16, head_dim=4, num_blocks=2, layers_per_block=2, ffn_dim=24,
                num_tasks=3, max_history_len=64, max_candidates=32, seed=11)
    base.update(kw)
    return fb.ModelConfig(**base)


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_candidate_permutation_permutes_rows(gpu, prec):
    cfg = small_config()
    params = fb.init_params(cfg)
    rng = np.random.default_rng(12)
    hist = rng.normal(size=(16, 16))
    cand = rng.normal(size=(6, 16))
    perm = rng.permutation(6)
    base = fb.model_forward(hist, cand, params, cfg, precision=prec)
    shuffled = fb.model_forward(hist, cand[perm], params, cfg, precision=prec)
    np.testing.assert_array_equal(shuffled, base[perm])


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_duplicate_candidates_duplicate_rows(gpu, prec):
    cfg = small_config()
    params = fb.init_params(cfg)
    rng = np.random.default_rng(13)
    hist = rng.normal(size=(8, 16))
    one = rng.normal(size=(1, 16))
    scores = fb.model_forward(hist, np.concatenate([one, one, one]), params, cfg, precision=prec)
    np.testing.assert_array_equal(scores[0], scores[1])
    np.testing.assert_array_equal(scores[0], scores[2])


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_candidate_isolation_end_to_end(gpu, prec):
    cfg = small_config()
    params = fb.init_params(cfg)
    rng = np.random.default_rng(14)
    hist = rng.normal(size=(16, 16))
    cand = rng.normal(size=(5, 16))
    base = fb.model_forward(hist, cand, params, cfg, precision=prec)
    bumped = cand.copy()
    bumped[2] += 0.5
    moved = fb.model_forward(hist, bumped, params, cfg, precision=prec)
    keep = [0, 1, 3, 4]
    np.testing.assert_array_equal(moved[keep], base[keep])
    assert np.abs(moved[2] - base[2]).max() > 1e-6


def test_determinism_and_graph_replay(gpu):
    cfg = small_config()
    params = fb.init_params(cfg)
    rng = np.random.default_rng(15)
    hist = rng.normal(size=(8, 16))
    cand = rng.normal(size=(3, 16))
    a = fb.model_forward(hist, cand, params, cfg)
    b = fb.model_forward(hist, cand, params, cfg)
    np.testing.assert_array_equal(a, b)
    eng = fb.get_engine(params, cfg, "bf16")
    ex = eng.executor(1, *eng.bucket(8, 3))
    eager = ex.score([(hist, cand)], graph=False)[0]
    np.testing.assert_array_equal(eager, a)


def test_zero_weights_constant_scores(gpu):
    cfg = small_config()
    params = fb.init_params(cfg)
    for _, arr in fb.iter_param_arrays(params):
        arr[...] = 0.0
    for b in params.blocks:
        b.temperature = 1.0
    rng = np.random.default_rng(11)
    s = fb.model_forward(rng.normal(size=(8, 16)), rng.normal(size=(4, 16)), params, cfg,
                         precision="fp32")
    np.testing.assert_array_equal(s, np.full((4, 3), 0.5, dtype=s.dtype))


def test_forward_input_validation(gpu):
    cfg = small_config()
    params = fb.init_params(cfg)
    d = 16
    good_hist, good_cand = np.zeros((8, d)), np.zeros((2, d))
    for hist, cand in [(np.zeros((8, d + 1)), good_cand),
                       (np.zeros((cfg.max_history_len + 2, d)), good_cand),
                       (good_hist, np.zeros((0, d))),
                       (good_hist, np.zeros((cfg.max_candidates + 1, d))),
                       (np.zeros((7, d)), good_cand)]:
        with pytest.raises(ValueError):
            fb.model_forward(hist, cand, params, cfg)
    with pytest.raises(ValueError):
        fb.model_forward(good_hist, good_cand, params, cfg, attn_impl="flash")


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_batch_equals_per_request(gpu, prec):
    """Many requests with ragged H and C in ONE device pass == one at a time, bit for bit."""
    cfg = fb.ModelConfig(64, 16, 2, 1, 256, 2, 256, 300, seed=4)
    params = fb.init_params(cfg)
    rng = np.random.default_rng(21)
    reqs = []
    for h, c in [(256, 64), (128, 300), (0, 5), (2, 129), (256, 1), (64, 200)]:
        reqs.append((rng.uniform(-1, 1, (h, 64)), rng.uniform(-1, 1, (c, 64))))
    batch = fb.model_forward_batch(reqs, params, cfg, precision=prec)
    for (h, c), got in zip(reqs, batch):
        solo = fb.model_forward(h, c, params, cfg, precision=prec)
        np.testing.assert_array_equal(got, solo)


def test_bf16_and_fp32_paths_agree_at_cfg2(gpu):
    cfg, params, hist, cand, blob = golden_forward("cfg2")
    a = fb.model_forward(hist, cand, params, cfg, precision="bf16")
    b = fb.model_forward(hist, cand, params, cfg, precision="fp32")
    assert np.abs(a - b).max() <= 2e-2


def test_full_size_batch_invariance_cfg3_ids(gpu):
    """BASELINE cfg3 shape (8 blocks, d=512, H=2048, C=512) through the id path:
    an 8-request batch equals the same requests split 3 + 5 (partially filled
    executors: the device-side active count skips the unused slots) and one at a
    time, bit for bit; a duplicated request scores identically."""
    from paper_2509_22681_b200.pda import build_item_table

    cfg = fb.ModelConfig(512, 64, 8, 1, 2048, 2, 2048, 512, seed=0)
    eng = fb.FlameEngine(fb.init_params(cfg), cfg, "bf16")
    eng.set_table(build_item_table(3000, 512), dtype="fp32")
    rng = np.random.default_rng(2509)
    reqs = [(rng.integers(0, 3000, 2048), rng.integers(0, 3000, int(c))) for c in (512, 17, 512, 300, 511, 64, 512, 1)]
    reqs[6] = reqs[0]
    ex8 = eng.executor(8, 256, 512, with_ids=True)
    full = ex8.score_ids(reqs)
    split = ex8.score_ids(reqs[:3]) + ex8.score_ids(reqs[3:])
    one = [ex8.score_ids([r])[0] for r in reqs[:2]]
    for a, b in zip(full, split):
        np.testing.assert_array_equal(a, b)
    for a, b in zip(full[:2], one):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(full[0], full[6])
    assert all(np.isfinite(s).all() and s.shape == (len(c), 2) for (_, c), s in zip(reqs, full))


def test_batch_with_empty_and_full_histories_matches_oracle(gpu):
    # many units per CTA (R * G * heads > 148) and several tile pairs per unit, with
    # requests without history (out = v_self, no S / P phase) mixed in: the fused
    # kernel's epilogue must not release the projection accumulator early
    from oracle import flame_oracle as orc

    cfg = fb.ModelConfig(128, 64, 2, 1, 256, 2, 256, 512, seed=4)
    params = fb.init_params(cfg)
    rng = np.random.default_rng(12)
    reqs = [(rng.uniform(-1, 1, ((0 if i % 3 else 256), 128)), rng.uniform(-1, 1, (300 + i, 128))) for i in range(64)]
    outs = fb.model_forward_batch(reqs, params, cfg)
    for (h, c), o in zip(reqs[:12], outs[:12]):
        assert np.abs(o - orc.model_forward(h, c, params, cfg)).max() <= 2e-2
    for (h, c), o in zip(reqs, outs):  # batch composition invariance, bit for bit
        np.testing.assert_array_equal(o, fb.model_forward(h, c, params, cfg))
