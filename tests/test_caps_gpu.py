"""Model shapes beyond the round-1 kernel limits, on the device, against the
reference's outputs (oracle/gen_golden_caps.py): head_dim 96 and 128 (128-lane
head slots, the SIMT attention kernel in both precisions; L = 2 covers the
causal history attention), an empty history at head_dim 128, and 12 task
heads (the expert output kernel in groups of 8 tasks)."""

import numpy as np
import pytest

import paper_2509_22681_b200 as fb
from conftest import golden_forward

pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-4, "bf16": 2e-2}


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
@pytest.mark.parametrize("name", ["dh128_l2", "dh96", "dh128_nohist", "tasks12", "d1536"])
def test_capability_forward_matches_reference(gpu, name, prec):
    cfg, params, hist, cand, blob = golden_forward(name)
    out = fb.model_forward(hist, cand, params, cfg, precision=prec)
    assert out.shape == blob["scores"].shape
    err = float(np.abs(out - blob["scores"]).max())
    assert err <= TOL[prec], f"{name}/{prec}: max abs {err:.3e}"


@pytest.mark.parametrize("name", ["dh128_l2", "tasks12"])
def test_capability_single_candidate_rows_bit_exact(gpu, name):
    cfg, params, hist, cand, blob = golden_forward(name)
    full = fb.model_forward(hist, cand, params, cfg, precision="fp32")
    assert np.abs(full - blob["sequential"]).max() <= 1e-4
    for i in range(3):
        np.testing.assert_array_equal(fb.model_forward(hist, cand[i:i + 1], params, cfg, precision="fp32")[0],
                                      full[i])


@pytest.mark.parametrize("nb,H", [(1, 20000), (4, 17000 - 17000 % 4)])
def test_long_id_lists_are_deduplicated_in_segments(gpu, nb, H):
    # history id lists longer than one dedup CTA's 8192 ids are split into
    # segments (a duplicate across segments is only gathered twice): the scores
    # equal the oracle's on the rows the reference store resolves
    from oracle import flame_oracle as orc
    from paper_2509_22681_b200.pda import build_item_table

    cfg = fb.ModelConfig(64, 16, nb, 1, 128, 2, H, 64, seed=9)
    params = fb.init_params(cfg)
    table = build_item_table(3000, 64)
    eng = fb.FlameEngine(params, cfg, precision="fp32")
    try:
        eng.set_table(table, dtype="fp32")
        rng = np.random.default_rng(5)
        hist = (rng.zipf(1.3, H) % 3000).astype(np.int64)  # many repeats, across segments too
        cand = rng.integers(0, 3000, 37)
        ex = eng.executor(1, H // nb, 64, with_ids=True)
        got = ex.score_ids([(hist, cand)])[0]
        want = orc.model_forward(table[hist].astype(np.float64), table[cand].astype(np.float64), params, cfg)
        assert np.abs(got - want).max() <= 1e-4
    finally:
        eng.close()
