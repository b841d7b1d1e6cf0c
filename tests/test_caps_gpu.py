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
@pytest.mark.parametrize("name", ["dh128_l2", "dh96", "dh128_nohist", "tasks12"])
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
