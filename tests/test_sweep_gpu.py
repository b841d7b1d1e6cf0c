"""Seeded sweep of odd model shapes against the CPU oracle (device path through the
C ABI, both precisions).

The golden fixtures pin the reference's own configurations; this sweep covers the
shapes in between that the kernels tile around: hidden sizes that are not multiples
of 64 (row padding of every GEMM operand), head sizes from 8 to 128, ffn / task
counts that leave partial epilogue chunks, 1 to 5 blocks, 1 to 3 layers, and batches
whose requests have ragged history (including none) and candidate counts (including
one, and counts just past a 128-row tile).  Reference semantics:
model/forward.py:186-204 (model_forward), :75-140 (block_forward),
model/attention.py:118-178 (SUMI attention).

Tolerances (north star): fp32 verification mode <= 1e-4, bf16 <= 2e-2 max-abs on
the sigmoid scores.
"""

import numpy as np
import pytest

import paper_2509_22681_b200 as fb

pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-4, "bf16": 2e-2}

# (d, dh, N_b, L, f, tasks, hb_max, C_max): hb_max is the per-block history cap
SHAPES = [
    (48, 8, 3, 1, 100, 1, 40, 129),
    (80, 16, 5, 2, 72, 5, 24, 33),
    (96, 32, 1, 1, 200, 3, 300, 257),
    (136, 8, 2, 3, 64, 2, 17, 20),
    (200, 40, 4, 1, 520, 9, 64, 130),
    (192, 96, 2, 2, 384, 2, 129, 64),
    (256, 128, 3, 1, 260, 4, 100, 200),
    (320, 64, 2, 1, 1280, 7, 256, 384),
    (64, 64, 1, 2, 64, 1, 257, 1),
    (24, 24, 2, 1, 48, 6, 9, 300),
]


def _case(i):
    d, dh, nb, L, f, tasks, hb_max, c_max = SHAPES[i]
    cfg = fb.ModelConfig(d, dh, nb, L, f, tasks, nb * hb_max, c_max, seed=100 + i)
    rng = np.random.default_rng(7000 + i)
    reqs = []
    hbs = [hb_max, 0, int(rng.integers(1, hb_max + 1))]
    cs = [c_max, int(rng.integers(1, c_max + 1)), 1]
    for hb, c in zip(hbs, cs):
        reqs.append((rng.uniform(-1, 1, (nb * hb, d)), rng.uniform(-1, 1, (c, d))))
    return cfg, reqs


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
@pytest.mark.parametrize("i", range(len(SHAPES)))
def test_shape_sweep_matches_oracle(gpu, i, prec):
    from oracle import flame_oracle as orc

    cfg, reqs = _case(i)
    params = fb.init_params(cfg)
    outs = fb.model_forward_batch(reqs, params, cfg, precision=prec)
    assert len(outs) == len(reqs)
    for k, ((h, c), o) in enumerate(zip(reqs, outs)):
        ref = orc.model_forward(h, c, params, cfg)
        assert o.shape == ref.shape == (c.shape[0], cfg.num_tasks)
        err = float(np.abs(o - ref).max())
        assert err <= TOL[prec], f"shape {SHAPES[i]} request {k} ({h.shape[0]} hist, {c.shape[0]} cand) {prec}: {err:.3e}"
        # a request scored alone gives the same rows, bit for bit, as inside the batch
        solo = fb.model_forward(h, c, params, cfg, precision=prec)
        np.testing.assert_array_equal(solo, o)
