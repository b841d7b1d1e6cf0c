"""PDA device kernels: dedup maps bit-exact with np.unique (the contract of
Service.resolve_embeddings, reference service.py:97-108) and assembled rows
equal to the reference store's embeddings."""

import numpy as np
import pytest

import paper_2509_22681_b200 as fb
from conftest import load_golden
from paper_2509_22681_b200.pda import DeviceFeatureAssembler, build_item_table

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def assembler(gpu):
    cfg = fb.ModelConfig(16, 4, 2, 1, 32, 2, 512, 512, seed=3)
    eng = fb.FlameEngine(fb.init_params(cfg), cfg, precision="fp32")
    eng.set_table(build_item_table(500, 16, store_seed=1234), dtype="fp32")
    return DeviceFeatureAssembler(eng, max_ids=8192)


@pytest.mark.parametrize("key", ["hist", "cand", "single", "dups"])
def test_resolve_matches_reference_service(assembler, key):
    g = load_golden("pda.npz")
    rows, uq, inv = assembler.resolve(g[f"{key}_ids"])
    np.testing.assert_array_equal(uq, g[f"{key}_unique"])
    np.testing.assert_array_equal(inv, g[f"{key}_inverse"])
    np.testing.assert_array_equal(rows, g[f"{key}_rows"].astype(np.float32))


@pytest.mark.parametrize("n,seed", [(1, 0), (2, 1), (37, 2), (1000, 3), (2048, 4), (4097, 5), (8184, 6), (8192, 7)])
def test_dedup_bit_exact_random(assembler, n, seed):
    rng = np.random.default_rng(seed)
    ids = rng.integers(-50, 700, n)  # includes unknown ids (< 0, >= 500)
    ids[rng.integers(0, n, max(1, n // 4))] = np.iinfo(np.int64).max
    rows, uq, inv = assembler.resolve(ids)
    want_u, want_i = np.unique(ids, return_inverse=True)
    np.testing.assert_array_equal(uq, want_u)
    np.testing.assert_array_equal(inv, want_i)
    np.testing.assert_array_equal(uq[inv], ids)  # round trip
    table = build_item_table(500, 16, store_seed=1234)
    known = (ids >= 0) & (ids < 500)
    np.testing.assert_array_equal(rows[known], table[ids[known]])
    assert not rows[~known].any()


def test_all_equal_and_sorted_inputs(assembler):
    for ids in (np.full(3000, 9), np.arange(5000), np.arange(5000)[::-1].copy()):
        rows, uq, inv = assembler.resolve(ids)
        want_u, want_i = np.unique(ids, return_inverse=True)
        np.testing.assert_array_equal(uq, want_u)
        np.testing.assert_array_equal(inv, want_i)


def test_id_path_scores_match_embedding_path(gpu):
    """Service path (ids -> PDA -> forward) == model_forward on the same rows."""
    cfg = fb.ModelConfig(64, 16, 2, 1, 256, 2, 256, 128, seed=8)
    params = fb.init_params(cfg)
    table = build_item_table(300, 64)
    eng = fb.get_engine(params, cfg, "bf16")
    eng.set_table(table, dtype="fp32")
    rng = np.random.default_rng(3)
    reqs = [(rng.integers(0, 300, h), rng.integers(0, 320, c)) for h, c in [(256, 100), (128, 7), (0, 3)]]
    ex = eng.executor(len(reqs), 128, 128, with_ids=True)
    got = ex.score_ids(reqs)
    for (hid, cid), s in zip(reqs, got):
        hist = np.where((hid < 300)[:, None], table[np.clip(hid, 0, 299)], 0.0)
        cand = np.where((cid < 300)[:, None], table[np.clip(cid, 0, 299)], 0.0)
        want = fb.model_forward(hist, cand, params, cfg)
        np.testing.assert_array_equal(s, want)
