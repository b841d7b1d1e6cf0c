"""The CPU oracle (oracle/flame_oracle.py) against golden vectors produced by
the reference implementation itself (oracle/gen_golden.py)."""

import numpy as np
import pytest

from conftest import FORWARD_CASES, golden_forward, load_golden
from oracle import flame_oracle as orc


@pytest.mark.parametrize("name", FORWARD_CASES)
def test_oracle_forward_matches_reference(name):
    cfg, params, hist, cand, blob = golden_forward(name)
    out = orc.model_forward(hist, cand, params, cfg)
    assert out.shape == blob["scores"].shape
    assert np.abs(out - blob["scores"]).max() <= 1e-12


@pytest.mark.parametrize("name", ["cfg1", "ref_instance", "l2_wide", "l3_nb4"])
def test_reference_parallel_equals_sequential_fixture(name):
    _, _, _, _, blob = golden_forward(name)
    assert np.abs(blob["scores"] - blob["sequential"]).max() <= 1e-10


def test_oracle_item_embedding_matches_reference_store():
    g = load_golden("pda.npz")
    for k, row in zip(g["emb_ids"], g["emb_values"]):
        np.testing.assert_array_equal(orc.item_embedding(1234, int(k), 0, 64), row)


@pytest.mark.parametrize("key", ["hist", "cand", "single", "dups"])
def test_oracle_resolve_matches_reference_service(key):
    g = load_golden("pda.npz")
    ids = g[f"{key}_ids"]
    table = np.stack([orc.item_embedding(1234, i, 0, 16) for i in range(int(ids.max()) + 1)])
    rows, uq, inv = orc.resolve_embeddings(ids, table)
    np.testing.assert_array_equal(uq, g[f"{key}_unique"])
    np.testing.assert_array_equal(inv, g[f"{key}_inverse"])
    np.testing.assert_array_equal(rows, g[f"{key}_rows"])


def test_oracle_unknown_ids_decode_to_zero():
    table = np.ones((4, 3))
    rows, uq, inv = orc.resolve_embeddings(np.array([5, 1, -2, 1]), table)
    np.testing.assert_array_equal(rows, [[0, 0, 0], [1, 1, 1], [0, 0, 0], [1, 1, 1]])
    np.testing.assert_array_equal(uq, [-2, 1, 5])
    np.testing.assert_array_equal(inv, [2, 1, 0, 1])


def test_algorithmic_flops_survey_values():
    import paper_2509_22681_b200 as fb

    cfg3 = fb.ModelConfig(512, 64, 8, 1, 2048, 2, 2048, 512)
    assert abs(orc.algorithmic_flops(cfg3, 2048, 512) / 3.115e10 - 1) < 2e-3
    cfg2 = fb.ModelConfig(256, 64, 4, 1, 1024, 2, 1024, 256)
    assert abs(orc.algorithmic_flops(cfg2, 1024, 256) / 2.28e9 - 1) < 5e-3


def test_package_flop_formula_matches_oracle_formula():
    import paper_2509_22681_b200 as fb
    from paper_2509_22681_b200.flops import algorithmic_flops

    for dims, H, C in [((64, 16, 2, 2, 256, 2, 256, 64), 256, 64), ((512, 64, 8, 1, 2048, 2, 2048, 512), 2048, 512)]:
        cfg = fb.ModelConfig(*dims)
        assert algorithmic_flops(cfg, H, C) == orc.algorithmic_flops(cfg, H, C)


@pytest.mark.parametrize("name", ["cfg4_c16", "cfg4_c2048"])
def test_oracle_cfg4_candidate_range_ends(name):
    # round-2 fixtures (oracle/gen_golden_r2.py): both ends of the DSO candidate range
    cfg, params, hist, cand, blob = golden_forward(name)
    assert np.abs(orc.model_forward(hist, cand, params, cfg) - blob["scores"]).max() <= 1e-12


def test_oracle_bench_id_path_first_request():
    """The oracle's resolve + forward on the first request of bench.py's cfg3 batch
    (Zipf ids over 100k items) equals the reference Service + model_forward."""
    import paper_2509_22681_b200 as fb

    g = load_golden("ids_cfg3.npz")
    dims = [int(x) for x in g["dims"]]
    cfg = fb.ModelConfig(*dims[:8], seed=dims[8])
    h, c = g["hist_ids"][0], g["cand_ids"][0]
    ids = np.union1d(h, c)
    table = np.zeros((int(ids.max()) + 1, cfg.hidden_dim))
    for i in ids:
        table[i] = orc.item_embedding(int(g["store_seed"]), int(i), 0, cfg.hidden_dim)
    hist, _, _ = orc.resolve_embeddings(h, table)
    cand, _, _ = orc.resolve_embeddings(c, table)
    out = orc.model_forward(hist, cand, fb.init_params(cfg), cfg)
    assert np.abs(out - g["scores"][0]).max() <= 1e-12


def test_bench_generator_reproduces_fixture_ids():
    """bench.make_requests draws the same ids as the reference _KeySampler did for the fixture."""
    import bench

    g = load_golden("ids_cfg3.npz")
    reqs = bench.make_requests(8, 2048, 512, int(g["workload_seed"]))
    for (h, c), hh, cc in zip(reqs, g["hist_ids"], g["cand_ids"]):
        np.testing.assert_array_equal(h, hh)
        np.testing.assert_array_equal(c, cc)


CAP_CASES = ["dh128_l2", "dh96", "dh128_nohist", "tasks12", "d1536"]


@pytest.mark.parametrize("name", CAP_CASES)
def test_oracle_capability_cases(name):
    # oracle/gen_golden_caps.py: head_dim 96 / 128 and 12 tasks, from the reference
    cfg, params, hist, cand, blob = golden_forward(name)
    assert np.abs(orc.model_forward(hist, cand, params, cfg) - blob["scores"]).max() <= 1e-12
    assert np.abs(blob["scores"] - blob["sequential"]).max() <= 1e-10
