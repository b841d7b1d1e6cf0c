"""Parity cases round 1 never compared against the reference:

* the cfg4 model at both ends of the DSO candidate range (C = 2048: 16 attention
  tiles, the largest bucket; C = 16: the smallest), through ``model_forward`` and
  through ``BucketScheduler.score`` in one mixed batch;
* the bench's exact id path: the first 8 requests of bench.py's cfg3 batch
  (Zipf ids over the 100k-item fp32 HBM table) through
  ``BucketScheduler.score(ids=True)`` and ``DeviceExecutor.score_ids``, against
  the reference ``Service.resolve_embeddings`` + ``model_forward``;
* ``flame_create_flmp``'s success path: a reference-written FLMP image loaded by
  the C library scores bit-identically to the array-built context.

Fixtures: oracle/gen_golden_r2.py (runs the reference itself).
"""

import tempfile
from pathlib import Path

import numpy as np
import pytest

import paper_2509_22681_b200 as fb
from conftest import golden_forward, load_golden
from paper_2509_22681_b200.orchestrator import BucketScheduler
from paper_2509_22681_b200.pda import build_item_table

pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-4, "bf16": 2e-2}


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
@pytest.mark.parametrize("name", ["cfg4_c2048", "cfg4_c16"])
def test_cfg4_candidate_range_ends(gpu, name, prec):
    cfg, params, hist, cand, blob = golden_forward(name)
    out = fb.model_forward(hist, cand, params, cfg, precision=prec)
    err = np.abs(out - blob["scores"]).max()
    assert err <= TOL[prec], f"{name}/{prec}: max abs {err:.3e}"


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_cfg4_range_through_bucket_scheduler(gpu, prec):
    cfg, params, h1, c1, b1 = golden_forward("cfg4_c2048")
    _, _, h2, c2, b2 = golden_forward("cfg4_c16")
    eng = fb.get_engine(params, cfg, prec)
    sched = BucketScheduler(eng, target_rows=4096)
    got = sched.score([(h1, c1), (h2, c2), (h1, c1[:700])])
    assert np.abs(got[0] - b1["scores"]).max() <= TOL[prec]
    assert np.abs(got[1] - b2["scores"]).max() <= TOL[prec]
    # the 700-candidate prefix is the first 700 rows of the full request (candidate isolation)
    np.testing.assert_array_equal(got[2], fb.model_forward(h1, c1[:700], params, cfg, precision=prec))
    assert np.abs(got[2] - b1["scores"][:700]).max() <= TOL[prec]


@pytest.fixture(scope="module")
def cfg3_ids():
    blob = load_golden("ids_cfg3.npz")
    dims = [int(x) for x in blob["dims"]]
    cfg = fb.ModelConfig(*dims[:8], seed=dims[8])
    table = build_item_table(int(blob["num_items"]), cfg.hidden_dim, int(blob["store_seed"]))
    return cfg, fb.init_params(cfg), table, blob


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_bench_id_path_cfg3_matches_reference(gpu, cfg3_ids, prec):
    cfg, params, table, blob = cfg3_ids
    eng = fb.FlameEngine(params, cfg, prec)
    try:
        eng.set_table(table, dtype="fp32")  # bench.py's table: 100k items, fp32 rows
        reqs = list(zip(blob["hist_ids"], blob["cand_ids"]))
        want = blob["scores"]
        sched = BucketScheduler(eng, target_rows=16384, with_ids=True)
        got = sched.score(reqs, ids=True)
        errs = [float(np.abs(g - w).max()) for g, w in zip(got, want)]
        assert max(errs) <= TOL[prec], errs
        ex = eng.executor(len(reqs), 256, 512, with_ids=True)
        direct = ex.score_ids(reqs)
        for g, d in zip(got, direct):
            np.testing.assert_array_equal(g, d)
    finally:
        eng.close()


def test_flmp_loaded_by_the_c_library(gpu):
    blob = load_golden("params.npz")
    image = blob["flmp_tiny"].tobytes()
    cfg = fb.params.config_from_header(image)
    rng = np.random.default_rng(5)
    hist = rng.uniform(-1, 1, (32, cfg.hidden_dim))
    cand = rng.uniform(-1, 1, (7, cfg.hidden_dim))
    for prec in ("fp32", "bf16"):
        from_file = fb.FlameEngine.from_flmp(image, precision=prec)
        with tempfile.TemporaryDirectory() as tmp:
            p = Path(tmp) / "m.flmp"
            p.write_bytes(image)
            _, params = fb.load_params(p)
        from_arrays = fb.FlameEngine(params, cfg, precision=prec)
        try:
            assert from_file.config == cfg
            a = from_file.executor(1, 16, 8).score([(hist, cand)])[0]
            b = from_arrays.executor(1, 16, 8).score([(hist, cand)])[0]
            np.testing.assert_array_equal(a, b)
            assert a.shape == (7, cfg.num_tasks)
        finally:
            from_file.close()
            from_arrays.close()
