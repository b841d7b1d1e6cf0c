"""Load generator / report layer (paper_2509_22681_b200.loadgen) on the CPU:
the reference's tests/test_bench.py generator and report cases, pinned to the
reference's own stream digests and CSV bytes (tests/golden/workload.json, made
by oracle/gen_golden_workload.py)."""

import hashlib
import json
import itertools
from pathlib import Path

import numpy as np
import pytest

from paper_2509_22681_b200.config import ModelConfig
from paper_2509_22681_b200.loadgen import (CSV_HEADER, AblationConfig, EmptyRunError, KeyDistribution, RunReport,
                                           Scenario, WorkloadSpec, emit_report, generate_workload, load_report,
                                           run_scenario)
from paper_2509_22681_b200.service import ServiceConfig

GOLDEN = json.loads((Path(__file__).parent / "golden" / "workload.json").read_text())


def spec_of(scenario, n, seed=3, dist=KeyDistribution("zipf", 1.0), num_items=5000):
    return WorkloadSpec(scenario=scenario, duration_s=60.0, concurrency=4, key_distribution=dist, seed=seed,
                        num_requests=n, num_items=num_items)


@pytest.mark.parametrize("case", GOLDEN["streams"], ids=lambda c: f"{c['scenario']}-{c['kind']}-{c['seed']}")
def test_stream_matches_reference_digest(case):
    spec = spec_of(Scenario(case["scenario"]), case["n"], case["seed"],
                   KeyDistribution(case["kind"], case["exponent"]), case["num_items"])
    reqs = list(generate_workload(spec))
    h = hashlib.sha256()
    for r in reqs:
        h.update(np.int64(r.user_id).tobytes())
        h.update(r.history_item_ids.astype(np.int64).tobytes())
        h.update(r.candidate_item_ids.astype(np.int64).tobytes())
    assert [len(r.candidate_item_ids) for r in reqs] == case["cand_counts"]
    assert reqs[0].user_id == case["first_user_id"]
    assert reqs[0].history_item_ids[:8].tolist() == case["first_hist_head"]
    assert h.hexdigest() == case["sha256"]


def test_same_seed_identical_streams_and_scenario_shapes():
    a = list(generate_workload(spec_of(Scenario.MIXED, 25)))
    b = list(generate_workload(spec_of(Scenario.MIXED, 25)))
    for ra, rb in zip(a, b):
        assert ra.user_id == rb.user_id
        np.testing.assert_array_equal(ra.candidate_item_ids, rb.candidate_item_ids)
    for r in generate_workload(spec_of(Scenario.BASE, 10)):
        assert (len(r.history_item_ids), len(r.candidate_item_ids)) == (512, 128)
    for r in generate_workload(spec_of(Scenario.LONG, 3)):
        assert (len(r.history_item_ids), len(r.candidate_item_ids)) == (1024, 512)
    counts = {128: 0, 256: 0, 512: 0, 1024: 0}
    for r in generate_workload(spec_of(Scenario.MIXED, 2000)):
        counts[len(r.candidate_item_ids)] += 1
    assert all(400 <= n <= 600 for n in counts.values()), counts


def test_infinite_stream_and_zipf_skew():
    stream = generate_workload(WorkloadSpec(scenario=Scenario.BASE, duration_s=1.0, concurrency=1, seed=1))
    assert len(list(itertools.islice(stream, 50))) == 50
    ids = np.concatenate([r.history_item_ids for r in generate_workload(spec_of(Scenario.MIXED, 30))])
    assert (ids < 50).mean() > 0.3
    uids = np.concatenate([r.history_item_ids for r in
                           generate_workload(spec_of(Scenario.MIXED, 30, dist=KeyDistribution("uniform")))])
    assert (uids < 50).mean() < 0.05


def test_spec_validation():
    with pytest.raises(ValueError):
        KeyDistribution("pareto")
    with pytest.raises(ValueError):
        KeyDistribution("zipf", 0.0)
    with pytest.raises(ValueError):
        WorkloadSpec(concurrency=0)
    with pytest.raises(ValueError):
        WorkloadSpec(num_requests=0)
    with pytest.raises(ValueError):
        WorkloadSpec(num_items=0)


def sample_report():
    return RunReport(**GOLDEN["report"]["fields"])


def test_report_bytes_match_reference(tmp_path):
    path = tmp_path / "r.csv"
    emit_report(sample_report(), path)
    assert path.read_text() == GOLDEN["report"]["csv"]
    assert path.read_text().splitlines()[0] == CSV_HEADER


def test_report_round_trip_and_reload_of_reference_bytes(tmp_path):
    path = tmp_path / "r.csv"
    emit_report(sample_report(), path)
    assert load_report(path) == sample_report()
    ref = tmp_path / "ref.csv"
    ref.write_text(GOLDEN["report"]["csv"])
    assert load_report(ref) == sample_report()
    bad = tmp_path / "nope.csv"
    bad.write_text("a,b,c\n1,2,3\n")
    with pytest.raises(ValueError):
        load_report(bad)


def test_zero_duration_run_is_an_error():
    cfg = ServiceConfig(model=ModelConfig(32, 8, 2, 1, 64, 2, 1024, 1024, seed=5))
    with pytest.raises(EmptyRunError):
        run_scenario(WorkloadSpec(scenario=Scenario.BASE, duration_s=0.0, concurrency=1), AblationConfig(), cfg)


def test_service_config_from_reference_json():
    d = {"model": {"hidden_dim": 32, "head_dim": 8, "num_blocks": 2, "layers_per_block": 1, "ffn_dim": 64,
                   "num_tasks": 2, "max_history_len": 1024, "max_candidates": 1024, "seed": 5},
         "cache": {"bucket_count": 16}, "remote_store": {"latency_ms_mean": 1.0}, "listen_addr": "127.0.0.1:9000",
         "cache_enabled": False, "mem_opt": True,
         "orchestrator": {"profile_shapes": [128, 256], "executors_per_shape": 2, "routing": "implicit"}}
    cfg = ServiceConfig.from_dict(d)
    assert cfg.model.hidden_dim == 32 and cfg.model.max_history_len == 1024
    assert (cfg.cache_enabled, cfg.mem_opt, cfg.routing, cfg.profile_shapes) == (False, True, "implicit", (128, 256))
    abl = cfg.with_ablation(True, False, "explicit")
    assert (abl.cache_enabled, abl.mem_opt, abl.routing) == (True, False, "explicit")
    with pytest.raises(ValueError):
        ServiceConfig(model=cfg.model, routing="adaptive")
