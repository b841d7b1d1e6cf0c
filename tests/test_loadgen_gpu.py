"""Ablation runner over the device request path (reference tests/test_bench.py
runner cases): reports, cache / mem_opt / routing toggles, request coalescing
under concurrency, and the remote HTTP driver."""

import socket
import threading
import time

import numpy as np
import pytest

from paper_2509_22681_b200.config import ModelConfig
from paper_2509_22681_b200.loadgen import (AblationConfig, KeyDistribution, Scenario, WorkloadSpec,
                                           generate_workload, run_scenario, run_scenario_remote)
from paper_2509_22681_b200.service import DeviceService, ServiceConfig

pytestmark = pytest.mark.gpu

MODEL = ModelConfig(32, 8, 2, 1, 64, 2, 1024, 1024, seed=5)


def bench_config(**kw):
    kw.setdefault("target_rows", 2048)
    return ServiceConfig(model=MODEL, num_items=5000, **kw)


def spec_of(scenario, n, seed=3, concurrency=4):
    return WorkloadSpec(scenario=scenario, duration_s=60.0, concurrency=concurrency,
                        key_distribution=KeyDistribution("zipf", 1.0), seed=seed, num_requests=n, num_items=5000)


def test_small_run_produces_sane_report(gpu):
    captured = {}
    t0 = time.perf_counter()
    report = run_scenario(spec_of(Scenario.BASE, 30), AblationConfig(), bench_config(),
                          on_drained=lambda s: captured.update(s.metrics_snapshot()))
    wall = time.perf_counter() - t0
    assert captured["pairs_processed"] == 30 * 128
    assert report.scenario == "base" and report.routing == "explicit"
    assert 0 < captured["pairs_processed"] / report.throughput_pairs_per_s <= wall
    assert report.overall_ms_mean >= report.compute_ms_mean >= 0
    assert report.cache_hit_rate == 1.0  # every Zipf id is inside the 5000-row table
    assert report.steady_state_allocs == 0
    assert report.network_bytes == 30 * (512 + 128) * 8


def test_cache_toggle(gpu):
    spec = spec_of(Scenario.BASE, 12)
    on = run_scenario(spec, AblationConfig(cache=True), bench_config())
    off = run_scenario(spec, AblationConfig(cache=False), bench_config())
    assert on.network_bytes < off.network_bytes == 12 * (512 + 128) * 4 * MODEL.hidden_dim
    assert off.cache_hit_rate == 0.0


def test_routing_toggle_flips_allocation_counter(gpu):
    spec = spec_of(Scenario.BASE, 6)
    assert run_scenario(spec, AblationConfig(routing="explicit"), bench_config()).steady_state_allocs == 0
    assert run_scenario(spec, AblationConfig(routing="implicit"), bench_config()).steady_state_allocs > 0


def test_ablations_score_alike(gpu):
    """Every (cache, mem_opt, routing) combination scores the same requests
    within bf16 tolerance of the default path (identically for mem_opt)."""
    reqs = list(generate_workload(spec_of(Scenario.MIXED, 6)))
    base = None
    for cache in (True, False):
        for mem_opt in (True, False):
            for routing in ("explicit", "implicit"):
                svc = DeviceService.from_config(bench_config().with_ablation(cache, mem_opt, routing))
                got = [svc.handle_request(r).scores for r in reqs]
                svc.close()
                if base is None:
                    base = got
                for g, b in zip(got, base):
                    assert g.shape == b.shape
                    assert np.abs(g - b).max() <= 2e-2, (cache, mem_opt, routing)
                    if routing == "explicit" and cache:
                        np.testing.assert_array_equal(g, b)


def test_concurrent_callers_are_coalesced(gpu):
    """Many client threads: results equal one-at-a-time scoring, and the
    service dispatched fewer batches than requests."""
    svc = DeviceService.from_config(bench_config())
    reqs = list(generate_workload(spec_of(Scenario.MIXED, 48, seed=9)))
    want = [svc.handle_request(r).scores for r in reqs[:12]]
    calls = {"n": 0}
    orig = svc._submit

    def counting(batch):
        calls["n"] += 1
        return orig(batch)

    svc._submit = counting
    got = [None] * len(reqs)

    def worker(k):
        for i in range(k, len(reqs), 8):
            got[i] = svc.handle_request(reqs[i]).scores

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(8)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for g, w in zip(got[:12], want):
        np.testing.assert_array_equal(g, w)
    assert all(g is not None for g in got)
    assert calls["n"] < len(reqs)
    svc.close()


def test_remote_driver_against_live_server(gpu):
    import uvicorn

    from paper_2509_22681_b200.api import create_app

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    service = DeviceService.from_config(bench_config())
    server = uvicorn.Server(uvicorn.Config(create_app(service), host="127.0.0.1", port=port, log_level="warning"))
    thread = threading.Thread(target=server.run, daemon=True)
    thread.start()
    deadline = time.time() + 20
    while not server.started:
        assert time.time() < deadline, "server did not start"
        time.sleep(0.02)
    try:
        spec = WorkloadSpec(scenario=Scenario.BASE, duration_s=30.0, concurrency=2, seed=5, num_requests=6,
                            num_items=1000)
        report = run_scenario_remote(spec, AblationConfig(), f"http://127.0.0.1:{port}")
        assert report.throughput_pairs_per_s > 0
        assert report.network_bytes > 0
        assert report.cache_hit_rate == 1.0
    finally:
        server.should_exit = True
        thread.join(timeout=10)
