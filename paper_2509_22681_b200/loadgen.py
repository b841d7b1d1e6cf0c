"""Load generator and ablation runner over the device request path — the
reference's ``flameserve.bench`` (pkg/src/flameserve/bench.py) driving a
``DeviceService`` instead of the host service.

Same scenarios (``SCENARIO_SHAPES``, bench.py:50-55), the same deterministic
request stream for a seed (``generate_workload``, bench.py:130-144: one
``default_rng(seed)`` drawing, per request, the candidate count, a 32-bit user
id, the history ids and the candidate ids, Zipf through an explicit rank CDF),
the same ablation toggles and the same one-row CSV report (``CSV_HEADER``,
byte-identical header, ``repr`` floats, ``on``/``off`` flags) so reports from
either implementation load with either ``load_report``.

What the columns measure here:

* ``throughput_pairs_per_s`` — candidates scored per second of the run window,
  with ``concurrency`` client threads calling ``handle_request``; concurrent
  requests are coalesced into DSO batches by the service;
* ``compute_ms_*`` — dispatch to collection of the request's group on the GPU;
* ``cache_hit_rate`` — share of ids served by the HBM item table (0 with
  ``cache`` off, when the host resolves every id from its store copy); with a
  ``cache`` section in the service config the table runs the reference's cache
  semantics (``feature_cache.py``) and the rate is the reference's
  (fresh + stale hits) / lookups;
* ``network_bytes`` — feature bytes moved host -> device in the run (8 B per
  id with the device table, 4·d B per id without, plus row refreshes);
* ``steady_state_allocs`` — executor buffers allocated after startup (0 for
  ``explicit`` routing over warmed buckets; every request allocates with
  ``implicit``).
"""

from __future__ import annotations

import argparse
import csv
import dataclasses
import threading
import time
from dataclasses import dataclass
from enum import Enum
from pathlib import Path
from typing import Callable, Iterator

import numpy as np

from .service import DeviceService, ScoreRequest, ServiceConfig, _percentile

CSV_HEADER = ("scenario,cache,mem_opt,routing,throughput_pairs_per_s,overall_ms_mean,overall_ms_p99,"
              "compute_ms_mean,compute_ms_p99,cache_hit_rate,network_bytes,steady_state_allocs")


class EmptyRunError(RuntimeError):
    """The run completed no request to report on."""


class Scenario(Enum):
    BASE = "base"
    LONG = "long"
    MIXED = "mixed"


#: scenario -> (history length, candidate-count choices)
SCENARIO_SHAPES = {
    Scenario.BASE: (512, (128,)),
    Scenario.LONG: (1024, (512,)),
    Scenario.MIXED: (1024, (128, 256, 512, 1024)),
}


@dataclass(frozen=True)
class KeyDistribution:
    kind: str = "zipf"  # "uniform" | "zipf"
    exponent: float = 1.0

    def __post_init__(self) -> None:
        if self.kind not in ("uniform", "zipf"):
            raise ValueError(f"unknown key distribution {self.kind!r}")
        if self.kind == "zipf" and self.exponent <= 0:
            raise ValueError("zipf exponent must be positive")

    def sampler(self, num_items: int) -> Callable[[np.random.Generator, int], np.ndarray]:
        """Id sampler over [0, num_items) (reference _KeySampler, bench.py:112-127):
        uniform integers, or Zipf ranks by inverse CDF, ``searchsorted(cdf, u)``."""
        if self.kind == "uniform":
            return lambda rng, n: rng.integers(0, num_items, size=n, dtype=np.int64)
        return _ZipfInverseCdf(num_items, self.exponent)


class _ZipfInverseCdf:
    """``np.searchsorted(cdf, u)`` (first rank whose CDF reaches u) through a
    guide table: ``K`` equal slices of [0, 1), each knowing the first rank at
    or above its lower edge, so a draw resolves in a few vectorised compares
    instead of a 17-level binary search over the whole CDF.  Exact: with K a
    power of two, slice j = floor(u·K) satisfies j/K <= u < (j+1)/K in floating
    point, so the answer lies in [guide[j], guide[j+1]].  Results are identical
    to the reference's sampler; the driver just stops being the bottleneck."""

    def __init__(self, num_items: int, exponent: float) -> None:
        w = 1.0 / np.arange(1, num_items + 1, dtype=np.float64) ** exponent
        self.cdf = np.cumsum(w / w.sum())
        self.K = int(min(1 << 22, max(1024, 16 << int(np.ceil(np.log2(num_items))))))
        self.guide = np.searchsorted(self.cdf, np.arange(self.K + 1, dtype=np.float64) / self.K)
        self.span = int(np.max(np.diff(self.guide)))
        self.cdf_pad = np.append(self.cdf, np.inf)  # cdf[n] = inf stops the walk at n

    def __call__(self, rng: np.random.Generator, n: int) -> np.ndarray:
        u = rng.random(n)
        j = (u * self.K).astype(np.int64)
        r = self.guide[j]
        for _ in range(self.span):
            r += self.cdf_pad[r] < u
        return r.astype(np.int64, copy=False)


@dataclass(frozen=True)
class WorkloadSpec:
    scenario: Scenario = Scenario.MIXED
    duration_s: float = 10.0
    concurrency: int = 8
    key_distribution: KeyDistribution = KeyDistribution()
    seed: int = 0
    num_requests: int | None = None  # finite stream when set, else bounded by duration_s
    num_items: int = 100_000

    def __post_init__(self) -> None:
        if self.concurrency < 1:
            raise ValueError("concurrency must be >= 1")
        if self.num_items < 1:
            raise ValueError("num_items must be >= 1")
        if self.num_requests is not None and self.num_requests < 1:
            raise ValueError("num_requests must be >= 1 when set")


@dataclass(frozen=True)
class AblationConfig:
    cache: bool = True
    mem_opt: bool = True
    routing: str = "explicit"


@dataclass(frozen=True)
class RunReport:
    scenario: str
    cache: bool
    mem_opt: bool
    routing: str
    throughput_pairs_per_s: float
    overall_ms_mean: float
    overall_ms_p99: float
    compute_ms_mean: float
    compute_ms_p99: float
    cache_hit_rate: float
    network_bytes: int
    steady_state_allocs: int


def generate_workload(spec: WorkloadSpec) -> Iterator[ScoreRequest]:
    """The deterministic request stream of a spec (finite iff num_requests)."""
    rng = np.random.default_rng(spec.seed)
    sample = spec.key_distribution.sampler(spec.num_items)
    hist_len, choices = SCENARIO_SHAPES[spec.scenario]
    k = 0
    while spec.num_requests is None or k < spec.num_requests:
        # rng.choice over a short tuple draws exactly integers(0, len): same stream, 5x cheaper
        c = choices[int(rng.integers(0, len(choices)))] if len(choices) > 1 else choices[0]
        user = int(rng.integers(0, 2**32))
        hist = sample(rng, hist_len)
        yield ScoreRequest(user_id=user, history_item_ids=hist, candidate_item_ids=sample(rng, c), context={})
        k += 1


def _drive(spec: WorkloadSpec, call: Callable[[ScoreRequest], None]) -> float:
    """Run ``concurrency`` threads pulling from the stream until it ends or the
    deadline passes; returns the active seconds; re-raises the first error."""
    stream = generate_workload(spec)
    feed = threading.Lock()
    errors: list = []
    t0 = time.perf_counter()
    deadline = None if spec.num_requests is not None else t0 + spec.duration_s

    def worker() -> None:
        while deadline is None or time.perf_counter() < deadline:
            with feed:
                req = next(stream, None)
            if req is None:
                return
            try:
                call(req)
            except BaseException as exc:  # noqa: BLE001 - re-raised after join
                errors.append(exc)
                return

    threads = [threading.Thread(target=worker, daemon=True) for _ in range(spec.concurrency)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    return time.perf_counter() - t0


def _report(spec, ablation, metrics: dict, active_s: float, overall=None, compute=None) -> RunReport:
    if overall is None:
        o, c = metrics["overall_ms"], metrics["compute_ms"]
        if not o.get("count"):
            raise EmptyRunError("no requests completed in the run window")
        o_mean, o_p99, c_mean, c_p99, pairs = o["mean"], o["p99"], c["mean"], c["p99"], metrics["pairs_processed"]
    else:
        if not overall:
            raise EmptyRunError("no requests completed against the remote server")
        pairs = metrics["pairs_client"]
        o_mean, o_p99 = sum(overall) / len(overall), _percentile(overall, 0.99)
        c_mean, c_p99 = sum(compute) / len(compute), _percentile(compute, 0.99)
    return RunReport(scenario=spec.scenario.value, cache=ablation.cache, mem_opt=ablation.mem_opt,
                     routing=ablation.routing, throughput_pairs_per_s=pairs / active_s,
                     overall_ms_mean=o_mean, overall_ms_p99=o_p99, compute_ms_mean=c_mean, compute_ms_p99=c_p99,
                     cache_hit_rate=float(metrics["cache"]["hit_rate"]),
                     network_bytes=int(metrics["network_bytes"]),
                     steady_state_allocs=int(metrics["steady_state_allocs"]))


def scenario_shapes(spec: WorkloadSpec) -> list[tuple[int, int]]:
    hist_len, choices = SCENARIO_SHAPES[spec.scenario]
    return [(hist_len, c) for c in choices]


def run_scenario(spec: WorkloadSpec, ablation: AblationConfig, service_config: ServiceConfig,
                 on_drained: "Callable[[DeviceService], None] | None" = None) -> RunReport:
    """Start a DeviceService in-process with the ablation applied, warm the
    scenario's buckets, drive the workload, drain and report (reference
    run_scenario, bench.py:147-199)."""
    if spec.num_requests is None and spec.duration_s <= 0:
        raise EmptyRunError("duration_s must be positive for duration-bound runs")
    cfg = service_config.with_ablation(ablation.cache, ablation.mem_opt, ablation.routing)
    if cfg.num_items != spec.num_items:
        cfg = dataclasses.replace(cfg, num_items=spec.num_items)
    service = DeviceService.from_config(cfg)
    try:
        service.warm(scenario_shapes(spec))
        active = _drive(spec, service.handle_request)
        report = _report(spec, ablation, service.metrics_snapshot(), active)
        if on_drained is not None:
            on_drained(service)
    finally:
        service.close()
    return report


def run_scenario_remote(spec: WorkloadSpec, ablation: AblationConfig, base_url: str) -> RunReport:
    """Drive a separately started server over HTTP (``api.create_app``) and
    report client-side latencies (reference bench.py:228-301)."""
    import httpx

    overall: list = []
    compute: list = []
    pairs = [0]
    lock = threading.Lock()
    local = threading.local()

    def call(req: ScoreRequest) -> None:
        if not hasattr(local, "client"):
            local.client = httpx.Client(base_url=base_url, timeout=60.0)
        t0 = time.perf_counter()
        resp = local.client.post("/score", json={"user_id": req.user_id, "history": req.history_item_ids.tolist(),
                                                 "candidates": req.candidate_item_ids.tolist(),
                                                 "context": req.context})
        resp.raise_for_status()
        body = resp.json()
        with lock:
            overall.append((time.perf_counter() - t0) * 1000.0)
            compute.append(body["compute_latency_ms"])
            pairs[0] += len(req.candidate_item_ids)

    active = _drive(spec, call)
    with httpx.Client(base_url=base_url, timeout=10.0) as client:
        metrics = client.get("/metrics").json()
    metrics["pairs_client"] = pairs[0]
    return _report(spec, ablation, metrics, active, overall, compute)


# ------------------------------------------------------------------ reports

def _cell(report: RunReport, f: dataclasses.Field) -> str:
    v = getattr(report, f.name)
    if f.type in ("bool", bool):
        return "on" if v else "off"
    if f.type in ("float", float):
        return repr(float(v))
    return str(v)


def _parse(f: dataclasses.Field, text: str):
    if f.type in ("bool", bool):
        return text == "on"
    if f.type in ("float", float):
        return float(text)
    if f.type in ("int", int):
        return int(text)
    return text


def emit_report(report: RunReport, path: str | Path) -> None:
    """Write the one-row CSV report and print a one-line summary."""
    fields = dataclasses.fields(RunReport)
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(CSV_HEADER.split(","))
        w.writerow([_cell(report, f) for f in fields])
    r = report
    print(f"{r.scenario} cache={'on' if r.cache else 'off'} mem_opt={'on' if r.mem_opt else 'off'} "
          f"routing={r.routing}: {r.throughput_pairs_per_s:.1f} pairs/s, "
          f"overall {r.overall_ms_mean:.2f} ms (p99 {r.overall_ms_p99:.2f}), "
          f"compute {r.compute_ms_mean:.2f} ms (p99 {r.compute_ms_p99:.2f}), "
          f"hit rate {r.cache_hit_rate:.2%}, net {r.network_bytes} B, allocs {r.steady_state_allocs}")


def load_report(path: str | Path) -> RunReport:
    """Parse a report written by ``emit_report`` (either implementation's)."""
    with open(path, newline="") as fh:
        rows = list(csv.reader(fh))
    if len(rows) != 2 or rows[0] != CSV_HEADER.split(","):
        raise ValueError(f"{path} is not a single-run report file")
    fields = dataclasses.fields(RunReport)
    if len(rows[1]) != len(fields):
        raise ValueError(f"{path}: expected {len(fields)} columns")
    return RunReport(**{f.name: _parse(f, t) for f, t in zip(fields, rows[1])})


def main(argv=None) -> None:
    """``python -m paper_2509_22681_b200.loadgen --config service.json ...``:
    one ablation run, CSV report to ``--out`` (reference flame-bench)."""
    import json

    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--config", required=True, help="service JSON (reference format)")
    ap.add_argument("--scenario", choices=[s.value for s in Scenario], default="mixed")
    ap.add_argument("--duration", type=float, default=10.0)
    ap.add_argument("--requests", type=int, default=None)
    ap.add_argument("--concurrency", type=int, default=8)
    ap.add_argument("--keys", choices=["zipf", "uniform"], default="zipf")
    ap.add_argument("--zipf-exponent", type=float, default=1.0)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--num-items", type=int, default=100_000)
    ap.add_argument("--cache", choices=["on", "off"], default="on")
    ap.add_argument("--mem-opt", choices=["on", "off"], default="on")
    ap.add_argument("--routing", choices=["explicit", "implicit"], default="explicit")
    ap.add_argument("--remote", default=None, help="base URL of a running server")
    ap.add_argument("--out", default="report.csv")
    a = ap.parse_args(argv)
    spec = WorkloadSpec(Scenario(a.scenario), a.duration, a.concurrency, KeyDistribution(a.keys, a.zipf_exponent),
                        a.seed, a.requests, a.num_items)
    abl = AblationConfig(a.cache == "on", a.mem_opt == "on", a.routing)
    if a.remote:
        report = run_scenario_remote(spec, abl, a.remote)
    else:
        report = run_scenario(spec, abl, ServiceConfig.from_dict(json.loads(Path(a.config).read_text())))
    emit_report(report, a.out)


if __name__ == "__main__":
    main()
