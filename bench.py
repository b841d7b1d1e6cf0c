#!/usr/bin/env python
"""FLAME SUMI-ranker hot path on B200 — benchmark (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg3] [--impl ours|reference]

A *step* is one pass of the hot path over one batch of R synthetic requests:
device feature assembly (PDA dedup + gather from the HBM item table) ->
per-block LN+QKV -> SUMI attention -> O-proj -> LN2+FFN -> gated fusion ->
expert heads, i.e. reference ``Service.resolve_embeddings`` + ``model_forward``
(pkg/src/flameserve/service.py:97-108, model/forward.py:186-204), replayed as
one CUDA graph.  Metric: candidates scored / s (whole job, all ranks).

* ``value``  device-timed (CUDA events on the executor stream) with the ids
  already resident in HBM; K back-to-back graph replays.  Per-step working set
  is several GB, far larger than the 126 MB L2, so no flush is needed.
* ``e2e``    the same metric through the public API (``DeviceExecutor.score_ids``):
  host ids -> pinned staging -> H2D -> forward -> D2H scores -> numpy, per step.
* ``roofline`` the dominant kernel, timed live with per-launch CUDA events in
  an eager profiling pass before the timed region (``roofline.hot``: the same
  right after it); FLOPs are algorithmic.
* ``fp32_verify`` the same step in the fp32 verification mode.
* ``cpu_baseline`` the unmodified reference (installed in baseline/_ref) on
  this host's cores — or, without that install, the numpy oracle port of it
  (oracle/) — rank 0, N = 1 only, a bounded sample of the same workload.
* ``--impl reference`` times that CPU reference path alone (rank 0; other
  ranks exit without work).

Multi-GPU (torchrun, one process per GPU): requests are sharded whole across
ranks with no collective on the data path (weak scaling: R requests per rank
per step); barrier + device sync bracket the timed region and the duration is
the MAX over ranks.
"""

from __future__ import annotations

import argparse
import gc
import json
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# name: (d, dh, N_b, L, f, tasks, H, C, requests per step per GPU, description)
WORKLOADS = {
    "cfg1": (64, 16, 2, 1, 256, 2, 256, 64, 1024,
             "smallest GR ranker: 2 blocks d=64 4 heads, user seq 256, 64 candidates"),
    "cfg2": (256, 64, 4, 1, 1024, 2, 1024, 256, 128,
             "Climber ranker: 4 blocks d=256, user seq 1024, 256 candidates/request"),
    "cfg3": (512, 64, 8, 1, 2048, 2, 2048, 512, 64,
             "production shape: 8 blocks d=512, user seq 2048, 512 candidates/request"),
    "cfg4": (256, 64, 4, 1, 1024, 2, 1024, 2048, 256,
             "DSO: Climber ranker d=256 4 blocks, user seq 1024, Zipf candidate counts 16-2048 per request"),
    "cfg3_l2": (512, 64, 8, 2, 2048, 2, 2048, 512, 64,
                "SURVEY 8 sensitivity row: cfg3 with 2 layers per block (non-final layer: causal history "
                "attention + full-row Q/K/V, O-proj, FFN)"),
    "cfg5": (768, 64, 12, 1, 3072, 2, 8184, 1024, 8,
             "long-history stress: 12 blocks d=768, user seq 8184 (=12x682), 1024 candidates"),
}
NUM_ITEMS = 100_000       # reference bench default universe (bench.py:78)
WORKLOAD_SEED = 2509
WEIGHT_SEED = 0
STORE_SEED = 1234
METRIC = "candidates scored/sec (1/2/4/8 B200) and p99 request latency vs CPU ref"
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def zipf_sampler(num_items: int, exponent: float = 1.0):
    """Reference bench.py:112-127 _KeySampler (Zipf over ranks, explicit CDF)."""
    w = 1.0 / np.arange(1, num_items + 1, dtype=np.float64) ** exponent
    cdf = np.cumsum(w / w.sum())
    return lambda rng, n: np.searchsorted(cdf, rng.random(n)).astype(np.int64)


ZIPF_C = {"cfg4"}  # workloads with per-request candidate counts C = 16 + Zipf(1.0) rank over 2033


def make_requests(n: int, H: int, C: int, seed: int, zipf_c: bool = False):
    """n requests of (H history ids, C candidate ids), ids Zipf(1.0) over the item
    universe (reference bench.py:130-144).  zipf_c: C_i = 16 + Zipf rank in
    [0, 2033), so 16 <= C_i <= 2048 = C."""
    rng = np.random.default_rng(seed)
    sample = zipf_sampler(NUM_ITEMS)
    if zipf_c:
        counts = 16 + zipf_sampler(C - 16 + 1)(rng, n)
    else:
        counts = np.full(n, C)
    return [(sample(rng, H), sample(rng, int(c))) for c in counts]


def model_config(name: str):
    import paper_2509_22681_b200 as fb

    d, dh, nb, L, f, tasks, H, C, *_ = WORKLOADS[name]
    return fb.ModelConfig(d, dh, nb, L, f, tasks, H, C, seed=WEIGHT_SEED)


def load_peaks() -> tuple[dict, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return json.loads(p.read_text()), "measured"
        except Exception:
            pass
    return dict(FALLBACK_PEAKS), "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock + throttle reasons sampled every 10 ms through NVML on a
    background thread while the timed region runs (nvidia-smi's 200 ms loop
    would see only a couple of samples of a short region)."""

    REASONS = {
        "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4,
    }

    def __init__(self, index: int, period_s: float = 0.01) -> None:
        self.index = index
        self.period = period_s
        self.samples: list[tuple[int, int]] = []
        self.max_mhz = None
        self._stop = threading.Event()
        self._thread = None
        self.error = None

    def start(self) -> None:
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception as exc:  # NVML unavailable: record why
            self.error = str(exc)
            return

        def loop():
            while not self._stop.is_set():
                try:
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((sm, rs))
                except Exception as exc:
                    self.error = str(exc)
                    return
                time.sleep(self.period)

        self._thread = threading.Thread(target=loop, daemon=True)
        self._thread.start()

    def begin(self) -> None:
        """The timed region starts now: earlier (idle) samples are not reported."""
        self._begin = len(self.samples)

    def stop(self) -> dict:
        self._stop.set()
        if self._thread is not None:
            self._thread.join(timeout=2)
        # samples from begin() to stop(); the last pre-begin sample if the region was shorter than a period
        b = getattr(self, "_begin", 0)
        samples = self.samples[b:] or self.samples[max(0, b - 1):b]
        if not samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "samples": 0,
                    "reasons": [f"no samples: {self.error}"]}
        reasons = sorted({n for _, rs in samples for n, bit in self.REASONS.items() if rs & bit})
        return {"sm_mhz": statistics.median(sm for sm, _ in samples), "sm_min_mhz": min(sm for sm, _ in samples),
                "sm_max_mhz": self.max_mhz, "samples": len(samples), "reasons": reasons,
                "source": "NVML, 10 ms, timed region only"}


# ------------------------------------------------------------- CPU oracle
def _oracle_worker(args):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    name, reqs = args
    sys.path.insert(0, str(ROOT))
    import paper_2509_22681_b200 as fb
    from oracle import flame_oracle as orc
    from paper_2509_22681_b200.pda import item_embedding

    cfg = model_config(name)
    params = fb.init_params(cfg)
    lat = []
    t_all = time.perf_counter()
    for hid, cid in reqs:
        t0 = time.perf_counter()
        # resolve_embeddings (service.py:97-108): unique ids -> store rows -> expand
        rows = []
        for ids in (hid, cid):
            uq, inv = np.unique(ids, return_inverse=True)
            tab = np.stack([item_embedding(STORE_SEED, int(u), 0, cfg.hidden_dim) for u in uq])
            rows.append(tab[inv])
        orc.model_forward(rows[0], rows[1], params, cfg)
        lat.append(time.perf_counter() - t0)
    return time.perf_counter() - t_all, lat


# the unmodified reference, pip-installed offline into baseline/_ref;
# when present the CPU arm runs IT, else the oracle port pinned to it
REF_PKG = ROOT / "baseline" / "_ref"
REF_AVAILABLE = (REF_PKG / "flameserve" / "service.py").exists()
CPU_KIND = "reference" if REF_AVAILABLE else "port"
CPU_WHAT = ("unmodified reference (baseline/_ref) Service.handle_request: sync feature cache over the "
            "simulated store (0 ms latency), implicit-shape runner -> numpy fp64 model_forward"
            if REF_AVAILABLE else
            "numpy fp64 oracle port of reference resolve_embeddings + model_forward")


def _reference_worker(args):
    """The reference's own request path (service.py:127-171) on one host process."""
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    name, reqs = args
    sys.path.insert(0, str(REF_PKG))
    from flameserve.cache import CacheConfig, CacheMode
    from flameserve.config import OrchestratorConfig, ServiceConfig
    from flameserve.model import ModelConfig
    from flameserve.service import ScoreRequest, Service
    from flameserve.store import RemoteStoreConfig

    c = model_config(name)
    cfg = ServiceConfig(
        model=ModelConfig(c.hidden_dim, c.head_dim, c.num_blocks, c.layers_per_block, c.ffn_dim, c.num_tasks,
                          c.max_history_len, c.max_candidates, seed=c.seed),
        cache=CacheConfig(mode=CacheMode.SYNC), remote_store=RemoteStoreConfig(0.0, 0.0, seed=STORE_SEED),
        orchestrator=OrchestratorConfig(routing="implicit"))
    svc = Service(cfg)
    lat = []
    t_all = time.perf_counter()
    for k, (hid, cid) in enumerate(reqs):
        t0 = time.perf_counter()
        svc.handle_request(ScoreRequest(user_id=k, history_item_ids=hid, candidate_item_ids=cid))
        lat.append(time.perf_counter() - t0)
    busy = time.perf_counter() - t_all
    svc.close()
    return busy, lat


def cpu_reference_sample(name: str, n_requests: int, procs: int, seed: int) -> dict:
    """Time the reference CPU path (or, without baseline/_ref, the oracle port) on
    ``procs`` host processes (1 BLAS thread each)."""
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    reqs = make_requests(n_requests, WORKLOADS[name][6], WORKLOADS[name][7], seed, name in ZIPF_C)
    chunks = [(name, reqs[i::procs]) for i in range(procs) if reqs[i::procs]]
    ctx = mp.get_context("spawn")
    t0 = time.perf_counter()
    with ctx.Pool(len(chunks)) as pool:
        res = pool.map(_reference_worker if REF_AVAILABLE else _oracle_worker, chunks)
    wall = time.perf_counter() - t0
    lat = sorted(x for _, l in res for x in l)
    return {"wall_s": wall, "busy_s": max(r[0] for r in res), "requests": n_requests,
            "cands": sum(len(c) for _, c in reqs), "lat": lat, "procs": len(chunks)}


def nearest_rank(series, p):
    """Reference metrics.py:11-19 nearest-rank percentile."""
    s = sorted(series)
    k = max(1, int(np.ceil(p * len(s))))
    return s[k - 1]


# ------------------------------------------------------------------- main
REF_REQS_PER_PROC = {"cfg1": 32, "cfg2": 2, "cfg3": 1, "cfg3_l2": 1, "cfg4": 2, "cfg5": 1}


def run_reference(args, dist) -> None:
    if dist.rank != 0:
        return
    name = args.workload
    cores = len(os.sched_getaffinity(0))
    procs = max(1, min(cores, 32, int(os.environ.get("FLAME_BENCH_CPU_PROCS", "32"))))
    per = REF_REQS_PER_PROC.get(name, 1)
    C = WORKLOADS[name][7]
    cpu = _cpu_name()
    for w in range(args.warmup):
        cpu_reference_sample(name, procs, procs, WORKLOAD_SEED + 7 + w)
    step_s, lats, cands = [], [], 0
    for k in range(args.steps):
        r = cpu_reference_sample(name, per * procs, procs, WORKLOAD_SEED + 100 + k)
        step_s.append(r["busy_s"])  # compute loop only: excludes worker spawn / imports
        lats += r["lat"]
        cands += r["cands"]
    total = sum(step_s)
    value = cands / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "candidates/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (Zipf ids over 100k items, seeded)",
        "config": {"workload": name, "desc": WORKLOADS[name][9], "requests_per_step": per * procs,
                   "candidates_per_request": C, "history_len": WORKLOADS[name][6]},
        "p99_ms": 1000 * nearest_rank(lats, 0.99),
        "cpu_baseline": {"value": value, "unit": "candidates/s", "cores": procs, "kind": CPU_KIND,
                         "sample": f"{per * procs} requests per step ({procs} processes x 1 BLAS thread) "
                                   f"on {cpu}; {CPU_WHAT}"},
        "e2e": {"value": value, "unit": "candidates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _cpu_name() -> str:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown CPU"


def choose_peak(tensor: bool, clk: dict | None) -> tuple[float, str]:
    """Roofline denominator for a kernel timed under the clocks ``clk`` (the
    profile pass's own NVML record): the burst bf16 figure when the SM clock sat
    at its maximum with no power cap, the sustained one otherwise; HBM: the
    measured copy bandwidth."""
    peaks, src = load_peaks()
    if not tensor:
        return peaks.get("hbm_gbs", FALLBACK_PEAKS["hbm_gbs"]), f"{src} (hbm_gbs)"
    burst = bool(clk and clk.get("sm_mhz") and clk.get("sm_max_mhz")
                 and clk["sm_mhz"] >= 0.97 * clk["sm_max_mhz"]
                 and not {"sw_power_cap", "after-load"} & set(clk.get("reasons", [])))
    key = "bf16_tflops" if burst else "bf16_tflops_sustained"
    why = ("profile-pass SM clock at max, no power cap" if burst
           else "profile-pass SM clock below max, power-capped, or right after sustained load")
    return peaks.get(key, FALLBACK_PEAKS[key]), f"{src} ({key}: {why})"


def pda_algorithmic_bytes(ex, d: int, table_bytes: int) -> dict:
    """SURVEY §8(d) PDA bytes of the executor's last id pass, from the unique-id
    counts the dedup kernel wrote (n_unique): dedup = ids in + unique ids and
    inverse out; gather = one table row per UNIQUE id + the assembled rows
    (centered bf16 for every position, + the fp32 residual copy of candidates)."""
    import torch

    torch.cuda.synchronize()
    nu = ex.n_unique.cpu().numpy().astype(np.int64)
    R = ex.R
    meta = ex.meta.cpu().numpy().astype(np.int64)
    n = int(meta[3, 0])  # active slots (the dedup kernel skips the others)
    hl, cl = meta[0, :n], meta[1, :n]
    n_pos = int(hl.sum() + cl.sum())
    n_uniq = int(nu[:n].sum() + nu[R:R + n].sum())
    dedup = 8 * n_pos + 8 * n_uniq + 8 * n_pos
    gather = n_uniq * d * table_bytes + n_pos * d * 2 + int(cl.sum()) * d * 4
    return {"pda_dedup": float(dedup), "pda_gather": float(gather), "unique_rows": n_uniq, "positions": n_pos}


def roofline(prof_runs: list, name: str, prof_clk: dict | None = None, byte_override: dict | None = None):
    """Aggregate per-launch profiles ([[{name, ms, flops, bytes}]] of eager runs)
    into per-kernel figures and the dominant kernel's roofline point.  The peak
    follows the profile pass's own clock record (``choose_peak``)."""
    n_runs = len(prof_runs)
    agg: dict = {}
    times: dict = {}
    for run in prof_runs:
        for rec in run:
            a = agg.setdefault(rec["name"], {"ms": 0.0, "n": 0, "flops": 0.0, "bytes": 0.0})
            a["ms"] += rec["ms"]
            a["n"] += 1
            a["flops"] += rec["flops"]
            a["bytes"] += (byte_override or {}).get(rec["name"], rec["bytes"])
            times.setdefault(rec["name"], []).append(rec["ms"])
    # per-launch time = the median over the eager passes (one launch per role and
    # pass): robust to a single pass disturbed by host scheduling
    for k, a in agg.items():
        a["ms"] = statistics.median(times[k]) * a["n"]
    step_prof_ms = sum(a["ms"] for a in agg.values()) / n_runs
    top = max(agg, key=lambda k: agg[k]["ms"])
    t = agg[top]
    avg_ms = t["ms"] / t["n"]
    tensor = t["flops"] > 0
    per_launch = (t["flops"] if tensor else t["bytes"]) / t["n"]
    achieved = per_launch / (avg_ms / 1e3) / (1e12 if tensor else 1e9)
    peak, peak_src = choose_peak(tensor, prof_clk)
    peak_t, _ = choose_peak(True, prof_clk)
    peak_b, _ = choose_peak(False, prof_clk)
    traffic = None
    ncu = ROOT / "profiles" / "ncu_dram_per_launch.json"
    if ncu.exists():
        try:
            traffic = json.loads(ncu.read_text()).get(name, {}).get(top)
        except Exception:
            traffic = None
    kernels = {}
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1]["ms"]):
        tf = v["flops"] / (v["ms"] / 1e3) / 1e12 if v["flops"] else None
        gb = v["bytes"] / (v["ms"] / 1e3) / 1e9
        kernels[k] = {"ms_per_step": round(v["ms"] / n_runs, 4), "share": round(v["ms"] / n_runs / step_prof_ms, 4),
                      "tflops": round(tf, 1) if tf is not None else None, "gbs": round(gb, 1),
                      "frac": round(tf / peak_t, 4) if tf is not None else round(gb / peak_b, 4)}
    return tensor, top, achieved, peak, traffic, peak_src, per_launch, avg_ms, kernels


def profile_pass(ex, mode, runs: int, dev_index: int):
    """Per-launch CUDA-event profile of ``runs`` eager passes with its own NVML
    clock record (the roofline's peak is chosen from these clocks)."""
    ex.profile(mode)  # one untimed eager pass: host-side first-use work stays out of the record
    clocks = ClockSampler(dev_index, period_s=0.002)
    clocks.start()
    clocks.begin()
    prof = [ex.profile(mode) for _ in range(runs)]
    return prof, clocks.stop()


def cpu_baseline_line(args, dist, name: str):
    """The reference CPU path (or the oracle port) on this host's cores (rank 0,
    N = 1 only), bounded sample."""
    if dist.world_size != 1 or args.no_cpu_baseline:
        return None
    cores = len(os.sched_getaffinity(0))
    procs = max(1, min(cores, 32, int(os.environ.get("FLAME_BENCH_CPU_PROCS", "32"))))
    n_req = procs * 2 * REF_REQS_PER_PROC.get(name, 1)
    r = cpu_reference_sample(name, n_req, procs, WORKLOAD_SEED + 99)
    return {"value": r["cands"] / r["busy_s"], "unit": "candidates/s", "cores": r["procs"], "kind": CPU_KIND,
            "sample": f"{n_req} requests of {name} on {r['procs']} processes x 1 BLAS thread "
                      f"({_cpu_name()}), {CPU_WHAT}; compute {r['busy_s']:.1f}s; "
                      f"p99 {1000 * nearest_rank(r['lat'], 0.99):.0f} ms"}


def fp32_verify_line(eng, params, cfg, reqs, R, C, dev, step_flops, steps: int = 3) -> dict:
    """The same step in the fp32 verification mode (true-fp32 SIMT GEMMs and
    attention, the north star's <= 1e-4 mode): device-timed cand/s over a few
    graph replays, and the largest |fp32 - bf16| score difference on the batch."""
    import torch

    import paper_2509_22681_b200 as fb
    from paper_2509_22681_b200 import _lib
    from paper_2509_22681_b200.pda import build_item_table

    e32 = fb.FlameEngine(params, cfg, precision="fp32", device=dev.index)
    try:
        e32.set_table(build_item_table(NUM_ITEMS, cfg.hidden_dim, STORE_SEED), dtype="fp32")
        ex32 = e32.executor(R, cfg.max_history_len // cfg.num_blocks, C, with_ids=True)
        s32 = ex32.score_ids(reqs)
        s16 = eng.executor(R, cfg.max_history_len // cfg.num_blocks, C, with_ids=True).score_ids(reqs)
        diff = max(float(np.abs(a - b).max()) for a, b in zip(s32, s16))
        ex32.stage_ids(reqs)
        ex32.run(_lib.INPUT_IDS, graph=True)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        with torch.cuda.stream(ex32.stream):
            ev[0].record(ex32.stream)
            for _ in range(steps):
                ex32.run(_lib.INPUT_IDS, graph=True)
            ev[1].record(ex32.stream)
        ex32.stream.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / steps
    finally:
        e32.close()
    return {"value": R * C / (ms / 1e3), "unit": "candidates/s", "ms_per_step": ms, "steps": steps,
            "tflops": round(step_flops / (ms / 1e3) / 1e12, 1), "max_abs_vs_bf16": diff,
            "kernels": "fp32 FFMA SIMT GEMMs + fp32 SUMI attention (precision='fp32')"}


def run_ours(args, dist) -> None:
    import torch

    import paper_2509_22681_b200 as fb
    from paper_2509_22681_b200 import _lib
    from paper_2509_22681_b200.pda import build_item_table

    name = args.workload
    d, dh, nb, L, f, tasks, H, C, R_default, desc = WORKLOADS[name]
    R = args.requests or R_default
    dev = torch.device("cuda", dist.device_index)
    torch.cuda.set_device(dev)
    cfg = model_config(name)
    params = fb.init_params(cfg)
    eng = fb.FlameEngine(params, cfg, precision="bf16", device=dist.device_index)
    eng.set_table(build_item_table(NUM_ITEMS, d, STORE_SEED), dtype="fp32")
    reqs = make_requests(R, H, C, WORKLOAD_SEED + dist.rank)
    ex = eng.executor(R, H // nb, C, with_ids=True)
    ex.stage_ids(reqs)
    ex.run(_lib.INPUT_IDS, graph=True)  # capture + first replay
    ex.stream.synchronize()
    launches = ex.launch_count()

    # --------------------------------------------------- roofline (live)
    # eager per-launch CUDA events with their own clock record, BEFORE the timed
    # region: the kernels timed alone, at burst clocks (after sustained load the
    # power-capped state stretches the L2-bound kernels by up to 30 %,
    # dev/prof_ab.py; that state is reported separately as roofline.hot)
    prof, prof_clk = profile_pass(ex, _lib.INPUT_IDS, 5, dev.index)

    # ---------------------------------------------------- device-timed region
    for _ in range(args.warmup):
        ex.run(_lib.INPUT_IDS, graph=True)
    ex.stream.synchronize()
    torch.cuda.synchronize()
    dist.barrier()
    clocks = ClockSampler(dev.index)
    clocks.start()
    time.sleep(0.3)
    clocks.begin()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with torch.cuda.stream(ex.stream):
        evs[0].record(ex.stream)
        for k in range(args.steps):
            ex.run(_lib.INPUT_IDS, graph=True)
            evs[k + 1].record(ex.stream)
    ex.stream.synchronize()
    torch.cuda.synchronize()
    clk = clocks.stop()
    dist.barrier()
    step_ms = [evs[k].elapsed_time(evs[k + 1]) for k in range(args.steps)]
    total_ms = dist.max(sum(step_ms))
    p99_local = nearest_rank(step_ms, 0.99)
    p99 = dist.max(p99_local)
    cands = R * C * args.steps * dist.world_size
    value = cands / (total_ms / 1e3)

    pda = pda_algorithmic_bytes(ex, d, 4)
    tensor, top, achieved, peak, traffic, peak_src, per_launch, avg_ms, kernels = roofline(
        prof, name, prof_clk, {k: pda[k] for k in ("pda_dedup", "pda_gather")})
    # the same profile right after the timed region (the hot state of the step)
    prof_hot, hot_clk = profile_pass(ex, _lib.INPUT_IDS, 5, dev.index)
    h = roofline(prof_hot, name, hot_clk, {k: pda[k] for k in ("pda_dedup", "pda_gather")})
    hot_peak, hot_src = choose_peak(h[0], {**(hot_clk or {}), "reasons": ["after-load"]})
    hot = {"kernel": h[1], "avg_launch_ms": h[7], "achieved": round(h[2], 1), "peak": hot_peak,
           "frac": round(h[2] / hot_peak, 4), "peak_source": hot_src + " (after the timed region)",
           "clocks": hot_clk, "step_sum_ms": round(sum(v["ms_per_step"] for v in h[8].values()), 4)}

    # -------------------------------------------------------------- e2e
    # through the public streaming API: numpy ids in, numpy scores out, every step
    # staged into pinned buffers, copied H2D, replayed, copied D2H; consecutive
    # steps overlap (one step in flight ahead on a second executor)
    from paper_2509_22681_b200.orchestrator import BucketScheduler

    sched = BucketScheduler(eng, target_rows=R * C, max_slots=R, with_ids=True)
    e2e_steps = e2e_step_count(args, step_ms)
    for _ in sched.score_stream([reqs] * 2, ids=True):
        pass
    torch.cuda.synchronize()
    gc.collect()
    dist.barrier()
    t0 = time.perf_counter()
    req_lat = []
    for _ in sched.score_stream([reqs] * e2e_steps, ids=True):
        req_lat += sched.last_latencies
    e2e_s = dist.max(time.perf_counter() - t0)
    e2e_value = R * C * e2e_steps * dist.world_size / e2e_s
    # per-request latency end to end: from the submission of the request's batch
    # (numpy ids on the host) to its scores back on the host, in the streaming
    # (throughput) mode, i.e. including the wait behind the batch in flight ahead
    e2e_p99 = dist.max(1000 * nearest_rank(req_lat, 0.99))
    e2e_p50 = dist.max(1000 * nearest_rank(req_lat, 0.5))
    h2d = R * (nb * (H // nb) + C) * 8 + 3 * R * 4
    d2h = R * C * tasks * 4

    from paper_2509_22681_b200.flops import algorithmic_flops

    step_flops = algorithmic_flops(cfg, H, C) * R
    step_tf = step_flops / (sum(step_ms) / args.steps / 1e3) / 1e12

    # ------------------------------------------ fp32 verification mode
    fp32 = None if args.no_fp32_line else fp32_verify_line(eng, params, cfg, reqs, R, C, dev, step_flops)

    # ------------------------------------------------------ CPU baseline
    cpu_baseline = cpu_baseline_line(args, dist, name)

    emit_line(args, dist, name, desc, R, C, H, nb, d, L, f, value, total_ms, p99, step_tf, e2e_value, e2e_steps,
              h2d, d2h, launches, tensor, top, achieved, peak, traffic, peak_src, per_launch, avg_ms, kernels, clk,
              cpu_baseline, prof_clk=prof_clk, pda=pda, e2e_lat=(e2e_p50, e2e_p99), fp32=fp32, hot=hot)


def run_dso(args, dist) -> None:
    """cfg4: non-uniform candidate counts through the DSO (BucketScheduler).

    A step is one batch of R requests with C_i = 16 + Zipf rank (16..2048),
    H = 1024.  The scheduler buckets them by (history, candidate) powers of
    two into groups of up to slots_for(c_bkt) requests, one CUDA-graph replay
    per group, each bucket's executors on their own streams.
    * value: every group pre-staged in its own executor (ids resident in HBM);
      a step replays all groups concurrently on their streams (fork/join
      events on the step stream); real candidates / device time.
    * e2e:   BucketScheduler.score(ids=True) from numpy ids to numpy scores per
      step (pinned staging, async submit/collect across a ring of executors
      per bucket); p99 = per-request time from the call to its group's
      collection, nearest rank over all steps, max over ranks.
    """
    import torch

    import paper_2509_22681_b200 as fb
    from paper_2509_22681_b200 import _lib
    from paper_2509_22681_b200.flops import algorithmic_flops
    from paper_2509_22681_b200.orchestrator import BucketScheduler
    from paper_2509_22681_b200.pda import build_item_table

    name = args.workload
    d, dh, nb, L, f, tasks, H, C, R_default, desc = WORKLOADS[name]
    R = args.requests or R_default
    dev = torch.device("cuda", dist.device_index)
    torch.cuda.set_device(dev)
    cfg = model_config(name)
    eng = fb.FlameEngine(fb.init_params(cfg), cfg, precision="bf16", device=dist.device_index)
    eng.set_table(build_item_table(NUM_ITEMS, d, STORE_SEED), dtype="fp32")
    reqs = make_requests(R, H, C, WORKLOAD_SEED + dist.rank, zipf_c=True)
    counts = [len(c) for _, c in reqs]
    n_cand = sum(counts)
    sched = BucketScheduler(eng, with_ids=True)
    plan = sched.plan([(len(h), len(c)) for h, c in reqs])
    bucket_rows = sum(len(idx) * cb for (hb, cb), idx in plan)  # unused slots are skipped on the device
    # device-timed: one dedicated executor per group, ids staged once
    groups = []
    for (hb, cb), idx in plan:
        ex = eng.executor(sched.slots_for(cb), hb, cb, with_ids=True)
        ex.stage_ids([reqs[i] for i in idx])
        ex.run(_lib.INPUT_IDS, graph=True)
        groups.append(ex)
    torch.cuda.synchronize()
    launches = sum(ex.launch_count() for ex in groups)
    # per-launch profile before the timed region (kernels timed alone, as in run_ours)
    clocks_p = ClockSampler(dev.index, period_s=0.002)
    clocks_p.start()
    clocks_p.begin()
    # each group's launch marks count its full bucket (slots x c_bkt rows); the
    # kernels skip unused slots and padded candidate rows, so scale every record to
    # the group's REAL rows: history-row kernels by active / slots, candidate-row
    # kernels by sum(C_i) / (slots x c_bkt)
    ratios = []
    for (hb, cb), idx in plan:
        slots = sched.slots_for(cb)
        ratios.append((len(idx) / slots, sum(counts[i] for i in idx) / (slots * cb)))

    def scaled(recs, rh, rc):
        out = []
        for rec in recs:
            k = rh if "hist" in rec["name"] else rc
            out.append({**rec, "flops": rec["flops"] * k, "bytes": rec["bytes"] * k})
        return out

    prof = [[rec for ex, (rh, rc) in zip(groups, ratios) for rec in scaled(ex.profile(_lib.INPUT_IDS), rh, rc)]
            for _ in range(2)]
    prof_clk = clocks_p.stop()
    main = torch.cuda.Stream(device=dev)

    def step(ev_start, ev_end):
        with torch.cuda.stream(main):
            ev_start.record(main)
        joins = []
        for ex in groups:
            ex.stream.wait_event(ev_start)
            ex.run(_lib.INPUT_IDS, graph=True)
            j = torch.cuda.Event()
            j.record(ex.stream)
            joins.append(j)
        for j in joins:
            main.wait_event(j)
        with torch.cuda.stream(main):
            ev_end.record(main)

    for _ in range(args.warmup):
        step(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    torch.cuda.synchronize()
    dist.barrier()
    clocks = ClockSampler(dev.index)
    clocks.start()
    time.sleep(0.3)
    clocks.begin()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for a, b in evs:
        step(a, b)
    torch.cuda.synchronize()
    clk = clocks.stop()
    dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = dist.max(sum(step_ms))
    value = n_cand * args.steps * dist.world_size / (total_ms / 1e3)

    pdas = [pda_algorithmic_bytes(ex, d, 4) for ex in groups]
    pda = {k: sum(p[k] for p in pdas) for k in pdas[0]}
    tensor, top, achieved, peak, traffic, peak_src, per_launch, avg_ms, kernels = roofline(
        prof, name, prof_clk, {k: pda[k] / len(groups) for k in ("pda_dedup", "pda_gather")})

    # e2e through the scheduler's streaming API (async submit / collect over the
    # executor rings; the next batch is staged while the previous one runs)
    e2e_steps = e2e_step_count(args, step_ms)
    sched.executors_per_bucket = 3
    for _ in sched.score_stream([reqs] * 2, ids=True):
        pass
    torch.cuda.synchronize()
    gc.collect()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in sched.score_stream([reqs] * e2e_steps, ids=True):
        pass
    e2e_s = dist.max(time.perf_counter() - t0)
    # request latency in the latency-optimised mode: one batch at a time (no queueing
    # behind a previous batch), call -> the request's group collected on the host
    lats = []
    for _ in range(e2e_steps):
        sched.score(reqs, ids=True)
        lats += sched.last_latencies
    e2e_value = n_cand * e2e_steps * dist.world_size / e2e_s
    p99 = dist.max(1000 * nearest_rank(lats, 0.99))
    h2d = sum(len(h) + len(c) for h, c in reqs) * 8 + 3 * 4 * len(plan)
    d2h = n_cand * tasks * 4

    step_flops = sum(algorithmic_flops(cfg, H, c) for c in counts)
    step_tf = step_flops / (sum(step_ms) / args.steps / 1e3) / 1e12
    cpu_baseline = cpu_baseline_line(args, dist, name)
    hist = {}
    for (hb, cb), idx in plan:
        hist[str(cb)] = hist.get(str(cb), 0) + len(idx)
    step_p99 = dist.max(nearest_rank(step_ms, 0.99))
    emit_line(args, dist, name, desc, R, C, H, nb, d, L, f, value, total_ms, p99, step_tf,
              e2e_value, e2e_steps, h2d, d2h, launches, tensor, top, achieved, peak, traffic, peak_src, per_launch,
              avg_ms, kernels, clk, cpu_baseline, prof_clk=prof_clk, pda=pda,
              extra_config={"candidates_per_request": "16 + Zipf(1.0) rank over 2033 (16..2048)",
                            "candidates_per_step_per_gpu": n_cand, "groups_per_step": len(plan),
                            "step_p99_ms": step_p99,
                            "requests_per_bucket": hist, "padding_efficiency": round(n_cand / bucket_rows, 4),
                            "dso": "BucketScheduler: pow2 (history, candidate) buckets, one graph replay per group, "
                                   "one stream per executor, groups concurrent"},
              e2e_path="BucketScheduler.score_stream(ids=True): numpy ids -> pinned -> H2D -> graph per group -> D2H "
                       "-> numpy, next batch staged while the previous runs",
              latency_note="p99_ms: per-request latency through BucketScheduler.score (one batch at a time: "
                           "call -> its group's scores on the host), nearest rank over e2e steps, max over ranks; "
                           "device step p99 in step_p99_ms")


def e2e_step_count(args, step_ms) -> int:
    """Batches in the e2e region: about 0.3 s of device work (at least --steps,
    at most 400), so one host hiccup (a GC pass, a page fault) cannot swing it."""
    per = max(1e-3, sum(step_ms) / len(step_ms)) / 1e3
    return int(min(400, max(args.steps, 3, round(0.3 / per))))


def emit_line(args, dist, name, desc, R, C, H, nb, d, L, f, value, total_ms, p99, step_tf, e2e_value, e2e_steps,
              h2d, d2h, launches, tensor, top, achieved, peak, traffic, peak_src, per_launch, avg_ms, kernels, clk,
              cpu_baseline, extra_config=None, e2e_path=None, latency_note=None, prof_clk=None, pda=None, e2e_lat=None,
              fp32=None, hot=None):
    if dist.rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "candidates/s", "n_gpus": dist.world_size,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic: Zipf(1.0) item ids over 100k items (reference _KeySampler), "
                    "store embeddings item_embedding(seed 1234), random-init weights init_params(seed 0)",
            "config": {"workload": name, "desc": desc, "requests_per_step_per_gpu": R,
                       "candidates_per_request": C, "history_len": H, "num_blocks": nb,
                       "hidden_dim": d, "layers_per_block": L, "ffn_dim": f,
                       "parallelism": f"request-sharded dp{dist.world_size}, no collective",
                       "l2": "per-step working set (activations, several GB) >> 126 MB L2; no flush",
                       "input": "item ids resident in HBM; PDA gather from the fp32 HBM item table"},
            "p99_ms": p99,
            "latency_note": latency_note or ("a request completes when its step's graph replay completes; "
                                             "p99 over steps (nearest rank), max over ranks"),
            "step_tflops": round(step_tf, 1),
            "e2e": {"value": e2e_value, "unit": "candidates/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": e2e_steps,
                    **({"request_p50_ms": e2e_lat[0], "request_p99_ms": e2e_lat[1],
                        "latency": "per request: submission of its batch (numpy ids) -> its scores on the host, "
                                   "streaming mode (one batch in flight ahead), nearest rank, max over ranks"}
                       if e2e_lat else {}),
                    "timing": "host wall clock over ~0.3 s of device work (sustained, power-capped rate)",
                    "path": e2e_path or ("BucketScheduler.score_stream(ids=True): numpy ids -> pinned -> H2D -> "
                                         "graph -> D2H -> numpy, one step in flight ahead")},
            "gpu_launches": launches * args.steps,
            "launches_per_step": launches,
            "roofline": {"bound": "tensor" if tensor else "hbm", "kernel": top,
                         "achieved": round(achieved, 1), "peak": peak,
                         "unit": "TFLOP/s" if tensor else "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": traffic,
                         "peak_source": peak_src,
                         "per_launch": per_launch, "avg_launch_ms": avg_ms,
                         "timing": "per-launch CUDA events on the executor stream, eager pass enqueued behind "
                                   "a gate kernel (launches back to back), median of 5, run before the timed "
                                   "region (kernels timed alone)",
                         **({"hot": hot} if hot else {}),
                         "profile_clocks": prof_clk,
                         "traffic_source": "profiles/ncu_dram_per_launch.json (ncu --set full of tools/prof_step.py: "
                                           "the bench's own workload, 100k-item fp32 table)"},
            "pda": pda and {"unique_rows_per_step": pda["unique_rows"], "positions_per_step": pda["positions"],
                            "bytes": "SURVEY 8(d): one table row per unique id; dedup = ids in + unique + inverse out"},
            "kernels": kernels,
            "clocks": clk,
            "cpu_baseline": cpu_baseline,
        }
        if fp32:
            line["fp32_verify"] = fp32
        if extra_config:
            line["config"].update(extra_config)
        print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="cfg3", choices=sorted(WORKLOADS))
    ap.add_argument("--requests", type=int, default=0, help="requests per step per GPU (0 = default)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-fp32-line", action="store_true", help="skip the fp32 verification-mode line")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU without an external launcher: re-run this command
        # under torch.distributed.run (rendezvous on 127.0.0.1)
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(args.gpus),
               "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()),
               *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    from paper_2509_22681_b200.sharding import Dist

    dist = Dist(backend="gloo" if args.impl == "reference" else None)
    try:
        if args.impl == "reference":
            run_reference(args, dist)
        elif args.workload in ZIPF_C:
            run_dso(args, dist)
        else:
            run_ours(args, dist)
    finally:
        dist.close()


if __name__ == "__main__":
    main()
