"""Served-stream throughput and per-request latency through the process-per-GPU
dispatcher (paper_2509_22681_b200.dispatch.MultiDeviceService).

One request stream (bench.make_requests: Zipf ids over the 100k-item table) is
routed over N GPU workers, least outstanding work first, with at most
``--window`` requests in flight, submitted in frames of ``--frame`` requests
(``submit_many``: one message per worker per frame).  Per-request latency runs from submit (numpy
ids in the caller's process) to the scores back in it: IPC to the worker,
coalescing, staging, H2D, the graph replay, D2H, IPC back.

    python tools/serve_bench.py --workload cfg3 --gpus 1 --requests 2000 --window 256
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from collections import deque
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2509_22681_b200.dispatch import MultiDeviceService  # noqa: E402
from paper_2509_22681_b200.service import ServiceConfig  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg3")
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--requests", type=int, default=2000)
    ap.add_argument("--window", type=int, default=256)
    ap.add_argument("--warmup", type=int, default=300)
    ap.add_argument("--frame", type=int, default=16, help="requests per submit_many call (one message per worker)")
    ap.add_argument("--workers-per-gpu", type=int, default=1,
                    help="worker processes per GPU (the host side of a worker is the limit of one)")
    a = ap.parse_args()
    d, dh, nb, L, f, tasks, H, C, *_ = bench.WORKLOADS[a.workload]
    cfg = ServiceConfig(model=bench.model_config(a.workload), num_items=bench.NUM_ITEMS,
                        store_seed=bench.STORE_SEED, target_rows=64 * 512, max_batch=64)
    reqs = bench.make_requests(a.requests + a.warmup, H, C, bench.WORKLOAD_SEED, a.workload in bench.ZIPF_C)
    t_start = time.perf_counter()
    devices = [g for g in range(a.gpus) for _ in range(a.workers_per_gpu)]
    with MultiDeviceService(cfg, n_devices=len(devices), devices=devices) as svc:
        startup = time.perf_counter() - t_start
        for fut in svc.submit_many(reqs[: a.warmup]):
            fut.result()
        inflight: deque = deque()
        lat = []
        cands = 0
        t0 = time.perf_counter()
        body = reqs[a.warmup:]
        for f0 in range(0, len(body), a.frame):
            while len(inflight) >= a.window:
                s, _, e2e = inflight.popleft().result()
                lat.append(e2e)
                cands += s.shape[0]
            inflight.extend(svc.submit_many(body[f0:f0 + a.frame]))
        while inflight:
            s, _, e2e = inflight.popleft().result()
            lat.append(e2e)
            cands += s.shape[0]
        wall = time.perf_counter() - t0
        routed = list(svc.routed)
    lat.sort()
    line = {"metric": "served candidates/s through the process-per-GPU dispatcher", "workload": a.workload,
            "n_gpus": a.gpus, "workers_per_gpu": a.workers_per_gpu, "requests": a.requests, "window": a.window, "frame": a.frame, "value": cands / wall,
            "unit": "candidates/s", "wall_s": wall, "startup_s": startup,
            "p50_ms": 1000 * bench.nearest_rank(lat, 0.5), "p99_ms": 1000 * bench.nearest_rank(lat, 0.99),
            "routed_per_worker": routed,
            "latency": "submit (numpy ids, caller process) -> scores back in the caller, per request"}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
