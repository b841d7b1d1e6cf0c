"""Generate tests/golden/*.npz by running the REFERENCE implementation itself.

Test infrastructure only.  Run in the build container (where the read-only
reference lives at /root/reference):

    python oracle/gen_golden.py

The fixtures pin (a) the oracle restatement in oracle/flame_oracle.py and
(b) the device path, to the reference's own outputs:

* params_*      sha256 of reference ``params_to_bytes(init_params(cfg))`` and a
                small FLMP file image written by reference ``save_params``
* forward_*     reference ``model_forward`` (fp64, attn_impl="fused") outputs;
                small cases also carry the inputs and the sequential-oracle
                output (``model_forward_sequential``), large cases carry the
                input seed (numpy PCG64 ``uniform(-1, 1)`` draws, stable by
                numpy's stream-compatibility policy)
* pda_*         reference ``Service.resolve_embeddings`` rows for Zipf ids
                drawn with the reference ``_KeySampler``, plus the np.unique
                maps it computes, and reference ``item_embedding`` values
"""

from __future__ import annotations

import hashlib
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"

FORWARD_CASES = [
    # name, (d, dh, Nb, L, f, tasks, maxH, maxC, seed), H, C, store_inputs
    ("cfg1", (64, 16, 2, 1, 256, 2, 256, 64, 0), 256, 64, True),
    ("ref_instance", (16, 4, 2, 2, 24, 3, 64, 32, 13), 32, 5, True),
    ("sample_json", (16, 8, 2, 1, 32, 2, 1024, 2048, 7), 64, 20, True),
    ("l2_wide", (64, 16, 2, 2, 128, 2, 512, 300, 3), 256, 40, True),
    ("nohist", (32, 8, 2, 1, 64, 2, 64, 16, 5), 0, 9, True),
    ("l3_nb4", (32, 8, 4, 3, 96, 3, 128, 64, 9), 64, 33, True),
    ("cfg2", (256, 64, 4, 1, 1024, 2, 1024, 256, 0), 1024, 256, False),
    ("cfg3", (512, 64, 8, 1, 2048, 2, 2048, 512, 0), 2048, 512, False),
    ("long_hist_l2", (128, 64, 2, 2, 256, 2, 1200, 700, 12), 1200, 700, False),
    ("cfg5", (768, 64, 12, 1, 3072, 2, 8184, 1024, 0), 8184, 1024, False),
]


def _inputs(seed: int, H: int, C: int, d: int):
    rng = np.random.default_rng(seed)
    return rng.uniform(-1.0, 1.0, (H, d)), rng.uniform(-1.0, 1.0, (C, d))


def main() -> None:
    sys.path.insert(0, str(REF))
    from flameserve.bench import KeyDistribution, _KeySampler
    from flameserve.cache import CacheConfig, CacheMode, FeatureKey, KeyKind
    from flameserve.config import OrchestratorConfig, ServiceConfig
    from flameserve.model import (ModelConfig, init_params, model_forward,
                                  model_forward_sequential, params_to_bytes, save_params)
    from flameserve.service import Service
    from flameserve.store import RemoteStoreConfig, item_embedding

    OUT.mkdir(parents=True, exist_ok=True)
    meta = {"numpy": np.__version__, "reference": str(REF)}

    # ---------------------------------------------------------------- params
    shas = {}
    for name, dims, *_ in FORWARD_CASES:
        cfg = ModelConfig(*dims[:8], seed=dims[8])
        shas[name] = hashlib.sha256(params_to_bytes(init_params(cfg), cfg)).hexdigest()
    tiny = ModelConfig(16, 4, 2, 2, 24, 3, 64, 32, seed=(1 << 40) + 17)
    with tempfile.TemporaryDirectory() as tmp:
        path = Path(tmp) / "tiny.flmp"
        save_params(init_params(tiny), tiny, path)
        flmp = np.frombuffer(path.read_bytes(), dtype=np.uint8)
    np.savez_compressed(OUT / "params.npz", flmp_tiny=flmp,
                        sha_names=np.array(list(shas)), sha_values=np.array(list(shas.values())))

    # --------------------------------------------------------------- forward
    for i, (name, dims, H, C, store) in enumerate(FORWARD_CASES):
        cfg = ModelConfig(*dims[:8], seed=dims[8])
        params = init_params(cfg)
        seed = 1000 + i
        hist, cand = _inputs(seed, H, C, cfg.hidden_dim)
        out = model_forward(hist, cand, params, cfg)
        blob = {"dims": np.array(dims, dtype=np.int64), "H": H, "C": C, "input_seed": seed,
                "scores": out}
        if store:
            blob["history"] = hist
            blob["candidates"] = cand
            blob["sequential"] = model_forward_sequential(hist, cand, params, cfg)
        np.savez_compressed(OUT / f"forward_{name}.npz", **blob)
        print(f"forward_{name}: scores {out.shape} range [{out.min():.3f}, {out.max():.3f}]")

    # ------------------------------------------------------------------- PDA
    d = 16
    svc_cfg = ServiceConfig(
        model=ModelConfig(d, 4, 2, 1, 32, 2, 512, 512, seed=3),
        cache=CacheConfig(bucket_count=16, capacity_per_bucket=4096, ttl_s=600.0, mode=CacheMode.SYNC),
        remote_store=RemoteStoreConfig(latency_ms_mean=0.0, latency_ms_p99=0.0,
                                       bytes_per_value=d * 8, seed=1234),
        orchestrator=OrchestratorConfig(profile_shapes=(128,), executors_per_shape=1),
    )
    svc = Service(svc_cfg)
    try:
        rng = np.random.default_rng(2509)
        sampler = _KeySampler(KeyDistribution("zipf", 1.0), 500)
        lists = {"hist": sampler.sample(rng, 256), "cand": sampler.sample(rng, 37),
                 "single": np.array([42], dtype=np.int64),
                 "dups": np.array([7, 7, 7, 3, 3, 499, 0, 7], dtype=np.int64)}
        blob = {}
        for key, ids in lists.items():
            rows = svc.resolve_embeddings(ids)
            uq, inv = np.unique(ids, return_inverse=True)
            blob[f"{key}_ids"] = ids
            blob[f"{key}_rows"] = rows
            blob[f"{key}_unique"] = uq
            blob[f"{key}_inverse"] = inv.astype(np.int64)
    finally:
        svc.close()
    emb_ids = np.array([0, 1, 2, 17, 499, 99_999, 123_456], dtype=np.int64)
    blob["emb_ids"] = emb_ids
    blob["emb_values"] = np.stack([item_embedding(1234, FeatureKey(KeyKind.ITEM, int(k)), 0, 64)
                                   for k in emb_ids])
    np.savez_compressed(OUT / "pda.npz", **blob)
    (OUT / "META.json").write_text(json.dumps(meta, indent=1) + "\n")
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
