"""Proximal Data Accelerator (PDA) — device-resident feature assembly.

Replaces the per-id Python loop of ``Service.resolve_embeddings``
(pkg/src/flameserve/service.py:97-108) with the ``pda_dedup`` + ``pda_gather``
kernels: ids -> (np.unique values, inverse map) bit-exact, and the embedding
rows assembled straight into the row space the projection GEMMs read.

The dense item table is the reference store's deterministic embedding
function evaluated for every id of the universe: ``item_embedding`` restates
store.py:59-63 (splitmix64 mixing of cache.py:43-48 / FeatureKey.stable_hash
cache.py:60,75 -> numpy ``default_rng(mix).uniform(-1, 1, dim)``), so a
device row equals the value the reference store would serve for that id
(version 0).  Ids outside the table decode to zero rows, as empty store
values do (store.py:74-78).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .engine import FlameEngine

_MASK64 = 0xFFFFFFFFFFFFFFFF
_ITEM_SALT = 0xC2B2AE3D27D4EB4F
DEFAULT_STORE_SEED = 1234  # store.py:30


def _splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & _MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _MASK64
    return x ^ (x >> 31)


def item_embedding(store_seed: int, item_id: int, version: int, dim: int) -> np.ndarray:
    key_hash = _splitmix64((int(item_id) ^ _ITEM_SALT) & _MASK64)
    mix = _splitmix64(store_seed ^ _splitmix64(key_hash ^ _splitmix64(version)))
    return np.random.default_rng(mix).uniform(-1.0, 1.0, dim)


def build_item_table(num_items: int, dim: int, store_seed: int = DEFAULT_STORE_SEED,
                     dtype=np.float32) -> np.ndarray:
    """(num_items, dim) table, row i = the store's embedding of ITEM id i."""
    table = np.empty((num_items, dim), dtype=dtype)
    for i in range(num_items):
        table[i] = item_embedding(store_seed, i, 0, dim)
    return table


class DeviceFeatureAssembler:
    """``resolve_embeddings`` on the device for one id list at a time."""

    def __init__(self, engine: FlameEngine, max_ids: int = 8192) -> None:
        if engine.num_items == 0:
            raise ValueError("engine has no embedding table (FlameEngine.set_table)")
        self.engine = engine
        self.max_ids = max_ids
        self._ex = engine.executor(1, 0, max_ids, with_ids=True, cache=False)

    def resolve(self, item_ids) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """ids (n,) -> (rows (n, d) fp32, unique (U,) int64, inverse (n,) int64)."""
        ids = np.asarray(item_ids, dtype=np.int64).ravel()
        n = ids.size
        d = self.engine.config.hidden_dim
        if n == 0:
            return np.zeros((0, d), np.float32), np.zeros(0, np.int64), np.zeros(0, np.int64)
        if n > self.max_ids:
            raise ValueError(f"{n} ids exceed the assembler capacity {self.max_ids}")
        ex = self._ex
        with ex.lock:
            ex.stage_ids([(np.zeros(0, np.int64), ids)])
            ex.run(_lib.INPUT_GATHER_ONLY, graph=False)
            ex.stream.synchronize()
            nu = int(ex.n_unique[1].item())  # list R + 0 = candidate list of request 0
            unique = ex.unique[1, :nu].cpu().numpy()
            inverse = ex.inverse[1, :n].cpu().numpy()
            D = ((d + 63) // 64) * 64
            rows = ex.read_workspace("Ec", (ex.c_bkt, D))[:n, :d]
        return rows, unique, inverse
