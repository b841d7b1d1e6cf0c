"""Drop-in ``model_forward`` — mirror of the reference operator API
(pkg/src/flameserve/model/forward.py:186-204 and its input checks :169-183).

Same signature, same argument meaning, same ``ValueError`` behaviour; the
computation runs on the B200 through the C ABI.  ``attn_impl`` keeps its
reference meaning as an operator selector and is validated against the same
set (forward.py:31); every choice is served by the fused SUMI kernel, which
computes the identical masked softmax (the reference's three implementations
agree to 1e-10, tests/test_forward.py:138-147).  ``precision`` selects the
bf16 tcgen05 path (default) or the fp32 verification path.
"""

from __future__ import annotations

import threading
import weakref

import numpy as np

from .config import ModelConfig
from .engine import FlameEngine
from .params import ModelParams, iter_param_arrays, param_stream

ATTN_IMPLS = ("fused", "tiled", "naive")
DEFAULT_TILE = 128
DEFAULT_PRECISION = "bf16"

# engines per params object (keyed by identity: ModelParams is an unhashable
# dataclass); an entry is dropped when its params object is garbage collected
_engines: dict[int, dict] = {}
_engines_lock = threading.Lock()


def _drop_engines(key: int) -> None:
    with _engines_lock:
        per = _engines.pop(key, None)
    for eng in (per or {}).values():
        eng.close()


def split_sequence(history: np.ndarray, num_blocks: int, mode: str = "contiguous") -> list[np.ndarray]:
    """Reference forward.py:50-62 (host-side helper; the device path applies
    the same contiguous split inside the gather/scatter kernels)."""
    if num_blocks < 1:
        raise ValueError("num_blocks must be >= 1")
    if mode == "interleaved":
        raise NotImplementedError("interleaved split is reserved, only contiguous is implemented")
    if mode != "contiguous":
        raise ValueError(f"unknown split mode {mode!r}")
    length = history.shape[0]
    if length % num_blocks != 0:
        raise ValueError(f"history length {length} is not divisible by num_blocks {num_blocks}")
    step = length // num_blocks
    return [history[b * step:(b + 1) * step] for b in range(num_blocks)]


def check_forward_inputs(history: np.ndarray, candidates: np.ndarray, config: ModelConfig) -> None:
    """Reference forward.py:169-183 plus the split divisibility of :59-60."""
    if history.ndim != 2 or history.shape[1] != config.hidden_dim:
        raise ValueError(f"history must be (length, {config.hidden_dim})")
    if candidates.ndim != 2 or candidates.shape[1] != config.hidden_dim:
        raise ValueError(f"candidates must be (count, {config.hidden_dim})")
    if history.shape[0] > config.max_history_len:
        raise ValueError(f"history length {history.shape[0]} exceeds max {config.max_history_len}")
    if not 1 <= candidates.shape[0] <= config.max_candidates:
        raise ValueError(
            f"candidate count {candidates.shape[0]} outside [1, {config.max_candidates}]")
    if history.shape[0] % config.num_blocks != 0:
        raise ValueError(
            f"history length {history.shape[0]} is not divisible by num_blocks {config.num_blocks}")


def _fingerprint(params: ModelParams):
    """Content key for small models so in-place edits of a params object are
    picked up; large models are keyed by identity (the reference treats params
    as immutable)."""
    total = sum(a.size for _, a in iter_param_arrays(params))
    if total > (1 << 22):
        return None
    return hash(param_stream(params).tobytes())


def get_engine(params: ModelParams, config: ModelConfig, precision: str = DEFAULT_PRECISION,
               device=None) -> FlameEngine:
    """Device context for (params, precision, device), built once per params object."""
    with _engines_lock:
        per = _engines.get(id(params))
        if per is None:
            per = _engines[id(params)] = {}
            weakref.finalize(params, _drop_engines, id(params))
        key = (config, precision, device, _fingerprint(params))
        eng = per.get(key)
        if eng is None:
            eng = FlameEngine(params, config, precision=precision, device=device)
            per[key] = eng
        return eng


def find_engine(params: ModelParams, precision: str = DEFAULT_PRECISION, device=None):
    """An engine already built for ``params`` (any config), or None."""
    with _engines_lock:
        for (_, prec, dev, fp), eng in (_engines.get(id(params)) or {}).items():
            if prec == precision and dev == device and fp == _fingerprint(params):
                return eng
    return None


def model_forward(
    history: np.ndarray,
    candidates: np.ndarray,
    params: ModelParams,
    config: ModelConfig,
    attn_impl: str = "fused",
    tile: int = DEFAULT_TILE,
    *,
    precision: str = DEFAULT_PRECISION,
    device=None,
) -> np.ndarray:
    """Score all candidates against the history in one pass -> (C, num_tasks)."""
    if attn_impl not in ATTN_IMPLS:
        raise ValueError(f"attn_impl must be one of {ATTN_IMPLS}, got {attn_impl!r}")
    history = np.asarray(history)
    candidates = np.asarray(candidates)
    check_forward_inputs(history, candidates, config)
    for block in params.blocks:
        if block.temperature <= 0:
            raise ValueError("block temperature must be positive")
    eng = get_engine(params, config, precision, device)
    hb_bkt, c_bkt = eng.bucket(history.shape[0], candidates.shape[0])
    ex = eng.executor(1, hb_bkt, c_bkt)
    return ex.score([(history, candidates)])[0]


def model_forward_batch(requests, params: ModelParams, config: ModelConfig, *,
                        precision: str = DEFAULT_PRECISION, device=None) -> list[np.ndarray]:
    """Score many (history, candidates) requests in one device pass (one CUDA
    graph over a request bucket).  Results equal per-request ``model_forward``
    bit for bit: every kernel reduces each row in a fixed order."""
    reqs = [(np.asarray(h), np.asarray(c)) for h, c in requests]
    for h, c in reqs:
        check_forward_inputs(h, c, config)
    eng = get_engine(params, config, precision, device)
    hb = max(eng.bucket(h.shape[0], c.shape[0])[0] for h, c in reqs)
    cb = max(eng.bucket(h.shape[0], c.shape[0])[1] for h, c in reqs)
    ex = eng.executor(len(reqs), hb, cb)
    return ex.score(reqs)
