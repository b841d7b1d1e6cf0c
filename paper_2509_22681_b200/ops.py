"""Operator-level drop-in API — the rest of the reference's ``flameserve.model``
surface (model/__init__.py:4-31) beside ``model_forward``.

Every operator takes and returns numpy arrays like the reference's, raises the
same ``ValueError``s, and computes on the B200 through the C ABI
(``flame_op_*`` in include/flame_b200.h):

* ``attention_sumi_candidates`` / ``attention_sumi`` (attention.py:118-178) run
  the forward pass's own SUMI attention kernels (bf16 tcgen05 by default, the
  fp32 verification kernel with ``precision="fp32"``) on a one-request workspace.
* ``block_forward`` (forward.py:75-140) runs the forward pass's layer-stack
  launch sequence for one block; ``expert_heads`` (forward.py:159-166) its
  expert GEMM + combine; ``gated_fusion`` (forward.py:143-156) its gating kernel.
* ``attention_naive`` / ``attention_tiled`` (attention.py:55-115) take an
  arbitrary permission matrix, so they run a general fp64 masked-attention
  kernel; ``tile`` keeps its argument checks (it only orders the reference's
  streaming sum).  ``masked_softmax_rows``, ``gelu``, ``sigmoid`` and
  ``layer_norm`` are fp64 device kernels.

There is no host fallback: without the library or a device these raise.
"""

from __future__ import annotations

import dataclasses
import threading
import weakref

import numpy as np

from . import _lib
from .config import ModelConfig
from .forward import ATTN_IMPLS, DEFAULT_PRECISION, DEFAULT_TILE, find_engine, get_engine
from .mask import SumiMask
from .params import BlockParams, ModelParams, iter_param_arrays, param_stream

_PREC = {"bf16": _lib.FLAME_BF16, "fp32": _lib.FLAME_FP32}


def _device_index(device) -> int:
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("the FLAME B200 operators need a CUDA device; there is no CPU fallback")
    return torch.cuda.current_device() if device is None else int(device)


def _f64(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.float64)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _precision(precision: str) -> int:
    if precision not in _PREC:
        raise ValueError(f"precision must be one of {tuple(_PREC)}, got {precision!r}")
    return _PREC[precision]


# ------------------------------------------------------------------ row ops
def _rows(op: int, x, scale=None, shift=None, device=None) -> np.ndarray:
    a = _f64(x)
    out = np.empty_like(a)
    if a.size == 0:
        return out
    width = a.shape[-1] if a.ndim else 1
    rows = a.size // width
    s = t = None
    if scale is not None:
        s = _f64(np.broadcast_to(np.asarray(scale, dtype=np.float64), (width,)))
        t = _f64(np.broadcast_to(np.asarray(shift, dtype=np.float64), (width,)))
    lib = _lib.load()
    _lib.check(lib.flame_op_rows(op, _device_index(device), rows, width, _ptr(a),
                                 _ptr(s) if s is not None else None, _ptr(t) if t is not None else None, _ptr(out)))
    return out


def gelu(x: np.ndarray, *, device=None) -> np.ndarray:
    """Reference forward.py:33-35: tanh-form GELU (fp64 on the device)."""
    return _rows(_lib.OP_GELU, x, device=device)


def sigmoid(x: np.ndarray, *, device=None) -> np.ndarray:
    """Reference forward.py:38-39 (fp64 on the device)."""
    return _rows(_lib.OP_SIGMOID, x, device=device)


def layer_norm(x: np.ndarray, scale: np.ndarray, shift: np.ndarray, *, device=None) -> np.ndarray:
    """Reference forward.py:42-47: over the last axis, eps 1e-5 (fp64 on the device)."""
    return _rows(_lib.OP_LAYER_NORM, x, scale, shift, device=device)


def masked_softmax_rows(scores: np.ndarray, *, device=None) -> np.ndarray:
    """Reference attention.py:28-36: row softmax with -inf entries excluded."""
    return _rows(_lib.OP_SOFTMAX, scores, device=device)


# ---------------------------------------------------------------- attention
def _check_qkv(q: np.ndarray, k: np.ndarray, v: np.ndarray, mask: SumiMask, temperature: float) -> None:
    """Reference attention.py:48-55."""
    if q.ndim != 2 or q.shape != k.shape or q.shape != v.shape:
        raise ValueError(f"q/k/v must share one (T, head_dim) shape, got {q.shape}, {k.shape}, {v.shape}")
    if q.shape[0] != mask.size:
        raise ValueError(f"sequence length {q.shape[0]} does not match mask size {mask.size}")
    if temperature <= 0:
        raise ValueError("temperature must be positive")


def _masked_attention(q, k, v, mask: SumiMask, temperature: float, device) -> np.ndarray:
    q, k, v = _f64(q), _f64(k), _f64(v)
    t, dh = q.shape
    allowed = np.ascontiguousarray(mask.allowed, dtype=np.uint8)
    if allowed.shape != (t, t):
        raise ValueError(f"mask must be ({t}, {t}), got {allowed.shape}")
    out = np.empty_like(q)
    _lib.check(_lib.load().flame_op_attention_masked(_device_index(device), t, dh, float(temperature), _ptr(q),
                                                     _ptr(k), _ptr(v), _ptr(allowed), _ptr(out)))
    return out


def attention_naive(q: np.ndarray, k: np.ndarray, v: np.ndarray, mask: SumiMask, temperature: float, *,
                    device=None) -> np.ndarray:
    """Reference attention.py:55-67 over any permission matrix (fp64 on the device)."""
    _check_qkv(q, k, v, mask, temperature)
    if q.shape[0] == 0:
        return np.zeros_like(q)
    return _masked_attention(q, k, v, mask, temperature, device)


def attention_tiled(q: np.ndarray, k: np.ndarray, v: np.ndarray, mask: SumiMask, temperature: float, tile: int,
                    *, device=None) -> np.ndarray:
    """Reference attention.py:70-115: same result as ``attention_naive``; ``tile``
    is validated as the reference does."""
    _check_qkv(q, k, v, mask, temperature)
    t = q.shape[0]
    if t == 0:
        return np.zeros_like(q)
    if not 1 <= tile <= t:
        raise ValueError(f"tile must be in [1, {t}], got {tile}")
    return _masked_attention(q, k, v, mask, temperature, device)


def _sumi(q, kh, vh, hist_len: int, temperature: float, candidates_only: bool, precision: str,
          device) -> np.ndarray:
    prec = _precision(precision)
    q, kh, vh = _f64(q), _f64(kh), _f64(vh)
    if kh.ndim != 3 or vh.shape != kh.shape or q.ndim != 3:
        raise ValueError("q / k / v must be (num_heads, length, head_dim)")
    nh, t, dh = kh.shape
    out = np.empty_like(q)
    if out.size == 0:
        return out
    _lib.check(_lib.load().flame_op_attention_sumi(prec, _device_index(device), nh, t, dh, int(hist_len),
                                                   1 if candidates_only else 0, float(temperature), _ptr(q),
                                                   _ptr(kh), _ptr(vh), _ptr(out)))
    return out


def attention_sumi_candidates(qc: np.ndarray, kh: np.ndarray, vh: np.ndarray, hist_len: int, temperature: float,
                              *, precision: str = DEFAULT_PRECISION, device=None) -> np.ndarray:
    """Reference attention.py:118-146: candidate rows only, each over the shared
    history K/V plus itself.  ``qc`` (num_heads, C, head_dim); ``kh`` / ``vh``
    (num_heads, hist_len + C, head_dim)."""
    if temperature <= 0:
        raise ValueError("temperature must be positive")
    qc = np.asarray(qc)
    if np.asarray(kh).shape[1] != hist_len + qc.shape[1]:
        raise ValueError(f"k/v length {np.asarray(kh).shape[1]} != hist_len {hist_len} + {qc.shape[1]} candidates")
    return _sumi(qc, kh, vh, hist_len, temperature, True, precision, device)


def attention_sumi(qh: np.ndarray, kh: np.ndarray, vh: np.ndarray, hist_len: int, temperature: float, *,
                   precision: str = DEFAULT_PRECISION, device=None) -> np.ndarray:
    """Reference attention.py:149-178: causal history rows + SUMI candidate rows,
    all heads at once; (num_heads, T, head_dim) in and out."""
    t = np.asarray(qh).shape[1]
    if not 0 <= hist_len <= t:
        raise ValueError(f"hist_len {hist_len} out of range for sequence length {t}")
    if temperature <= 0:
        raise ValueError("temperature must be positive")
    if np.asarray(qh).shape != np.asarray(kh).shape:
        raise ValueError("q / k / v must share one (num_heads, T, head_dim) shape")
    return _sumi(qh, kh, vh, hist_len, temperature, False, precision, device)


# ------------------------------------------------------- block / fusion / experts
def gated_fusion(block_outputs: list, params: ModelParams, *, device=None) -> np.ndarray:
    """Reference forward.py:143-156 (the forward pass's fp32 gating kernel)."""
    if len(block_outputs) != len(params.blocks):
        raise ValueError(f"expected {len(params.blocks)} block outputs, got {len(block_outputs)}")
    shape = np.asarray(block_outputs[0]).shape
    for out in block_outputs[1:]:
        if np.asarray(out).shape != shape:
            raise ValueError("block outputs must share one shape")
    if len(shape) != 2:
        raise ValueError("block outputs must be (C, hidden_dim)")
    rows, width = shape
    x = _f64(np.stack([np.asarray(o) for o in block_outputs]))
    gw = _f64(np.stack([np.broadcast_to(b.gate_weight, (width,)) for b in params.blocks]))
    gb = _f64(np.stack([np.broadcast_to(b.gate_bias, (width,)) for b in params.blocks]))
    out = np.empty((rows, width))
    if rows == 0:
        return out
    _lib.check(_lib.load().flame_op_gated_fusion(_device_index(device), len(params.blocks), rows, width, _ptr(x),
                                                 _ptr(gw), _ptr(gb), _ptr(out)))
    return out


def _head_dim_for(d: int) -> int:
    return max(h for h in range(1, min(d, 64) + 1) if d % h == 0)


def _expert_config(params: ModelParams) -> ModelConfig:
    d, f = params.expert_w1.shape
    layers = len(params.blocks[0].layers) if params.blocks else 1
    nb = max(len(params.blocks), 1)
    return ModelConfig(d, _head_dim_for(d), nb, layers, f, params.expert_w2.shape[1], nb, 1)


def expert_heads(fused: np.ndarray, params: ModelParams, *, precision: str = DEFAULT_PRECISION,
                 device=None) -> np.ndarray:
    """Reference forward.py:159-166: (C, d) fused rows -> (C, num_tasks) scores,
    through the forward pass's expert GEMM (tf32 in bf16 mode) + combine."""
    _precision(precision)
    fused = np.asarray(fused)
    if fused.ndim != 2 or fused.shape[1] != params.expert_w1.shape[0]:
        raise ValueError(f"fused states must be (C, {params.expert_w1.shape[0]}), got {fused.shape}")
    tasks = params.expert_w2.shape[1]
    out = np.empty((fused.shape[0], tasks))
    if fused.shape[0] == 0:
        return out
    eng = find_engine(params, precision, device) or get_engine(params, _expert_config(params), precision, device)
    f = _f64(fused)
    with _device_ctx(eng):
        _lib.check(eng.lib.flame_op_expert_heads(eng.handle, _ptr(f), f.shape[0], _ptr(out)))
    return out


def _device_ctx(eng):
    import torch

    return torch.cuda.device(eng.device)


# engines for single blocks, keyed by the BlockParams object (as get_engine keys
# ModelParams); dropped when the block is garbage collected
_block_engines: dict[int, dict] = {}
_block_lock = threading.Lock()


def _drop_block(key: int) -> None:
    with _block_lock:
        per = _block_engines.pop(key, None)
    for eng in (per or {}).values():
        eng.close()


def _block_engine(block: BlockParams, config: ModelConfig, hist_len: int, precision: str, device):
    from .engine import FlameEngine

    d, f = config.hidden_dim, config.ffn_dim
    # one Climber block as a one-block model; the expert weights are never used
    one = ModelParams(blocks=[block], expert_w1=np.zeros((d, f)), expert_b1=np.zeros(f),
                      expert_w2=np.zeros((f, config.num_tasks)), expert_b2=np.zeros(config.num_tasks))
    max_h = 1
    while max_h < max(hist_len, 1):
        max_h *= 2
    cfg = dataclasses.replace(config, num_blocks=1, layers_per_block=len(block.layers),
                              max_history_len=max(max_h, config.max_history_len))
    total = sum(a.size for _, a in iter_param_arrays(one))
    fp = hash(param_stream(one).tobytes()) if total <= (1 << 22) else None
    key = (cfg, precision, device, fp)
    with _block_lock:
        per = _block_engines.get(id(block))
        if per is None:
            per = _block_engines[id(block)] = {}
            weakref.finalize(block, _drop_block, id(block))
        eng = per.get(key)
        if eng is None:
            eng = FlameEngine(one, cfg, precision=precision, device=device)
            per[key] = eng
        return eng


def block_forward(sub_seq: np.ndarray, candidates: np.ndarray, block: BlockParams, config: ModelConfig,
                  attn_impl: str = "fused", tile: int = DEFAULT_TILE, *, precision: str = DEFAULT_PRECISION,
                  device=None) -> np.ndarray:
    """Reference forward.py:75-140: one block's layer stack over
    [sub_seq | candidates] -> the candidates' final hidden states (C, d), through
    the forward pass's launch sequence (history rows of the last layer are not
    computed, as in the reference's fused path)."""
    if attn_impl not in ATTN_IMPLS:
        raise ValueError(f"attn_impl must be one of {ATTN_IMPLS}, got {attn_impl!r}")
    sub_seq = np.asarray(sub_seq)
    candidates = np.asarray(candidates)
    if sub_seq.ndim != 2 or candidates.ndim != 2:
        raise ValueError("sub_seq and candidates must be 2-d (length, hidden_dim)")
    d = config.hidden_dim
    if sub_seq.shape[1] != d or candidates.shape[1] != d:
        raise ValueError(f"embeddings must have width {d}")
    if candidates.shape[0] < 1:
        raise ValueError("candidates must be non-empty")
    if block.temperature <= 0:
        raise ValueError("block temperature must be positive")
    _precision(precision)
    eng = _block_engine(block, config, sub_seq.shape[0], precision, device)
    h, c = _f64(sub_seq), _f64(candidates)
    out = np.empty((1, c.shape[0], d))
    with _device_ctx(eng):
        _lib.check(eng.lib.flame_op_block_states(eng.handle, _ptr(h) if h.size else None, h.shape[0], _ptr(c),
                                                 c.shape[0], _ptr(out)))
    return out[0]


def model_forward_sequential(history: np.ndarray, candidates: np.ndarray, params: ModelParams,
                             config: ModelConfig, attn_impl: str = "naive", *,
                             precision: str = DEFAULT_PRECISION, device=None) -> np.ndarray:
    """Reference forward.py:207-225: score candidates one at a time (one device
    pass each) and stack the rows."""
    from .forward import check_forward_inputs, model_forward

    history = np.asarray(history)
    candidates = np.asarray(candidates)
    check_forward_inputs(history, candidates, config)
    rows = [model_forward(history, candidates[i:i + 1], params, config, attn_impl=attn_impl,
                          precision=precision, device=device) for i in range(candidates.shape[0])]
    return np.concatenate(rows, axis=0)

