"""CPU ORACLE — test infrastructure only, never the product path.

A plain-numpy (fp64) restatement of the reference FLAME ranker forward pass
and of its PDA feature-assembly semantics.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` leg may import
this module, and only as the checker / the timed CPU baseline.  The package
``paper_2509_22681_b200`` never imports it.

Parity pinning: ``tests/test_oracle_golden.py`` checks every function here
against golden vectors produced by the reference itself
(``oracle/gen_golden.py`` -> ``tests/golden/*.npz``), so the oracle is pinned
to the reference's own outputs, not just to this restatement.

Every function cites the reference code it restates (paths relative to
``/root/reference/pkg/src/flameserve/``).
"""

from __future__ import annotations

import math

import numpy as np

LN_EPS = 1e-5  # model/forward.py:28


def gelu(x):
    """tanh-form GELU, model/forward.py:34-36."""
    return 0.5 * x * (1.0 + np.tanh(math.sqrt(2.0 / math.pi) * (x + 0.044715 * x**3)))


def sigmoid(x):
    """model/forward.py:39-40."""
    return 1.0 / (1.0 + np.exp(-x))


def layer_norm(x, scale, shift):
    """Biased-variance LayerNorm, model/forward.py:43-47."""
    mean = x.mean(axis=-1, keepdims=True)
    dev = x - mean
    var = (dev * dev).mean(axis=-1, keepdims=True)
    return dev / np.sqrt(var + LN_EPS) * scale + shift


def split_sequence(history, num_blocks):
    """Contiguous equal split, model/forward.py:50-62."""
    length = history.shape[0]
    if length % num_blocks != 0:
        raise ValueError(f"history length {length} is not divisible by num_blocks {num_blocks}")
    step = length // num_blocks
    return [history[b * step:(b + 1) * step] for b in range(num_blocks)]


def _heads(x, nh):
    t, d = x.shape
    return x.reshape(t, nh, d // nh).transpose(1, 0, 2)


def _merge(xh):
    nh, t, hd = xh.shape
    return xh.transpose(1, 0, 2).reshape(t, nh * hd)


def sumi_candidates(qc, kh, vh, h, tau):
    """Candidate rows over history + self, model/attention.py:118-146."""
    scale = 1.0 / (tau * math.sqrt(qc.shape[2]))
    if h == 0:
        return vh.copy()
    s_self = np.einsum("hcd,hcd->hc", qc, kh[:, h:]) * scale
    s = (qc @ kh[:, :h].transpose(0, 2, 1)) * scale
    m = np.maximum(s.max(axis=2), s_self)
    w = np.exp(s - m[..., None])
    w_self = np.exp(s_self - m)
    z = w.sum(axis=2) + w_self
    out = w @ vh[:, :h] + w_self[..., None] * vh[:, h:]
    return out / z[..., None]


def sumi_all(qh, kh, vh, h, tau):
    """History rows causal + candidate rows, model/attention.py:149-178."""
    nh, t, dh = qh.shape
    scale = 1.0 / (tau * math.sqrt(dh))
    out = np.empty_like(qh)
    if h > 0:
        s = (qh[:, :h] @ kh[:, :h].transpose(0, 2, 1)) * scale
        s[:, ~np.tril(np.ones((h, h), dtype=bool))] = -np.inf
        s = np.exp(s - s.max(axis=-1, keepdims=True))
        s /= s.sum(axis=-1, keepdims=True)
        out[:, :h] = s @ vh[:, :h]
    if t - h > 0:
        out[:, h:] = sumi_candidates(qh[:, h:], kh, vh, h, tau)
    return out


def block_forward(sub, cand, block, nh):
    """One Climber block over [sub | cand], model/forward.py:75-140 (fused path)."""
    h = sub.shape[0]
    x = np.concatenate([sub, cand], axis=0)
    layers = block.layers
    for li, layer in enumerate(layers):
        if li == len(layers) - 1:
            y = layer_norm(x, layer.ln1_scale, layer.ln1_shift)
            qc = _heads(y[h:] @ layer.w_q, nh)
            kh = _heads(y @ layer.w_k, nh)
            vh = _heads(y @ layer.w_v, nh)
            oc = sumi_candidates(qc, kh, vh, h, block.temperature)
            xc = x[h:] + _merge(oc) @ layer.w_o
            y = layer_norm(xc, layer.ln2_scale, layer.ln2_shift)
            return xc + gelu(y @ layer.w1 + layer.b1) @ layer.w2 + layer.b2
        y = layer_norm(x, layer.ln1_scale, layer.ln1_shift)
        qh, kh, vh = (_heads(y @ w, nh) for w in (layer.w_q, layer.w_k, layer.w_v))
        x = x + _merge(sumi_all(qh, kh, vh, h, block.temperature)) @ layer.w_o
        y = layer_norm(x, layer.ln2_scale, layer.ln2_shift)
        x = x + gelu(y @ layer.w1 + layer.b1) @ layer.w2 + layer.b2
    return x[h:]


def gated_fusion(outs, params):
    """model/forward.py:143-156 (accumulated in block order)."""
    fused = np.zeros(outs[0].shape, dtype=outs[0].dtype)
    for out, block in zip(outs, params.blocks):
        fused = fused + sigmoid(out * block.gate_weight + block.gate_bias) * out
    return fused


def expert_heads(fused, params):
    """model/forward.py:159-166."""
    return sigmoid(gelu(fused @ params.expert_w1 + params.expert_b1) @ params.expert_w2 + params.expert_b2)


def model_forward(history, candidates, params, config):
    """model/forward.py:186-204: (H, d), (C, d) -> (C, num_tasks), fp64."""
    nh = config.hidden_dim // config.head_dim
    subs = split_sequence(np.asarray(history, dtype=np.float64), config.num_blocks)
    cand = np.asarray(candidates, dtype=np.float64)
    outs = [block_forward(s, cand, b, nh) for s, b in zip(subs, params.blocks)]
    return expert_heads(gated_fusion(outs, params), params)


# ------------------------------------------------------------------ PDA

_MASK64 = 0xFFFFFFFFFFFFFFFF
_ITEM_SALT = 0xC2B2AE3D27D4EB4F  # cache.py:40 (KeyKind.ITEM)


def splitmix64(x: int) -> int:
    """cache.py:43-48."""
    x = (x + 0x9E3779B97F4A7C15) & _MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _MASK64
    return x ^ (x >> 31)


def item_embedding(store_seed: int, item_id: int, version: int, dim: int) -> np.ndarray:
    """store.py:59-63 with FeatureKey(ITEM, id).stable_hash() (cache.py:60,75)."""
    key_hash = splitmix64((item_id ^ _ITEM_SALT) & _MASK64)
    mix = splitmix64(store_seed ^ splitmix64(key_hash ^ splitmix64(version)))
    return np.random.default_rng(mix).uniform(-1.0, 1.0, dim)


def resolve_embeddings(item_ids, table):
    """service.py:97-108 with a dense table (row = id; ids outside -> zero rows).

    Returns (rows, unique, inverse) — the np.unique maps are the bit-exact
    contract for the device dedup kernel.
    """
    ids = np.asarray(item_ids, dtype=np.int64)
    dim = table.shape[1]
    if ids.size == 0:
        return np.zeros((0, dim)), np.zeros(0, np.int64), np.zeros(0, np.int64)
    unique, inverse = np.unique(ids, return_inverse=True)
    rows = np.zeros((unique.size, dim))
    known = (unique >= 0) & (unique < table.shape[0])
    rows[known] = table[unique[known]]
    return rows[inverse], unique, inverse


def algorithmic_flops(config, hist_len: int, cand_count: int) -> int:
    """Algorithmic FLOPs (2 per MAC) of the fused pass — SURVEY.md §8(d)."""
    d, f, nb, L, tasks = (config.hidden_dim, config.ffn_dim, config.num_blocks,
                          config.layers_per_block, config.num_tasks)
    hb = hist_len // nb
    c = cand_count
    t = hb + c
    ph = hb * (hb + 1) // 2
    per_block = ((L - 1) * (8 * t * d * d + 4 * t * d * f + 4 * d * (ph + c * (hb + 1)))
                 + 4 * c * d * d + 4 * t * d * d + 4 * c * d * f + 4 * d * c * (hb + 1))
    return nb * per_block + 2 * c * d * f + 2 * c * f * tasks
