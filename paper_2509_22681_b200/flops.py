"""Algorithmic work of the fused forward pass (reporting only).

FLOPs count 2 per multiply-accumulate of the dense contractions the fused
path must perform; LayerNorm, softmax, GELU and gating
elementwise work is excluded.  Per request with hb = H / N_b, T = hb + C,
P_h = hb (hb + 1) / 2:

  F = N_b [ (L-1)(8 T d^2 + 4 T d f + 4 d (P_h + C (hb+1)))
            + 4 C d^2 + 4 T d^2 + 4 C d f + 4 d C (hb+1) ] + 2 C d f + 2 C f tasks

(last layer: Q and O on C rows, K and V on T rows, FFN on C rows, SUMI
attention over hb history keys + self).  The reference's ``estimate_flops``
(model/flops.py:58-101) counts the unfused scalar-operation pass instead; it
is mirrored below (``estimate_flops`` / ``matmul_flops`` / ``allowed_pairs`` /
``FlopsEstimate``) with the same counting convention and the same buckets, so a
caller of the reference estimator gets identical numbers.
"""

from __future__ import annotations

from dataclasses import dataclass

BUCKETS = ("attention", "softmax", "projections", "layer_norm", "ffn", "fusion", "experts")


@dataclass(frozen=True)
class FlopsEstimate:
    total: int
    breakdown: dict


def matmul_flops(m: int, k: int, n: int) -> int:
    """Reference flops.py:54-58: an (m, k) x (k, n) product costs m n (2k - 1)."""
    if min(m, k, n) == 0:
        return 0
    return m * n * (2 * k - 1)


def allowed_pairs(hist_len: int, cand_count: int) -> int:
    """Reference flops.py:61-63: allowed (row, key) pairs of the SUMI mask."""
    return hist_len * (hist_len + 1) // 2 + cand_count * (hist_len + 1)


def estimate_flops(config, hist_len: int, cand_count: int) -> FlopsEstimate:
    """Reference flops.py:66-110: scalar operations of one unfused forward pass,
    per bucket (mul / add each 1; softmax exponentials and divisions in the
    informational ``softmax`` bucket)."""
    if hist_len < 0 or cand_count < 0:
        raise ValueError("hist_len and cand_count must be non-negative")
    if hist_len % config.num_blocks != 0:
        raise ValueError(f"hist_len {hist_len} is not divisible by num_blocks {config.num_blocks}")
    d, dh, nh = config.hidden_dim, config.head_dim, config.num_heads
    f, tasks, nb, layers = config.ffn_dim, config.num_tasks, config.num_blocks, config.layers_per_block
    hb = hist_len // nb
    c = cand_count
    t = hb + c
    a = allowed_pairs(hb, c)
    # per layer and block: two LayerNorms of 7d - 1 over every row, four d x d
    # projections, attention (dot + scale per allowed pair, max-subtract and
    # normaliser adds, value aggregation) plus its residual, FFN plus residual
    per_layer = {
        "layer_norm": 2 * t * (7 * d - 1),
        "projections": 4 * matmul_flops(t, d, d),
        "attention": nh * (a * dh + a + a * dh) + nh * (a * (dh - 1) + a + (a - t) + (a - t) * dh) + t * d,
        "softmax": nh * 2 * a,
        "ffn": matmul_flops(t, d, f) + t * f + matmul_flops(t, f, d) + t * d + t * d,
    }
    stacks = nb * layers
    breakdown = {
        "attention": stacks * per_layer["attention"],
        "softmax": stacks * per_layer["softmax"],
        "projections": stacks * per_layer["projections"],
        "layer_norm": stacks * per_layer["layer_norm"],
        "ffn": stacks * per_layer["ffn"],
        "fusion": nb * 3 * c * d + (nb - 1) * c * d,
        "experts": matmul_flops(c, d, f) + c * f + matmul_flops(c, f, tasks) + c * tasks,
    }
    return FlopsEstimate(total=sum(breakdown.values()), breakdown=breakdown)


def algorithmic_flops(config, hist_len: int, cand_count: int) -> int:
    d, f, nb, L, tasks = (config.hidden_dim, config.ffn_dim, config.num_blocks,
                          config.layers_per_block, config.num_tasks)
    hb = hist_len // nb
    c = cand_count
    t = hb + c
    ph = hb * (hb + 1) // 2
    per_block = ((L - 1) * (8 * t * d * d + 4 * t * d * f + 4 * d * (ph + c * (hb + 1)))
                 + 4 * c * d * d + 4 * t * d * d + 4 * c * d * f + 4 * d * c * (hb + 1))
    return nb * per_block + 2 * c * d * f + 2 * c * f * tasks


def pda_bytes(hist_len: int, cand_count: int, unique: int, d: int, table_bytes: int = 2,
              act_bytes: int = 4) -> int:
    """Algorithmic HBM bytes of the PDA step for one request."""
    n = hist_len + cand_count
    return 8 * n + unique * d * table_bytes + n * d * act_bytes + 8 * unique + 8 * n
