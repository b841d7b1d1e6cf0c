"""Algorithmic work of the fused forward pass (reporting only).

FLOPs count 2 per multiply-accumulate of the dense contractions the fused
path must perform; LayerNorm, softmax, GELU and gating
elementwise work is excluded.  Per request with hb = H / N_b, T = hb + C,
P_h = hb (hb + 1) / 2:

  F = N_b [ (L-1)(8 T d^2 + 4 T d f + 4 d (P_h + C (hb+1)))
            + 4 C d^2 + 4 T d^2 + 4 C d f + 4 d C (hb+1) ] + 2 C d f + 2 C f tasks

(last layer: Q and O on C rows, K and V on T rows, FFN on C rows, SUMI
attention over hb history keys + self).  The reference's ``estimate_flops``
(model/flops.py:58-101) counts the unfused pass instead.
"""

from __future__ import annotations


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
