"""B200-native FLAME SUMI-ranker hot path (arXiv 2509.22681).

Drop-in for the reference's model/operator API (``flameserve.model``: every
name of its ``__all__``, model/__init__.py:36-66) and its executor-pool runner
(``flameserve.orchestrator``), executing on hand-written sm_100a kernels
(tcgen05/TMEM/TMA) through the C ABI in include/flame_b200.h.
"""

from .config import ModelConfig
from .params import (
    BlockParams,
    LayerParams,
    ModelParams,
    init_params,
    iter_param_arrays,
    load_params,
    param_stream,
    params_to_bytes,
    save_params,
)
from .mask import SumiMask, build_sumi_mask
from .flops import FlopsEstimate, allowed_pairs, estimate_flops, matmul_flops
from .forward import ATTN_IMPLS, check_forward_inputs, get_engine, model_forward, model_forward_batch, split_sequence
from .ops import (
    attention_naive,
    attention_sumi,
    attention_sumi_candidates,
    attention_tiled,
    block_forward,
    expert_heads,
    gated_fusion,
    gelu,
    layer_norm,
    masked_softmax_rows,
    model_forward_sequential,
    sigmoid,
)
from .engine import DeviceExecutor, FlameEngine

# the reference's flameserve.model.__all__ (model/__init__.py:36-66), in its order
REFERENCE_ALL = [
    "ModelConfig", "ModelParams", "BlockParams", "LayerParams", "SumiMask", "FlopsEstimate",
    "attention_naive", "attention_sumi", "attention_sumi_candidates", "attention_tiled", "masked_softmax_rows",
    "build_sumi_mask", "block_forward", "expert_heads", "gated_fusion", "gelu", "layer_norm", "model_forward",
    "model_forward_sequential", "sigmoid", "split_sequence", "allowed_pairs", "estimate_flops", "matmul_flops",
    "init_params", "iter_param_arrays", "load_params", "params_to_bytes", "save_params",
]

__all__ = REFERENCE_ALL + [
    "ATTN_IMPLS", "DeviceExecutor", "FlameEngine", "check_forward_inputs", "get_engine", "model_forward_batch",
    "param_stream",
]
