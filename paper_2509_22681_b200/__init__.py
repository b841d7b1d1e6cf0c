"""B200-native FLAME SUMI-ranker hot path (arXiv 2509.22681).

Drop-in for the reference's model/operator API (``flameserve.model``:
``ModelConfig``, ``init_params``/``load_params``, ``model_forward``) and its
executor-pool runner (``flameserve.orchestrator``), executing on hand-written
sm_100a kernels (tcgen05/TMEM/TMA) through the C ABI in include/flame_b200.h.
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
from .forward import ATTN_IMPLS, check_forward_inputs, get_engine, model_forward, model_forward_batch, split_sequence
from .engine import DeviceExecutor, FlameEngine

__all__ = [
    "ATTN_IMPLS",
    "BlockParams",
    "DeviceExecutor",
    "FlameEngine",
    "LayerParams",
    "ModelConfig",
    "ModelParams",
    "check_forward_inputs",
    "get_engine",
    "init_params",
    "iter_param_arrays",
    "load_params",
    "model_forward",
    "model_forward_batch",
    "param_stream",
    "params_to_bytes",
    "save_params",
    "split_sequence",
]
