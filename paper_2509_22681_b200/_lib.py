"""ctypes binding of the C ABI declared in include/flame_b200.h.

There is no fallback: if the sm_100a library is missing or fails to load, every
entry point raises ``RuntimeError`` — the product path never degrades to a CPU
or PyTorch implementation.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

# FLAME_B200_LIB: load an alternative build of the same library (dev A/B variants)
LIB_PATH = Path(os.environ.get("FLAME_B200_LIB") or Path(__file__).resolve().parent / "_flame_b200.so")

FLAME_BF16, FLAME_FP32 = 0, 1
INPUT_EMBEDDINGS, INPUT_IDS, INPUT_GATHER_ONLY = 0, 1, 2
TABLE_BF16, TABLE_FP32 = 0, 1

EXPORTED = (
    "flame_create", "flame_create_flmp", "flame_destroy", "flame_set_table", "flame_update_table",
    "flame_update_table_values", "flame_pack_padded", "flame_exec_set_staging", "flame_exec_submit",
    "flame_exec_wait", "flame_exec_query",
    "flame_exec_list_capacity", "flame_exec_create", "flame_exec_destroy", "flame_exec_run",
    "flame_exec_capture", "flame_exec_replay", "flame_exec_launch_count", "flame_exec_workspace",
    "flame_exec_profile",
    "flame_last_error", "flame_device_sm_count", "flame_copy_to_host",
    "flame_op_attention_sumi", "flame_op_attention_masked", "flame_op_rows", "flame_op_gated_fusion",
    "flame_op_block_states", "flame_op_expert_heads",
)
OP_GELU, OP_SIGMOID, OP_LAYER_NORM, OP_SOFTMAX = 0, 1, 2, 3


class FlameModelDesc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in (
        "hidden_dim", "head_dim", "num_blocks", "layers_per_block", "ffn_dim", "num_tasks",
        "max_history_len", "max_candidates")] + [("seed", ctypes.c_ulonglong)]


class FlameIO(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in (
        "hist_emb", "cand_emb", "hist_ids", "cand_ids", "hist_len", "cand_len", "out_offset",
        "scores", "unique_ids", "inverse", "n_unique", "active")]


class FlameStaging(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in (
        "h_meta", "d_meta", "h_hist_ids", "h_cand_ids", "h_hist_emb", "h_cand_emb", "h_scores")]


_lib = None
_lock = threading.Lock()


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"FLAME sm_100a library not built ({LIB_PATH}); run "
                "`python -m paper_2509_22681_b200.build` — there is no CPU fallback")
        lib = ctypes.CDLL(str(LIB_PATH))
        P, I, LL = ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong
        sig = {
            "flame_create": (I, [ctypes.POINTER(FlameModelDesc), P, LL, I, I, ctypes.POINTER(P)]),
            "flame_create_flmp": (I, [P, LL, I, I, ctypes.POINTER(P)]),
            "flame_destroy": (I, [P]),
            "flame_set_table": (I, [P, P, LL, I]),
            "flame_update_table": (I, [P, P, P, LL, P]),
            "flame_update_table_values": (I, [P, P, P, LL, P, LL, P]),
            "flame_pack_padded": (I, [P, LL, P, P, LL, LL]),
            "flame_exec_set_staging": (I, [P, ctypes.POINTER(FlameStaging)]),
            "flame_exec_submit": (I, [P, I, I, LL, P]),
            "flame_exec_wait": (I, [P]),
            "flame_exec_query": (I, [P]),
            "flame_exec_list_capacity": (I, [I, I, I]),
            "flame_exec_create": (I, [P, I, I, I, ctypes.POINTER(FlameIO), ctypes.POINTER(P)]),
            "flame_exec_destroy": (I, [P]),
            "flame_exec_run": (I, [P, I, P]),
            "flame_exec_capture": (I, [P, I, P]),
            "flame_exec_replay": (I, [P, P]),
            "flame_exec_launch_count": (I, [P, I]),
            "flame_exec_profile": (I, [P, I, P, I, P, P, P, P]),
            "flame_exec_workspace": (P, [P, ctypes.c_char_p]),
            "flame_last_error": (ctypes.c_char_p, []),
            "flame_device_sm_count": (I, [I]),
            "flame_copy_to_host": (I, [P, P, LL]),
            "flame_op_attention_sumi": (I, [I, I, I, I, I, I, I, ctypes.c_double, P, P, P, P]),
            "flame_op_attention_masked": (I, [I, I, I, ctypes.c_double, P, P, P, P, P]),
            "flame_op_rows": (I, [I, I, LL, I, P, P, P, P]),
            "flame_op_gated_fusion": (I, [I, I, LL, I, P, P, P, P]),
            "flame_op_block_states": (I, [P, P, LL, P, LL, P]),
            "flame_op_expert_heads": (I, [P, P, LL, P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc: int) -> None:
    """Map C status codes to the reference's exception types."""
    if rc == 0:
        return
    msg = (load().flame_last_error() or b"").decode(errors="replace")
    if rc == 1:
        raise ValueError(msg)
    raise RuntimeError(msg)
