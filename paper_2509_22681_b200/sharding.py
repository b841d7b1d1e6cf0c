"""Request-level data parallelism across the GPUs of one node.

Requests are independent (nothing in model_forward crosses requests,
reference model/forward.py:186-204), so the scoring path shards WHOLE
requests over ranks with no collective: each rank holds a full weight
replica and scores its own requests.  ``torch.distributed`` is used only for
plumbing outside the data path — a barrier around timed regions and a MAX
reduce of the per-rank device time (the bench reports max over ranks).

``assign_requests`` is the host dispatcher's routing rule: greedy
least-outstanding-work (longest-processing-time first), where a request's
work is its candidate-row count plus its history rows — deterministic, so
every rank computes the same assignment without communicating.
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist


def request_work(hist_len: int, cand_count: int, num_blocks: int) -> int:
    """Rows the device touches for one request (history rows feed K/V once)."""
    return cand_count * num_blocks + hist_len


def assign_requests(shapes, world_size: int, num_blocks: int = 1) -> list[list[int]]:
    """shapes: list of (H, C). Returns per-rank request-index lists."""
    if world_size < 1:
        raise ValueError("world_size must be >= 1")
    order = sorted(range(len(shapes)), key=lambda i: (-request_work(*shapes[i], num_blocks), i))
    load = [0] * world_size
    out: list[list[int]] = [[] for _ in range(world_size)]
    for i in order:
        r = min(range(world_size), key=lambda k: (load[k], k))
        out[r].append(i)
        load[r] += request_work(*shapes[i], num_blocks)
    for lst in out:
        lst.sort()
    return out


class Dist:
    """Process-group plumbing read from the torchrun environment."""

    def __init__(self, backend: str | None = None) -> None:
        self.world_size = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        self.enabled = self.world_size > 1
        self.backend = backend
        # FLAME_SHARE_GPU=1 (tests of the multi-rank path on a box with fewer GPUs
        # than ranks): ranks share GPUs round-robin and the plumbing runs over
        # gloo, since NCCL needs one GPU per rank.  Production runs one rank per GPU.
        n_dev = torch.cuda.device_count() if torch.cuda.is_available() else 0
        self.shared_gpu = (os.environ.get("FLAME_SHARE_GPU") == "1" and n_dev > 0
                           and self.world_size > n_dev)
        self.device_index = self.local_rank % n_dev if self.shared_gpu else self.local_rank
        if self.enabled and not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            be = backend or ("nccl" if torch.cuda.is_available() and not self.shared_gpu else "gloo")
            self.backend = be
            if be == "nccl":
                torch.cuda.set_device(self.local_rank)
                dist.init_process_group(be, device_id=torch.device("cuda", self.local_rank))
            else:
                dist.init_process_group(be)

    def barrier(self) -> None:
        if self.enabled:
            dist.barrier()

    def max(self, value: float) -> float:
        """Max over ranks of a scalar (e.g. the timed-region duration)."""
        if not self.enabled:
            return float(value)
        dev = torch.device("cuda", self.device_index) if self.backend == "nccl" else torch.device("cpu")
        t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, value: float) -> float:
        if not self.enabled:
            return float(value)
        dev = torch.device("cuda", self.device_index) if self.backend == "nccl" else torch.device("cpu")
        t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    def close(self) -> None:
        if self.enabled and dist.is_initialized():
            dist.destroy_process_group()
