"""Host side of the B200 path: device-resident model context and fixed-shape
executors over the C ABI (include/flame_b200.h).

PyTorch is used only as plumbing — device / pinned-host allocation and CUDA
streams.  Every arithmetic step of the forward pass runs in the sm_100a
kernels of ``_flame_b200.so``; if that library is missing the constructors
raise instead of falling back.
"""

from __future__ import annotations

import ctypes
import threading
import weakref

import numpy as np
import torch

from . import _lib
from .config import ModelConfig
from .params import ModelParams, param_stream

PRECISIONS = {"bf16": _lib.FLAME_BF16, "fp32": _lib.FLAME_FP32}


def _next_pow2(x: int) -> int:
    p = 1
    while p < x:
        p <<= 1
    return p


def _require_cuda(device) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the FLAME B200 path needs a CUDA device; there is no CPU fallback")
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else int(device))
    major, _ = torch.cuda.get_device_capability(dev)
    if major < 10:
        raise RuntimeError(f"device {dev} is not sm_100-class (capability major {major})")
    return dev


class FlameEngine:
    """One device context: repacked weights (+ optional embedding table)."""

    def __init__(self, params: ModelParams | None, config: ModelConfig, precision: str = "bf16",
                 device=None, *, flmp: bytes | None = None) -> None:
        if params is None and flmp is None:
            raise ValueError("params or an FLMP image is required")
        if precision not in PRECISIONS:
            raise ValueError(f"precision must be one of {tuple(PRECISIONS)}, got {precision!r}")
        self.lib = _lib.load()
        self.device = _require_cuda(device)
        self.config = config
        self.precision = precision
        ctx = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            if flmp is not None:
                # the C loader parses the FLMP header and body itself (flame_create_flmp)
                buf = np.frombuffer(flmp, dtype=np.uint8)
                _lib.check(self.lib.flame_create_flmp(buf.ctypes.data, buf.size, PRECISIONS[precision],
                                                      self.device.index, ctypes.byref(ctx)))
            else:
                desc = _lib.FlameModelDesc(
                    config.hidden_dim, config.head_dim, config.num_blocks, config.layers_per_block,
                    config.ffn_dim, config.num_tasks, config.max_history_len, config.max_candidates,
                    config.seed)
                stream = np.ascontiguousarray(param_stream(params), dtype=np.float64)
                _lib.check(self.lib.flame_create(ctypes.byref(desc), stream.ctypes.data, stream.size,
                                                 PRECISIONS[precision], self.device.index,
                                                 ctypes.byref(ctx)))
        self._ctx = ctx
        self._executors: dict[tuple, "DeviceExecutor"] = {}
        self._lock = threading.Lock()
        self.num_items = 0

    @classmethod
    def from_flmp(cls, source, precision: str = "bf16", device=None) -> "FlameEngine":
        """Device context straight from an FLMP parameter file (path or bytes,
        reference model/params.py:131-207): the C library parses the header and
        repacks the fp64 body; the host only reads the config for its own use."""
        from .params import config_from_header

        data = bytes(source) if isinstance(source, (bytes, bytearray, memoryview)) else open(source, "rb").read()
        config = config_from_header(data)
        return cls(None, config, precision=precision, device=device, flmp=data)

    @property
    def handle(self) -> ctypes.c_void_p:
        if self._ctx is None:
            raise RuntimeError("engine is closed")
        return self._ctx

    def set_table(self, table: np.ndarray, dtype: str = "bf16") -> None:
        """Upload a dense embedding table (row = item id) for the id-input path."""
        t = np.ascontiguousarray(table, dtype=np.float32)
        if t.ndim != 2 or t.shape[1] != self.config.hidden_dim:
            raise ValueError(f"table must be (num_items, {self.config.hidden_dim})")
        code = {"bf16": _lib.TABLE_BF16, "fp32": _lib.TABLE_FP32}[dtype]
        with torch.cuda.device(self.device):
            _lib.check(self.lib.flame_set_table(self.handle, t.ctypes.data, t.shape[0], code))
        self.num_items = t.shape[0]

    def update_rows(self, ids, rows: np.ndarray) -> None:
        """Overwrite table rows ``ids`` with ``rows`` (n, hidden_dim) in place on the
        device (incremental refresh; ids outside the table are ignored)."""
        if not self.num_items:
            raise RuntimeError("no embedding table set (set_table)")
        i = np.ascontiguousarray(ids, dtype=np.int64).reshape(-1)
        r = np.ascontiguousarray(rows, dtype=np.float32)
        if r.shape != (i.size, self.config.hidden_dim):
            raise ValueError(f"rows must be ({i.size}, {self.config.hidden_dim})")
        stream = torch.cuda.current_stream(self.device)
        with torch.cuda.device(self.device):
            _lib.check(self.lib.flame_update_table(self.handle, i.ctypes.data, r.ctypes.data, i.size,
                                                   ctypes.c_void_p(stream.cuda_stream)))

    def update_values(self, ids, values) -> None:
        """Overwrite table rows ``ids`` from raw store feature values (bytes in the
        reference wire format, store.py:66-78), decoded on the device; short or
        empty values give zero rows."""
        if not self.num_items:
            raise RuntimeError("no embedding table set (set_table)")
        i = np.ascontiguousarray(ids, dtype=np.int64).reshape(-1)
        if len(values) != i.size:
            raise ValueError("one value per id")
        stride = max([len(v) for v in values] + [8])
        stride = (stride + 7) // 8 * 8
        buf = np.zeros((i.size, stride), dtype=np.uint8)
        lens = np.zeros(i.size, dtype=np.int32)
        for k, v in enumerate(values):
            buf[k, :len(v)] = np.frombuffer(v, dtype=np.uint8)
            lens[k] = len(v)
        stream = torch.cuda.current_stream(self.device)
        with torch.cuda.device(self.device):
            _lib.check(self.lib.flame_update_table_values(self.handle, i.ctypes.data, buf.ctypes.data, stride,
                                                          lens.ctypes.data, i.size,
                                                          ctypes.c_void_p(stream.cuda_stream)))

    def bucket(self, hist_len: int, cand_count: int) -> tuple[int, int]:
        """(hb_bkt, c_bkt) shape bucket for one request (powers of two, capped)."""
        cfg = self.config
        hb = hist_len // cfg.num_blocks
        hb_max = cfg.max_history_len // cfg.num_blocks
        hb_bkt = min(_next_pow2(hb), hb_max) if hb > 0 else 0
        c_bkt = max(8, _next_pow2(cand_count))
        if c_bkt > cfg.max_candidates >= cand_count:
            c_bkt = max(cand_count, cfg.max_candidates)
        return hb_bkt, c_bkt

    def executor(self, R: int, hb_bkt: int, c_bkt: int, *, with_ids: bool = False,
                 cache: bool = True) -> "DeviceExecutor":
        key = (R, hb_bkt, c_bkt, with_ids)
        if not cache:
            return DeviceExecutor(self, R, hb_bkt, c_bkt, with_ids=with_ids)
        with self._lock:
            ex = self._executors.get(key)
            if ex is None:
                ex = DeviceExecutor(self, R, hb_bkt, c_bkt, with_ids=with_ids)
                self._executors[key] = ex
            return ex

    def close(self) -> None:
        with self._lock:
            for ex in self._executors.values():
                ex.close()
            self._executors.clear()
        if self._ctx is not None:
            self.lib.flame_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DeviceExecutor:
    """A fixed-shape compute slot (reference orchestrator.py:104-133 Executor):
    caller-owned device I/O buffers + pinned host mirrors allocated once, the
    C-side workspace, a private CUDA stream and (after ``capture``) a CUDA graph
    of the whole forward pass.  ``score`` runs H2D -> forward -> D2H."""

    def __init__(self, engine: FlameEngine, R: int, hb_bkt: int, c_bkt: int,
                 with_ids: bool = False, pinned: bool = True) -> None:
        cfg = engine.config
        self.engine = engine
        self.R, self.hb_bkt, self.c_bkt = R, hb_bkt, c_bkt
        self.H_bkt = hb_bkt * cfg.num_blocks
        self.cap = max(self.H_bkt, c_bkt)
        dev = engine.device
        d, tasks = cfg.hidden_dim, cfg.num_tasks
        self.lock = threading.Lock()
        self.allocations = 0

        def dalloc(shape, dtype):
            self.allocations += 1
            # never hand a null pointer to the C side for an empty (H = 0) buffer
            t = torch.zeros(max(1, int(np.prod(shape))), dtype=dtype, device=dev)
            return t[: int(np.prod(shape))].view(shape)

        def halloc(shape, dtype):
            self.allocations += 1
            # pageable staging (pinned=False) is the reference's mem_opt=off ablation:
            # the copies then go through the driver's bounce buffer, synchronously
            t = torch.zeros(max(1, int(np.prod(shape))), dtype=dtype, pin_memory=pinned)
            return t[: int(np.prod(shape))].view(shape)

        self.hist_emb = dalloc((R, self.H_bkt, d), torch.float32)
        self.cand_emb = dalloc((R, c_bkt, d), torch.float32)
        # per-slot metadata in one block (one H2D per batch): hist_len, cand_len,
        # out_offset, and [3][0] = active slot count
        self.meta = dalloc((4, R), torch.int32)
        self.hist_len, self.cand_len, self.out_offset = self.meta[0], self.meta[1], self.meta[2]
        self.active = self.meta[3, :1]
        self.scores = dalloc((R * c_bkt, tasks), torch.float32)
        self.h_meta = halloc((4, R), torch.int32)
        self.h_scores = halloc((R * c_bkt, tasks), torch.float32)
        self.h_hist = halloc((R, self.H_bkt, d), torch.float32)
        self.h_cand = halloc((R, c_bkt, d), torch.float32)
        self.with_ids = with_ids
        if with_ids:
            self.hist_ids = dalloc((R, self.H_bkt), torch.int64)
            self.cand_ids = dalloc((R, c_bkt), torch.int64)
            self.unique = dalloc((2 * R, self.cap), torch.int64)
            self.inverse = dalloc((2 * R, self.cap), torch.int64)
            self.n_unique = dalloc((2 * R,), torch.int32)
            self.h_hist_ids = halloc((R, self.H_bkt), torch.int64)
            self.h_cand_ids = halloc((R, c_bkt), torch.int64)
        self.stream = torch.cuda.Stream(device=dev)
        self._done = torch.cuda.Event()
        self._pending = None
        self._dummy = torch.zeros(16, dtype=torch.float32, device=dev)

        def ptr(t):
            if t is None:
                return None
            return t.data_ptr() if t.numel() > 0 else self._dummy.data_ptr()

        io = _lib.FlameIO(
            ptr(self.hist_emb), ptr(self.cand_emb),
            ptr(self.hist_ids) if with_ids else None,
            ptr(self.cand_ids) if with_ids else None,
            ptr(self.hist_len), ptr(self.cand_len), ptr(self.out_offset), ptr(self.scores),
            ptr(self.unique) if with_ids else None,
            ptr(self.inverse) if with_ids else None,
            ptr(self.n_unique) if with_ids else None,
            ptr(self.active))
        ex = ctypes.c_void_p()
        with torch.cuda.device(dev):
            _lib.check(engine.lib.flame_exec_create(engine.handle, R, hb_bkt, c_bkt, ctypes.byref(io),
                                                    ctypes.byref(ex)))
        self._ex = ex
        st = _lib.FlameStaging(self.h_meta.data_ptr(), self.meta.data_ptr(),
                               ptr(self.h_hist_ids) if with_ids else None,
                               ptr(self.h_cand_ids) if with_ids else None,
                               self.h_hist.data_ptr(), self.h_cand.data_ptr(), self.h_scores.data_ptr())
        _lib.check(engine.lib.flame_exec_set_staging(ex, ctypes.byref(st)))
        self._native = False
        self._graph_mode = None
        self._finalizer = weakref.finalize(self, engine.lib.flame_exec_destroy, ex)
        self.n_real = 0

    # ------------------------------------------------------------- staging
    def _set_meta(self, hist_lens, cand_lens) -> int:
        R = self.R
        if len(hist_lens) > R:
            raise ValueError(f"{len(hist_lens)} requests exceed executor capacity {R}")
        meta = self.h_meta.numpy()
        meta[:] = 0
        n = len(hist_lens)
        meta[0, :n] = hist_lens
        meta[1, :n] = cand_lens
        offs = np.zeros(R, dtype=np.int64)
        offs[1:n] = np.cumsum(np.asarray(cand_lens, dtype=np.int64))[:-1] if n > 1 else 0
        meta[2, :n] = offs[:n]
        meta[3, 0] = n  # slots n..R-1 are skipped by the kernels (one graph serves any n <= R)
        self.n_real = int(np.sum(cand_lens))
        self._counts = np.asarray(cand_lens, dtype=np.int64)
        return n

    def _check_lengths(self, h: int, c: int) -> None:
        cfg = self.engine.config
        if h % cfg.num_blocks != 0:
            raise ValueError(f"history length {h} is not divisible by num_blocks {cfg.num_blocks}")
        if h > self.H_bkt:
            raise ValueError(f"history length {h} exceeds executor capacity {self.H_bkt}")
        if not 1 <= c <= self.c_bkt:
            raise ValueError(f"candidate count {c} outside [1, {self.c_bkt}]")

    def _lengths(self, requests) -> tuple[np.ndarray, np.ndarray]:
        """Per-request (H, C) as int64 arrays, validated against the executor."""
        n = len(requests)
        if n > self.R:
            raise ValueError(f"{n} requests exceed executor capacity {self.R}")
        hl = np.fromiter((len(h) for h, _ in requests), dtype=np.int64, count=n)
        cl = np.fromiter((len(c) for _, c in requests), dtype=np.int64, count=n)
        bad = np.flatnonzero((hl % self.engine.config.num_blocks != 0) | (hl > self.H_bkt) | (cl < 1)
                             | (cl > self.c_bkt))
        if bad.size:
            self._check_lengths(int(hl[bad[0]]), int(cl[bad[0]]))  # raises the specific error
        return hl, cl

    def _pack(self, dst: torch.Tensor, arrays, lens: np.ndarray, dtype, width: int = 0) -> None:
        """Copy the requests' arrays into the pinned mirror ``dst`` ([R][slot...]),
        one C call for the batch (flame_pack_padded)."""
        if not lens.any():
            return
        # empty 2-D records may come as shape (0,): drop them (1-D id lists concatenate as they are)
        parts = arrays if not width or lens.all() else [a for a, l in zip(arrays, lens.tolist()) if l]
        flat = np.concatenate(parts, dtype=dtype, casting="unsafe") if len(parts) > 1 \
            else np.asarray(parts[0], dtype=dtype)
        if width and (flat.ndim != 2 or flat.shape[1] != width):
            raise ValueError(f"embedding rows must have hidden_dim {width} columns, got shape {flat.shape[1:]}")
        flat = np.ascontiguousarray(flat)
        lens = np.ascontiguousarray(lens, dtype=np.int64)
        elem = flat.itemsize * (width or 1)
        _lib.check(self.engine.lib.flame_pack_padded(dst.data_ptr(), dst.stride(0) * dst.element_size(),
                                                     flat.ctypes.data, lens.ctypes.data, lens.size, elem))

    def _fill_embeddings(self, requests) -> int:
        hl, cl = self._lengths(requests)
        d = self.engine.config.hidden_dim
        self._pack(self.h_hist, [h for h, _ in requests], hl, np.float32, d)
        self._pack(self.h_cand, [c for _, c in requests], cl, np.float32, d)
        return self._set_meta(hl, cl)

    def _fill_ids(self, requests) -> int:
        if not self.with_ids:
            raise RuntimeError("executor was built without id buffers")
        hl, cl = self._lengths(requests)
        self._pack(self.h_hist_ids, [h for h, _ in requests], hl, np.int64)
        self._pack(self.h_cand_ids, [c for _, c in requests], cl, np.int64)
        return self._set_meta(hl, cl)

    def stage_embeddings(self, requests) -> None:
        """requests: sequence of (history (H, d), candidates (C, d)) arrays."""
        n = self._fill_embeddings(requests)
        with torch.cuda.stream(self.stream):
            self.hist_emb[:n].copy_(self.h_hist[:n], non_blocking=True)
            self.cand_emb[:n].copy_(self.h_cand[:n], non_blocking=True)
            self._upload_meta()

    def stage_ids(self, requests) -> None:
        """requests: sequence of (history ids (H,), candidate ids (C,)) int arrays."""
        n = self._fill_ids(requests)
        with torch.cuda.stream(self.stream):
            # only the slots in use cross PCIe (the kernels skip the others)
            self.hist_ids[:n].copy_(self.h_hist_ids[:n], non_blocking=True)
            self.cand_ids[:n].copy_(self.h_cand_ids[:n], non_blocking=True)
            self._upload_meta()

    def _upload_meta(self) -> None:
        self.meta.copy_(self.h_meta, non_blocking=True)

    # ------------------------------------------------------------- running
    def run(self, mode: int = _lib.INPUT_EMBEDDINGS, graph: bool = True) -> None:
        lib = self.engine.lib
        s = ctypes.c_void_p(self.stream.cuda_stream)
        with torch.cuda.device(self.engine.device):
            if graph:
                if self._graph_mode != mode:
                    _lib.check(lib.flame_exec_capture(self._ex, mode, s))
                    self._graph_mode = mode
                _lib.check(lib.flame_exec_replay(self._ex, s))
            else:
                _lib.check(lib.flame_exec_run(self._ex, mode, s))

    def fetch_scores(self) -> np.ndarray:
        n = self.n_real
        with torch.cuda.stream(self.stream):
            self.h_scores[:n].copy_(self.scores[:n], non_blocking=True)
        self.stream.synchronize()
        return self.h_scores[:n].numpy().astype(np.float64)

    def score(self, requests, graph: bool = True) -> list[np.ndarray]:
        """Score a batch of (history, candidates) embedding requests."""
        with self.lock:
            self.submit(requests, ids=False, graph=graph)
            return self.collect()

    def score_ids(self, requests, graph: bool = True) -> list[np.ndarray]:
        """Score a batch of (history ids, candidate ids) requests via the PDA path."""
        with self.lock:
            self.submit(requests, ids=True, graph=graph)
            return self.collect()

    # ------------------------------------------------- asynchronous use (DSO)
    def submit(self, requests, ids: bool, graph: bool = True) -> None:
        """Stage a batch, replay the forward pass and queue the score D2H, all on
        this executor's stream, without waiting.  ``collect`` returns the scores.
        With ``graph`` the round trip is one C call (flame_exec_submit: H2D of the
        slots in use, graph replay, D2H, completion event).  The pinned staging
        buffers are reused, so a second ``submit`` must come after the first
        ``collect`` (the DSO keeps a ring of executors per bucket)."""
        if self._pending is not None:
            raise RuntimeError("executor has an uncollected batch")
        mode = _lib.INPUT_IDS if ids else _lib.INPUT_EMBEDDINGS
        if graph:
            n = self._fill_ids(requests) if ids else self._fill_embeddings(requests)
            _lib.check(self.engine.lib.flame_exec_submit(self._ex, mode, n, self.n_real,
                                                         ctypes.c_void_p(self.stream.cuda_stream)))
            self._graph_mode = mode
            self._native = True
        else:
            if ids:
                self.stage_ids(requests)
            else:
                self.stage_embeddings(requests)
            self.run(mode, graph=False)
            n = self.n_real
            with torch.cuda.stream(self.stream):
                self.h_scores[:n].copy_(self.scores[:n], non_blocking=True)
                self._done.record(self.stream)
            self._native = False
        self._pending = self._counts

    @property
    def pending(self) -> bool:
        return self._pending is not None

    def ready(self) -> bool:
        if self._pending is None:
            return False
        if not self._native:
            return self._done.query()
        rc = self.engine.lib.flame_exec_query(self._ex)
        if rc not in (0, 1):
            _lib.check(rc)
        return rc == 1

    def wait(self) -> None:
        """Block until the last submitted batch (if any) finished on the device."""
        if self._pending is None:
            return
        if self._native:
            _lib.check(self.engine.lib.flame_exec_wait(self._ex))
        else:
            self._done.synchronize()

    def collect(self) -> list[np.ndarray]:
        if self._pending is None:
            raise RuntimeError("nothing submitted")
        counts = self._pending
        try:
            self.wait()
            flat = self.h_scores[: self.n_real].numpy().astype(np.float64)
        finally:
            self._pending = None  # a failed batch must not leave the executor stuck
        return _split_rows(flat, counts)

    def profile(self, mode: int = _lib.INPUT_EMBEDDINGS, max_launches: int = 256) -> list[dict]:
        """One eager run with per-launch CUDA events on this executor's stream:
        [{name, ms, flops, bytes}] in launch order."""
        ms = np.zeros(max_launches, np.float32)
        names = ctypes.create_string_buffer(64 * max_launches)
        flops = np.zeros(max_launches, np.float64)
        byts = np.zeros(max_launches, np.float64)
        with torch.cuda.device(self.engine.device):
            n = self.engine.lib.flame_exec_profile(
                self._ex, mode, ctypes.c_void_p(self.stream.cuda_stream), max_launches,
                ms.ctypes.data, names, flops.ctypes.data, byts.ctypes.data)
        if n < 0:
            _lib.check(-n)
        raw = names.raw
        return [{"name": raw[64 * i:64 * i + 64].split(b"\0")[0].decode(), "ms": float(ms[i]),
                 "flops": float(flops[i]), "bytes": float(byts[i])} for i in range(n)]

    def launch_count(self) -> int:
        return int(self.engine.lib.flame_exec_launch_count(self._ex, 0))

    def workspace(self, name: str) -> int:
        return int(self.engine.lib.flame_exec_workspace(self._ex, name.encode()) or 0)

    def read_workspace(self, name: str, shape, dtype=np.float32) -> np.ndarray:
        """Copy an internal workspace tensor to the host (parity debugging)."""
        self.stream.synchronize()
        ptr = self.workspace(name)
        if not ptr:
            raise KeyError(name)
        out = np.empty(shape, dtype=dtype)
        _lib.check(self.engine.lib.flame_copy_to_host(out.ctypes.data, ptr, out.nbytes))
        return out

    def close(self) -> None:
        if self._finalizer.alive:
            self.stream.synchronize()
            self._finalizer()


def _split_rows(flat: np.ndarray, counts) -> list[np.ndarray]:
    ends = np.cumsum(counts).tolist()
    return [flat[a:b] for a, b in zip([0] + ends[:-1], ends)]
