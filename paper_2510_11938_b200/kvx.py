"""ctypes binding of the kvx C-ABI (include/kvx.h) -- the Python face of the
B200-native inflight-refactor KV transition.

Mirrors the reference's transition interface (RefactorCtx and the engine
handlers of /root/reference/proj/src/engine.cpp:532-772) with the same names
and meaning:

    t = Transition(geometry, old_plan, new_plan, device, ...)   # begin_refactor grant
    t.begin_refactor(live)                   # wave 0        engine.cpp:637-647
    t.on_kv_sync_complete(live, inflight)    # delta/barrier/final engine.cpp:651-688
    t.on_refactor_commit(live)               # Eq. 10 + compaction engine.cpp:690-713
    t.abort_refactor()                       # revocation    engine.cpp:759-772

`live` is the (request, kv_tokens) set of live requests homed on the
instance, as ``(req: int32[n], kv: int64[n])`` ascending in req.

There is no CPU fallback: if ``_lib/libkvx.so`` is missing the import fails
loudly (build it with ``python -m paper_2510_11938_b200.build``).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libkvx.so")

KVX_OK, KVX_EINVAL, KVX_ESTALE, KVX_ENOSPC, KVX_ECUDA, KVX_ESTATE = 0, -1, -2, -3, -4, -5
ACT_DELTA, ACT_BARRIER_WAIT, ACT_FINAL = 0, 1, 2
# per layer: [blocks][2][B][H][D] | [2][blocks][B][H][D] | [blocks][2][H][B][D] (HND, vLLM FlashInfer on B200)
LAYOUT_BLOCKS, LAYOUT_KV_PLANES, LAYOUT_HEADS = 0, 1, 2
IPC_HANDLE_BYTES = 64


class KvxError(RuntimeError):
    """A non-zero kvx status.  ``code`` is the KVX_E* value."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"kvx error {code}: {msg}")
        self.code = code


class StaleEpoch(KvxError):
    """Epoch mismatch -- the reference drops such events (engine.cpp:654,693)."""


class NoSpace(KvxError):
    """Destination full -- the reference turns this into a hold (engine.cpp:563)."""


class Geometry(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("num_kv_heads", C.c_int32), ("head_dim", C.c_int32),
                ("elem_bytes", C.c_int32), ("block_tokens", C.c_int32)]

    @property
    def token_bytes(self) -> int:
        return self.num_kv_heads * self.head_dim * self.elem_bytes

    @property
    def block_bytes(self) -> int:
        return 2 * self.block_tokens * self.token_bytes

    @property
    def kv_bytes_per_token(self) -> int:
        """ExecModelParams::kv_bytes_per_token (modelgraph.hpp:115)."""
        return 2 * self.num_layers * self.token_bytes


class _Plan(C.Structure):
    _fields_ = [("num_stages", C.c_int32), ("boundaries", C.POINTER(C.c_int32)),
                ("pools", C.POINTER(C.c_void_p))]


class _Desc(C.Structure):
    _fields_ = [("geometry", Geometry), ("old_plan", _Plan), ("new_plan", _Plan),
                ("device", C.c_int32), ("max_requests", C.c_int32), ("max_blocks", C.c_int32),
                ("dst_num_blocks", C.c_int32), ("src_block_table", C.POINTER(C.c_int32)),
                ("epoch", C.c_uint64), ("max_sync_rounds", C.c_int32),
                ("kv_bytes_per_token", C.c_double), ("stream", C.c_void_p),
                ("dst_blockmgr", C.c_void_p), ("pull", C.c_int32), ("layer_pull", C.POINTER(C.c_uint8)),
                ("max_ctas", C.c_int32), ("src_block_table_dev", C.POINTER(C.c_int32))]


class _CommitResult(C.Structure):
    _fields_ = [("violations", C.c_int64), ("row_ptr", C.POINTER(C.c_int32)),
                ("blocks", C.POINTER(C.c_int32)), ("blocks_cap", C.c_int32),
                ("n_blocks", C.c_int32), ("free_list", C.POINTER(C.c_int32)),
                ("free_cap", C.c_int32), ("n_free", C.c_int32)]


class MicroBatch(C.Structure):
    _fields_ = [("batch_id", C.c_int64), ("after_stage", C.c_int32), ("tokens", C.c_int32),
                ("src", C.c_void_p)]


class HandoffSlot(C.Structure):
    _fields_ = [("batch_id", C.c_int64), ("new_stage", C.c_int32), ("resume_layer", C.c_int32),
                ("offset", C.c_uint64), ("bytes", C.c_uint64)]


class _CtlState(C.Structure):
    _fields_ = [("rounds", C.c_int32), ("barrier", C.c_int32), ("commit_scheduled", C.c_int32),
                ("waves", C.c_int32), ("kv_synced_bytes", C.c_double),
                ("last_wave_tokens", C.c_int64)]


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: the kvx CUDA library is the only implementation of this "
            "path (no CPU fallback). Build it with `python -m paper_2510_11938_b200.build`.")
    lib = C.CDLL(LIB_PATH)
    P, I32, I64, U64, VP = C.POINTER, C.c_int32, C.c_int64, C.c_uint64, C.c_void_p
    sig = {
        "kvx_last_error": (C.c_char_p, []),
        "kvx_abi_version": (C.c_int, []),
        "kvx_launch_count": (U64, []),
        "kvx_device_count": (C.c_int, [P(I32)]),
        "kvx_preload": (C.c_int, [I32]),
        "kvx_pool_create": (C.c_int, [I32, P(Geometry), I32, I32, P(VP)]),
        "kvx_pool_wrap": (C.c_int, [I32, VP, U64, P(Geometry), I32, I32, P(VP)]),
        "kvx_pool_export": (C.c_int, [VP, C.c_char_p]),
        "kvx_pool_import": (C.c_int, [I32, C.c_char_p, P(Geometry), I32, I32, P(VP)]),
        "kvx_pool_create_layout": (C.c_int, [I32, P(Geometry), I32, I32, I32, P(VP)]),
        "kvx_pool_import_layout": (C.c_int, [I32, C.c_char_p, P(Geometry), I32, I32, I32, P(VP)]),
        "kvx_pool_wrap_layers": (C.c_int, [I32, I32, P(VP), U64, P(Geometry), I32, I32, P(VP)]),
        "kvx_pool_layout": (C.c_int, [VP, P(I32)]),
        "kvx_pool_info": (C.c_int, [VP, P(VP), P(U64), P(I32), P(I32)]),
        "kvx_pool_destroy": (C.c_int, [VP]),
        "kvx_pool_zero": (C.c_int, [VP]),
        "kvx_pool_read": (C.c_int, [VP, U64, U64, VP]),
        "kvx_pool_write": (C.c_int, [VP, U64, U64, VP]),
        "kvx_pool_fill_pattern": (C.c_int, [VP, U64, I32, I32, P(I32), P(I64), P(I32), I32, I32]),
        "kvx_pool_append_pattern": (C.c_int, [VP, VP, U64, I32, I32, P(I32), P(I64), P(I64), P(I32), I32, I32]),
        "kvx_bm_create": (C.c_int, [I32, I32, P(VP)]),
        "kvx_bm_reset": (C.c_int, [VP]),
        "kvx_bm_free_count": (C.c_int, [VP, P(I32)]),
        "kvx_bm_pop": (C.c_int, [VP, I32, P(I32)]),
        "kvx_bm_push": (C.c_int, [VP, I32, P(I32)]),
        "kvx_bm_snapshot": (C.c_int, [VP, P(I32), P(I32)]),
        "kvx_bm_pop_async": (C.c_int, [VP, I32, VP, VP]),
        "kvx_bm_push_async": (C.c_int, [VP, I32, VP, VP]),
        "kvx_stage_kv_bytes": (C.c_int, [P(Geometry), I32, P(I32), I32, P(U64)]),
        "kvx_bm_destroy": (C.c_int, [VP]),
        "kvx_begin": (C.c_int, [P(_Desc), P(VP)]),
        "kvx_wave": (C.c_int, [VP, U64, I32, P(I32), P(I64), P(I64)]),
        "kvx_wait": (C.c_int, [VP, U64, P(C.c_double)]),
        "kvx_src_rows": (C.c_int, [VP, U64, I32, P(I32), P(I32)]),
        "kvx_commit": (C.c_int, [VP, U64, I32, P(I32), P(I64), P(_CommitResult)]),
        "kvx_abort": (C.c_int, [VP]),
        "kvx_destroy": (C.c_int, [VP]),
        "kvx_epoch": (C.c_int, [VP, P(U64)]),
        "kvx_dst_block_table": (C.c_int, [VP, P(I32)]),
        "kvx_stream": (C.c_int, [VP, P(VP)]),
        "kvx_bytes_moved": (C.c_int, [VP, P(U64)]),
        "kvx_move_timings": (C.c_int, [VP, I32, P(C.c_double), P(U64), P(I32)]),
        "kvx_verify_pattern": (C.c_int, [VP, U64, I32, P(I32), P(I64), P(I64)]),
        "kvx_handoff": (C.c_int, [VP, U64, U64, I32, P(MicroBatch), P(VP), P(U64), P(HandoffSlot)]),
        "kvx_weights_migrate": (C.c_int, [I32, VP, I32, U64, I32, P(I32), P(VP), I32, P(I32), P(VP),
                                          VP, P(C.c_uint8), P(U64), P(U64)]),
        "kvx_ctl_begin": (C.c_int, [VP, I32, P(I32), P(I64), P(I64)]),
        "kvx_ctl_sync_complete": (C.c_int, [VP, U64, I32, P(I32), P(I64), I32, P(I32), P(I64)]),
        "kvx_ctl_commit": (C.c_int, [VP, U64, I32, P(I32), P(I64), P(_CommitResult)]),
        "kvx_ctl_commit_async": (C.c_int, [VP, U64, I32, P(I32), P(I64)]),
        "kvx_ctl_commit_collect": (C.c_int, [VP, P(_CommitResult)]),
        "kvx_commit_async": (C.c_int, [VP, U64, I32, P(I32), P(I64)]),
        "kvx_commit_collect": (C.c_int, [VP, P(_CommitResult)]),
        "kvx_ctl_state_get": (C.c_int, [VP, P(_CtlState)]),
        "kvx_ctl_set_handoff": (C.c_int, [VP, I32]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = _load()
EXPORTED = tuple(n for n in dir(_lib) if n.startswith("kvx_"))


def lib() -> C.CDLL:
    return _lib


def _check(rc: int) -> None:
    if rc == KVX_OK:
        return
    msg = _lib.kvx_last_error().decode(errors="replace")
    cls = {KVX_ESTALE: StaleEpoch, KVX_ENOSPC: NoSpace}.get(rc, KvxError)
    raise cls(rc, msg)


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def _p32(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def _p64(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


def launch_count() -> int:
    return int(_lib.kvx_launch_count())


def device_count() -> int:
    n = C.c_int32(0)
    rc = _lib.kvx_device_count(C.byref(n))
    return int(n.value) if rc == KVX_OK else 0


def preload(device: int) -> None:
    """Loads every kvx kernel on `device` now (kvx_preload)."""
    _check(_lib.kvx_preload(device))


def geometry(num_layers: int, num_kv_heads: int, head_dim: int = 128, elem_bytes: int = 2,
             block_tokens: int = 16) -> Geometry:
    return Geometry(num_layers, num_kv_heads, head_dim, elem_bytes, block_tokens)


def stage_ranges(num_layers: int, boundaries: Sequence[int]) -> list:
    """stage_loads (engine.cpp:115-126): [(begin, end)] per stage."""
    cuts = [0, *boundaries, num_layers]
    return [(cuts[k], cuts[k + 1]) for k in range(len(cuts) - 1)]


class _Handle:
    """close() on scope exit: ``with kvx.Pool(...) as p: ...``."""

    def __enter__(self):
        return self

    def __exit__(self, *exc) -> None:
        self.close()


class Pool(_Handle):
    """One stage's paged KV pool on one GPU (local or imported from a peer)."""

    def __init__(self, device: int, geom: Geometry, num_layers: int, num_blocks: int,
                 layout: int = LAYOUT_BLOCKS, _handle: Optional[int] = None, imported: bool = False):
        self.geom, self.num_layers, self.num_blocks = geom, num_layers, num_blocks
        self.device, self.imported, self.layout = device, imported, layout
        if _handle is None:
            h = C.c_void_p()
            _check(_lib.kvx_pool_create_layout(device, C.byref(geom), num_layers, num_blocks, layout,
                                               C.byref(h)))
            self._h = h
        else:
            self._h = C.c_void_p(_handle)

    @classmethod
    def import_ipc(cls, device: int, handle: bytes, geom: Geometry, num_layers: int,
                   num_blocks: int, layout: int = LAYOUT_BLOCKS) -> "Pool":
        h = C.c_void_p()
        _check(_lib.kvx_pool_import_layout(device, handle, C.byref(geom), num_layers, num_blocks, layout,
                                           C.byref(h)))
        return cls(device, geom, num_layers, num_blocks, layout, _handle=h.value, imported=True)

    @classmethod
    def wrap_layers(cls, device: int, layer_ptrs: Sequence[int], layer_bytes: int, geom: Geometry,
                    num_blocks: int, layout: int = LAYOUT_KV_PLANES) -> "Pool":
        """A pool over one caller-owned allocation per layer (e.g. a serving
        engine's per-layer cache tensors, data_ptr() each)."""
        ptrs = (C.c_void_p * len(layer_ptrs))(*layer_ptrs)
        h = C.c_void_p()
        _check(_lib.kvx_pool_wrap_layers(device, len(layer_ptrs), ptrs, layer_bytes, C.byref(geom), num_blocks,
                                         layout, C.byref(h)))
        return cls(device, geom, len(layer_ptrs), num_blocks, layout, _handle=h.value)

    @classmethod
    def wrap(cls, device: int, ptr: int, nbytes: int, geom: Geometry, num_layers: int,
             num_blocks: int) -> "Pool":
        """A pool over caller-owned device memory (e.g. a torch tensor's data_ptr())."""
        h = C.c_void_p()
        _check(_lib.kvx_pool_wrap(device, ptr, nbytes, C.byref(geom), num_layers, num_blocks, C.byref(h)))
        return cls(device, geom, num_layers, num_blocks, LAYOUT_BLOCKS, _handle=h.value)

    def export_ipc(self) -> bytes:
        buf = C.create_string_buffer(IPC_HANDLE_BYTES)
        _check(_lib.kvx_pool_export(self._h, buf))
        return buf.raw

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    @property
    def nbytes(self) -> int:
        return self.num_layers * self.num_blocks * self.geom.block_bytes

    @property
    def ptr(self) -> int:
        """Device address of the pool (local, or this process's peer mapping)."""
        d = C.c_void_p()
        _check(_lib.kvx_pool_info(self._h, C.byref(d), None, None, None))
        return int(d.value or 0)

    def zero(self) -> None:
        _check(_lib.kvx_pool_zero(self._h))

    def read(self, offset: int = 0, nbytes: Optional[int] = None) -> np.ndarray:
        nbytes = self.nbytes - offset if nbytes is None else nbytes
        out = np.empty(nbytes, dtype=np.uint8)
        _check(_lib.kvx_pool_read(self._h, offset, nbytes, out.ctypes.data_as(C.c_void_p)))
        return out

    def write(self, data: np.ndarray, offset: int = 0) -> None:
        data = np.ascontiguousarray(data).view(np.uint8)
        _check(_lib.kvx_pool_write(self._h, offset, data.nbytes, data.ctypes.data_as(C.c_void_p)))

    def fill_pattern(self, seed: int, first_layer: int, req, tokens, block_table: np.ndarray) -> None:
        req, tokens = _i32(req), _i64(tokens)
        bt = _i32(block_table)
        _check(_lib.kvx_pool_fill_pattern(self._h, seed, first_layer, len(req), _p32(req),
                                          _p64(tokens), _p32(bt), bt.shape[0], bt.shape[1]))

    def append_pattern(self, seed: int, first_layer: int, req, frm, to, block_table: np.ndarray,
                       stream: int = 0) -> None:
        """Decode appends [frm, to) per request, asynchronous on `stream`."""
        req, frm, to = _i32(req), _i64(frm), _i64(to)
        bt = _i32(block_table)
        _check(_lib.kvx_pool_append_pattern(self._h, stream or None, seed, first_layer, len(req), _p32(req),
                                            _p64(frm), _p64(to), _p32(bt), bt.shape[0], bt.shape[1]))

    def close(self) -> None:
        if self._h is not None and self._h.value:
            _check(_lib.kvx_pool_destroy(self._h))
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class BlockManager(_Handle):
    """Device-resident free list of one pool set (kvx_bm_*)."""

    def __init__(self, device: int, capacity: int):
        h = C.c_void_p()
        _check(_lib.kvx_bm_create(device, capacity, C.byref(h)))
        self._h, self.capacity = h, capacity

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def free_count(self) -> int:
        n = C.c_int32()
        _check(_lib.kvx_bm_free_count(self._h, C.byref(n)))
        return int(n.value)

    def reset(self) -> None:
        _check(_lib.kvx_bm_reset(self._h))

    def pop(self, n: int) -> np.ndarray:
        out = np.zeros(max(n, 1), np.int32)
        _check(_lib.kvx_bm_pop(self._h, n, _p32(out)))
        return out[:n]

    def push(self, ids) -> None:
        ids = _i32(ids)
        _check(_lib.kvx_bm_push(self._h, len(ids), _p32(ids)))

    def pop_async(self, n: int, dev_ids_out: int, stream: int = 0) -> None:
        """Pop n ids into a device int32 array on `stream` (no host sync)."""
        _check(_lib.kvx_bm_pop_async(self._h, n, dev_ids_out or None, stream or None))

    def push_async(self, n: int, dev_ids: int, stream: int = 0) -> None:
        """Push n ids from a device int32 array on `stream` (no host sync)."""
        _check(_lib.kvx_bm_push_async(self._h, n, dev_ids or None, stream or None))

    def snapshot(self) -> np.ndarray:
        out = np.zeros(self.capacity, np.int32)
        top = C.c_int32()
        _check(_lib.kvx_bm_snapshot(self._h, _p32(out), C.byref(top)))
        return out[:top.value].copy()

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            _check(_lib.kvx_bm_destroy(self._h))
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class CommitResult:
    violations: int
    row_ptr: np.ndarray
    blocks: np.ndarray
    free_list: np.ndarray


class Transition(_Handle):
    """One inflight refactor of one pipeline instance (RefactorCtx,
    engine.hpp:149-158), on one local GPU."""

    def __init__(self, geom: Geometry, old_boundaries: Sequence[int], old_pools: Sequence[Optional[Pool]],
                 new_boundaries: Sequence[int], new_pools: Sequence[Pool], device: int,
                 max_requests: int, max_blocks: int, dst_num_blocks: int,
                 src_block_table: np.ndarray, epoch: int = 1, max_sync_rounds: int = 8,
                 kv_bytes_per_token: float = 0.0, stream: int = 0,
                 dst_blockmgr: Optional["BlockManager"] = None, pull: bool = False,
                 layer_pull: Optional[Sequence[int]] = None, max_ctas: int = 0,
                 src_block_table_dev: int = 0):
        self.geom = geom
        self.max_requests, self.max_blocks = max_requests, max_blocks
        self._ob = _i32(list(old_boundaries))
        self._nb = _i32(list(new_boundaries))
        self._old = list(old_pools)
        self._new = list(new_pools)
        self._op = (C.c_void_p * len(self._old))(*[p.handle.value if p else None for p in self._old])
        self._np = (C.c_void_p * len(self._new))(*[p.handle.value if p else None for p in self._new])
        # src_block_table_dev: device pointer of the same [max_requests, max_blocks]
        # int32 table (the serving engine's copy); the host table may then be None
        src = None if src_block_table is None else _i32(src_block_table)
        if src is None and not src_block_table_dev:
            raise ValueError("a source block table (host or device) is required")
        if src is not None and src.shape != (max_requests, max_blocks):
            raise ValueError("src_block_table must be [max_requests, max_blocks]")
        d = _Desc()
        d.geometry = geom
        d.old_plan = _Plan(len(self._old), _p32(self._ob), C.cast(self._op, C.POINTER(C.c_void_p)))
        d.new_plan = _Plan(len(self._new), _p32(self._nb), C.cast(self._np, C.POINTER(C.c_void_p)))
        d.device = device
        d.max_requests, d.max_blocks, d.dst_num_blocks = max_requests, max_blocks, dst_num_blocks
        d.src_block_table = _p32(src) if src is not None else None
        if src_block_table_dev:
            d.src_block_table_dev = C.cast(C.c_void_p(src_block_table_dev), C.POINTER(C.c_int32))
        d.epoch = epoch
        d.max_sync_rounds = max_sync_rounds
        d.kv_bytes_per_token = kv_bytes_per_token
        d.stream = stream or None
        d.dst_blockmgr = dst_blockmgr.handle.value if dst_blockmgr is not None else None
        self._bm = dst_blockmgr
        d.pull = 1 if pull else 0
        d.max_ctas = max_ctas
        if layer_pull is not None:   # per layer: 1 = destination pulls, 0 = source pushes
            self._layer_pull = np.ascontiguousarray(layer_pull, dtype=np.uint8)
            if self._layer_pull.shape != (geom.num_layers,):
                raise ValueError("layer_pull needs one entry per layer")
            d.layer_pull = self._layer_pull.ctypes.data_as(C.POINTER(C.c_uint8))
        h = C.c_void_p()
        _check(_lib.kvx_begin(C.byref(d), C.byref(h)))
        self._h = h

    # ------------------------------------------------------------ data plane
    @property
    def epoch(self) -> int:
        e = C.c_uint64()
        _check(_lib.kvx_epoch(self._h, C.byref(e)))
        return int(e.value)

    def wave(self, req, lo, hi, epoch: Optional[int] = None) -> None:
        req, lo, hi = _i32(req), _i64(lo), _i64(hi)
        _check(_lib.kvx_wave(self._h, self.epoch if epoch is None else epoch, len(req), _p32(req),
                             _p64(lo), _p64(hi)))

    def src_rows(self, req, rows, epoch: Optional[int] = None) -> None:
        """kvx_src_rows: replace source-table rows of `req` ([n, max_blocks])."""
        req = _i32(req)
        rows = np.ascontiguousarray(rows, dtype=np.int32).reshape(len(req), self.max_blocks)
        _check(_lib.kvx_src_rows(self._h, self.epoch if epoch is None else epoch, len(req), _p32(req), _p32(rows)))

    def wait(self, epoch: Optional[int] = None) -> float:
        ms = C.c_double()
        _check(_lib.kvx_wait(self._h, self.epoch if epoch is None else epoch, C.byref(ms)))
        return float(ms.value)

    def _commit_buffers(self, n: int):
        cap = self.max_requests * self.max_blocks
        row_ptr = np.zeros(n + 1, dtype=np.int32)
        blocks = np.zeros(max(cap, 1), dtype=np.int32)
        free = np.zeros(max(cap, 1), dtype=np.int32)
        res = _CommitResult(0, _p32(row_ptr), _p32(blocks), len(blocks), 0, _p32(free), len(free), 0)
        return res, row_ptr, blocks, free

    def commit(self, req, kv, epoch: Optional[int] = None) -> CommitResult:
        req, kv = _i32(req), _i64(kv)
        res, row_ptr, blocks, free = self._commit_buffers(len(req))
        _check(_lib.kvx_commit(self._h, self.epoch if epoch is None else epoch, len(req), _p32(req),
                               _p64(kv), C.byref(res)))
        return CommitResult(int(res.violations), row_ptr, blocks[:res.n_blocks].copy(),
                            free[:res.n_free].copy())

    def abort(self) -> None:
        _check(_lib.kvx_abort(self._h))

    def dst_block_table(self) -> np.ndarray:
        out = np.empty((self.max_requests, self.max_blocks), dtype=np.int32)
        _check(_lib.kvx_dst_block_table(self._h, _p32(out)))
        return out

    def stream_ptr(self) -> int:
        s = C.c_void_p()
        _check(_lib.kvx_stream(self._h, C.byref(s)))
        return int(s.value or 0)

    def move_timings(self) -> list:
        """[(ms, read+write bytes)] of every move-kernel launch, wave order."""
        n = C.c_int32()
        _check(_lib.kvx_move_timings(self._h, 0, None, None, C.byref(n)))
        ms = (C.c_double * max(n.value, 1))()
        b = (C.c_uint64 * max(n.value, 1))()
        _check(_lib.kvx_move_timings(self._h, n.value, ms, b, C.byref(n)))
        return [(float(ms[i]), int(b[i])) for i in range(n.value)]

    def bytes_moved(self) -> int:
        b = C.c_uint64()
        _check(_lib.kvx_bytes_moved(self._h, C.byref(b)))
        return int(b.value)

    def verify_pattern(self, seed: int, req, kv) -> int:
        req, kv = _i32(req), _i64(kv)
        bad = C.c_int64()
        _check(_lib.kvx_verify_pattern(self._h, seed, len(req), _p32(req), _p64(kv), C.byref(bad)))
        return int(bad.value)

    def handoff(self, row_bytes: int, batches, arenas, arena_bytes, epoch: Optional[int] = None):
        """Stage-boundary activation handoff.  batches: [(batch_id, after_stage,
        tokens, src_device_ptr)]; arenas: per-new-stage device pointers.
        Returns [(batch_id, new_stage, resume_layer, offset, bytes)]."""
        n = len(batches)
        mb = (MicroBatch * max(n, 1))(*[MicroBatch(int(b), int(a), int(tk), int(p) or None)
                                        for b, a, tk, p in batches])
        ar = (C.c_void_p * len(arenas))(*[int(a) or None for a in arenas])
        cap = (C.c_uint64 * len(arena_bytes))(*[int(x) for x in arena_bytes])
        out = (HandoffSlot * max(n, 1))()
        _check(_lib.kvx_handoff(self._h, self.epoch if epoch is None else epoch, row_bytes, n, mb,
                                ar, cap, out))
        return [(out[i].batch_id, out[i].new_stage, out[i].resume_layer, out[i].offset, out[i].bytes)
                for i in range(n)]

    # --------------------------------------------- reference-shaped handlers
    def begin_refactor(self, live: Tuple[np.ndarray, np.ndarray]) -> int:
        """Wave 0 over every live token (engine.cpp:637-647); returns tokens."""
        req, kv = _i32(live[0]), _i64(live[1])
        tok = C.c_int64()
        _check(_lib.kvx_ctl_begin(self._h, len(req), _p32(req), _p64(kv), C.byref(tok)))
        return int(tok.value)

    def on_kv_sync_complete(self, live, inflight_batches: int = 0,
                            epoch: Optional[int] = None) -> Tuple[int, int]:
        """engine.cpp:651-688 -> (action, tokens of the wave issued)."""
        req, kv = _i32(live[0]), _i64(live[1])
        act, tok = C.c_int32(), C.c_int64()
        _check(_lib.kvx_ctl_sync_complete(self._h, self.epoch if epoch is None else epoch, len(req),
                                          _p32(req), _p64(kv), inflight_batches, C.byref(act),
                                          C.byref(tok)))
        return int(act.value), int(tok.value)

    def on_refactor_commit(self, live, epoch: Optional[int] = None,
                           wait: bool = True) -> Optional[CommitResult]:
        """engine.cpp:690-713: final apply, Eq. 10 on the device, compaction.
        wait=False returns at once (kvx_ctl_commit_async); collect_commit()
        then returns the result."""
        req, kv = _i32(live[0]), _i64(live[1])
        _check(_lib.kvx_ctl_commit_async(self._h, self.epoch if epoch is None else epoch, len(req),
                                         _p32(req), _p64(kv)))
        self._pending_live = len(req)
        return self.collect_commit() if wait else None

    def collect_commit(self) -> CommitResult:
        res, row_ptr, blocks, free = self._commit_buffers(self._pending_live)
        _check(_lib.kvx_ctl_commit_collect(self._h, C.byref(res)))
        return CommitResult(int(res.violations), row_ptr, blocks[:res.n_blocks].copy(),
                            free[:res.n_free].copy())

    def abort_refactor(self) -> None:
        """engine.cpp:759-772."""
        self.abort()

    def set_handoff(self, enable: bool = True) -> None:
        """Hand in-flight micro-batches off at the barrier instead of draining."""
        _check(_lib.kvx_ctl_set_handoff(self._h, 1 if enable else 0))

    def ctl_state(self) -> dict:
        s = _CtlState()
        _check(_lib.kvx_ctl_state_get(self._h, C.byref(s)))
        return {f: getattr(s, f) for f, _ in _CtlState._fields_}

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            _check(_lib.kvx_destroy(self._h))
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def stage_kv_bytes(geom: Geometry, boundaries, dst_num_blocks: int) -> List[int]:
    """kvx_stage_kv_bytes: device KV bytes each new stage holds for a grant."""
    b = _i32(list(boundaries))
    out = (C.c_uint64 * (len(b) + 1))()
    _check(_lib.kvx_stage_kv_bytes(C.byref(geom), len(b) + 1, _p32(b), dst_num_blocks, out))
    return [int(x) for x in out]


def weights_migrate(device: int, num_layers: int, layer_bytes: int, old_boundaries, old_ptrs,
                    new_boundaries, new_ptrs, stream: int = 0, host_cache: int = 0,
                    from_host=None) -> Tuple[int, int]:
    """Stage weight migration (kvx_weights_migrate): returns (device bytes,
    host-tier bytes) scheduled on `stream`."""
    ob, nb = _i32(list(old_boundaries)), _i32(list(new_boundaries))
    op = (C.c_void_p * len(old_ptrs))(*[int(p) or None for p in old_ptrs])
    np_ = (C.c_void_p * len(new_ptrs))(*[int(p) or None for p in new_ptrs])
    fh = None
    if from_host is not None:
        fh_arr = np.ascontiguousarray(from_host, dtype=np.uint8)
        fh = fh_arr.ctypes.data_as(C.POINTER(C.c_uint8))
    db, hb = C.c_uint64(), C.c_uint64()
    _check(_lib.kvx_weights_migrate(device, stream or None, num_layers, layer_bytes, len(ob) + 1, _p32(ob),
                                    op, len(nb) + 1, _p32(nb), np_, host_cache or None, fh,
                                    C.byref(db), C.byref(hb)))
    return int(db.value), int(hb.value)
