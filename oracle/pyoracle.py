"""ctypes face of oracle/_build/libkvx_oracle.so (oracle/kvx_oracle.c).

TEST INFRASTRUCTURE ONLY: the checker, never the thing measured or shipped.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libkvx_oracle.so")

ACT_DELTA, ACT_BARRIER_WAIT, ACT_FINAL = 0, 1, 2


def build() -> str:
    """Compiles the C restatement (gcc) if the .so is missing or stale."""
    src = [os.path.join(HERE, f) for f in ("kvx_oracle.c", "kvx_oracle.h")]
    if not os.path.exists(LIB_PATH) or any(os.path.getmtime(s) > os.path.getmtime(LIB_PATH) for s in src):
        subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    return LIB_PATH


class Geo(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("num_kv_heads", C.c_int32), ("head_dim", C.c_int32),
                ("elem_bytes", C.c_int32), ("block_tokens", C.c_int32)]


class Ctx(C.Structure):
    _fields_ = [("max_requests", C.c_int32), ("synced", C.POINTER(C.c_int64)),
                ("target", C.POINTER(C.c_int64)), ("in_target", C.POINTER(C.c_uint8)),
                ("rounds", C.c_int32), ("barrier", C.c_int32), ("commit_scheduled", C.c_int32),
                ("max_sync_rounds", C.c_int32), ("kv_bytes_per_token", C.c_double),
                ("kv_synced_bytes", C.POINTER(C.c_double))]


class Dst(C.Structure):
    _fields_ = [("max_requests", C.c_int32), ("max_blocks", C.c_int32), ("num_blocks", C.c_int32),
                ("next_block", C.c_int32), ("bt", C.POINTER(C.c_int32)),
                ("synced_hi", C.POINTER(C.c_int64)), ("stack", C.POINTER(C.c_int32)),
                ("top", C.c_int32)]


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P, I32, I64, U8, U64, VP = C.POINTER, C.c_int32, C.c_int64, C.c_uint8, C.c_uint64, C.c_void_p
        PP = C.POINTER(C.c_void_p)
        sig = {
            "kvo_token_hash": (U64, [U64, I32, I32, I32, I64]),
            "kvo_word": (C.c_uint16, [U64, C.c_uint32]),
            "kvo_stage_of_layer": (I32, [I32, P(I32), I32]),
            "kvo_ctx_snapshot": (I64, [P(Ctx), I32, P(I32), P(I64), P(I64), P(I64)]),
            "kvo_ctx_unsynced": (I64, [P(Ctx), I32, P(I32), P(I64)]),
            "kvo_ctx_apply": (None, [P(Ctx)]),
            "kvo_ctx_violations": (I64, [P(Ctx), I32, P(I32), P(I64)]),
            "kvo_ctx_begin": (I64, [P(Ctx), I32, P(I32), P(I64), P(I64), P(I64)]),
            "kvo_ctx_on_sync_complete": (I32, [P(Ctx), I32, P(I32), P(I64), I32, P(I64), P(I64), P(I64)]),
            "kvo_fill": (None, [P(Geo), U64, I32, P(I32), PP, I32, I32, P(I32), P(I64), P(I32), I32]),
            "kvo_fill_layer": (None, [P(Geo), U64, I32, VP, I32, I32, P(I32), P(I64), P(I32), I32, I32]),
            "kvo_apply_wave": (C.c_int, [P(Geo), P(Dst), I32, P(I32), PP, I32, P(I32), I32, P(I32), PP,
                                         I32, P(I32), P(I64), P(I64)]),
            "kvo_apply_wave_mt": (C.c_int, [P(Geo), P(Dst), I32, P(I32), PP, I32, P(I32), I32, P(I32), PP,
                                            I32, P(I32), P(I64), P(I64), I32]),
            "kvo_commit": (I64, [P(Geo), P(Dst), I32, P(I32), P(I64), P(I32), P(I32), P(I32), P(I32), P(I32)]),
            "kvo_verify": (I64, [P(Geo), U64, P(Dst), I32, P(I32), PP, I32, P(I32), P(I64)]),
            "kvo_activation_owner": (I32, [I32, P(I32), I32, P(I32), I32]),
            "kvo_bm_init": (None, [P(I32), I32]),
            "kvo_abort": (None, [P(Geo), P(Dst)]),
            "kvo_weights_plan": (None, [I32, U64, I32, P(I32), I32, P(I32), P(I32), P(U64), P(I32), P(U64)]),
            "kvo_warm_start_ms": (C.c_double, [I32, P(C.c_double), P(C.c_uint8), C.c_double, C.c_double]),
            "kvo_handoff_plan": (C.c_int, [I32, P(I32), I32, P(I32), U64, I32, P(I32), P(I32), P(U64),
                                           P(I32), P(I32), P(U64), P(U64)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(_lib, name)
            fn.restype = res
            fn.argtypes = args
    return _lib


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def _pp(arrs):
    if arrs is None:
        return None
    return (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])


def geo(num_layers, num_kv_heads, head_dim, elem_bytes=2, block_tokens=16) -> Geo:
    return Geo(num_layers, num_kv_heads, head_dim, elem_bytes, block_tokens)


class ControlCtx:
    """RefactorCtx restated (kvo_ctx_*), engine.cpp:534-713."""

    def __init__(self, max_requests: int, max_sync_rounds: int, kv_bytes_per_token: float,
                 accumulator: Optional[np.ndarray] = None):
        self.synced = np.zeros(max_requests, np.int64)
        self.target = np.zeros(max_requests, np.int64)
        self.in_target = np.zeros(max_requests, np.uint8)
        self.acc = accumulator if accumulator is not None else np.zeros(1, np.float64)
        self.c = Ctx(max_requests, _p(self.synced, C.c_int64), _p(self.target, C.c_int64),
                     _p(self.in_target, C.c_uint8), 0, 0, 0, max_sync_rounds, kv_bytes_per_token,
                     _p(self.acc, C.c_double))

    def begin(self, req, kv):
        req, kv = _i32(req), _i64(kv)
        lo, hi = np.zeros(len(req), np.int64), np.zeros(len(req), np.int64)
        tok = lib().kvo_ctx_begin(C.byref(self.c), len(req), _p(req, C.c_int32), _p(kv, C.c_int64),
                                  _p(lo, C.c_int64), _p(hi, C.c_int64))
        return int(tok), lo, hi

    def on_sync_complete(self, req, kv, inflight: int):
        req, kv = _i32(req), _i64(kv)
        lo, hi = np.zeros(len(req), np.int64), np.zeros(len(req), np.int64)
        tok = C.c_int64()
        act = lib().kvo_ctx_on_sync_complete(C.byref(self.c), len(req), _p(req, C.c_int32),
                                             _p(kv, C.c_int64), inflight, _p(lo, C.c_int64),
                                             _p(hi, C.c_int64), C.byref(tok))
        return int(act), int(tok.value), lo, hi

    def snapshot(self, req, kv):
        req, kv = _i32(req), _i64(kv)
        lo, hi = np.zeros(len(req), np.int64), np.zeros(len(req), np.int64)
        tok = lib().kvo_ctx_snapshot(C.byref(self.c), len(req), _p(req, C.c_int32), _p(kv, C.c_int64),
                                     _p(lo, C.c_int64), _p(hi, C.c_int64))
        return int(tok), lo, hi

    def apply(self):
        lib().kvo_ctx_apply(C.byref(self.c))

    def violations(self, req, kv) -> int:
        req, kv = _i32(req), _i64(kv)
        return int(lib().kvo_ctx_violations(C.byref(self.c), len(req), _p(req, C.c_int32), _p(kv, C.c_int64)))

    @property
    def kv_synced_bytes(self) -> float:
        return float(self.acc[0])

    @property
    def rounds(self) -> int:
        return int(self.c.rounds)


def stage_layers(num_layers: int, boundaries: Sequence[int]):
    cuts = [0, *boundaries, num_layers]
    return [cuts[k + 1] - cuts[k] for k in range(len(cuts) - 1)]


class DataPlane:
    """Host pools + destination state of one transition (kvo_* data plane)."""

    def __init__(self, g: Geo, old_b, new_b, old_blocks: int, new_blocks: int, max_requests: int,
                 max_blocks: int, src_bt: np.ndarray, with_pools: bool = True,
                 bm: Optional["StackBM"] = None, old_pools=None, new_pools=None):
        self.g = g
        self.ob, self.nb = _i32(list(old_b)), _i32(list(new_b))
        self.old_blocks, self.new_blocks = old_blocks, new_blocks
        self.max_requests, self.max_blocks = max_requests, max_blocks
        self.src_bt = _i32(src_bt)
        bb = 2 * g.block_tokens * g.num_kv_heads * g.head_dim * g.elem_bytes
        self.old_pools = self.new_pools = None
        if with_pools:
            self.old_pools = old_pools if old_pools is not None else \
                [np.zeros(n * old_blocks * bb, np.uint8) for n in stage_layers(g.num_layers, old_b)]
            self.new_pools = new_pools if new_pools is not None else \
                [np.zeros(n * new_blocks * bb, np.uint8) for n in stage_layers(g.num_layers, new_b)]
        self.bt = np.full((max_requests, max_blocks), -1, np.int32)
        self.synced_hi = np.zeros(max_requests, np.int64)
        self.bm = bm  # block-manager restatement (its stack is mutated in place) or None
        self.d = Dst(max_requests, max_blocks, new_blocks, 0, _p(self.bt, C.c_int32),
                     _p(self.synced_hi, C.c_int64),
                     _p(bm.stack, C.c_int32) if bm is not None else None, 0)

    def _enter(self):
        if self.bm is not None:
            self.d.top = self.bm.top

    def _leave(self):
        if self.bm is not None:
            self.bm.top = int(self.d.top)

    def abort(self):
        self._enter()
        lib().kvo_abort(C.byref(self.g), C.byref(self.d))
        self._leave()

    def fill_source(self, seed: int, req, tokens):
        req, tokens = _i32(req), _i64(tokens)
        lib().kvo_fill(C.byref(self.g), seed, len(self.ob) + 1, _p(self.ob, C.c_int32),
                       _pp(self.old_pools), self.old_blocks, len(req), _p(req, C.c_int32),
                       _p(tokens, C.c_int64), _p(self.src_bt, C.c_int32), self.max_blocks)

    def wave(self, req, lo, hi, threads: int = 0) -> int:
        req, lo, hi = _i32(req), _i64(lo), _i64(hi)
        args = (C.byref(self.g), C.byref(self.d), len(self.ob) + 1, _p(self.ob, C.c_int32),
                _pp(self.old_pools), self.old_blocks, _p(self.src_bt, C.c_int32), len(self.nb) + 1,
                _p(self.nb, C.c_int32), _pp(self.new_pools), len(req), _p(req, C.c_int32),
                _p(lo, C.c_int64), _p(hi, C.c_int64))
        self._enter()
        try:
            if threads > 0:
                return lib().kvo_apply_wave_mt(*args, threads)
            return lib().kvo_apply_wave(*args)
        finally:
            self._leave()

    def commit(self, req, kv):
        req, kv = _i32(req), _i64(kv)
        cap = self.max_requests * self.max_blocks
        row_ptr = np.zeros(len(req) + 1, np.int32)
        blocks = np.zeros(max(cap, 1), np.int32)
        free = np.zeros(max(cap, 1), np.int32)
        nb, nf = C.c_int32(), C.c_int32()
        self._enter()
        v = lib().kvo_commit(C.byref(self.g), C.byref(self.d), len(req), _p(req, C.c_int32),
                             _p(kv, C.c_int64), _p(row_ptr, C.c_int32), _p(blocks, C.c_int32),
                             C.byref(nb), _p(free, C.c_int32), C.byref(nf))
        self._leave()
        return int(v), row_ptr, blocks[:nb.value].copy(), free[:nf.value].copy()

    def verify(self, seed: int, req, kv) -> int:
        req, kv = _i32(req), _i64(kv)
        return int(lib().kvo_verify(C.byref(self.g), seed, C.byref(self.d), len(self.nb) + 1,
                                    _p(self.nb, C.c_int32), _pp(self.new_pools), len(req),
                                    _p(req, C.c_int32), _p(kv, C.c_int64)))


def fill_layer(g: Geo, seed: int, layer: int, blocks_per_pool: int, req, tokens, bt: np.ndarray,
               out: Optional[np.ndarray] = None, threads: int = 0) -> np.ndarray:
    """kvo_fill_layer: the expected block-layout image of model layer `layer`
    of a pool with blocks_per_pool blocks, rows [0, tokens[i]) of req[i]
    through bt ([max_requests, max_blocks]), zeros elsewhere."""
    req, tokens, bt = _i32(req), _i64(tokens), _i32(bt)
    bb = 2 * g.block_tokens * g.num_kv_heads * g.head_dim * g.elem_bytes
    if out is None:
        out = np.empty(blocks_per_pool * bb, np.uint8)
    assert out.nbytes == blocks_per_pool * bb and out.flags.c_contiguous
    lib().kvo_fill_layer(C.byref(g), seed, layer, out.ctypes.data, blocks_per_pool, len(req),
                         _p(req, C.c_int32), _p(tokens, C.c_int64), _p(bt, C.c_int32), bt.shape[-1],
                         threads if threads > 0 else (os.cpu_count() or 1))
    return out


def activation_owner(old_b, new_b, from_old_stage: int) -> int:
    ob, nb = _i32(list(old_b)), _i32(list(new_b))
    return int(lib().kvo_activation_owner(len(ob) + 1, _p(ob, C.c_int32), len(nb) + 1,
                                          _p(nb, C.c_int32), from_old_stage))


def handoff_plan(old_b, new_b, row_bytes: int, after, tokens, arena_bytes):
    """kvo_handoff_plan -> (rc, new_stage, resume_layer, offset, bytes)."""
    ob, nb = _i32(list(old_b)), _i32(list(new_b))
    after, tokens = _i32(after), _i32(tokens)
    cap = np.ascontiguousarray(arena_bytes, dtype=np.uint64)
    n = len(after)
    ns, rl = np.zeros(n, np.int32), np.zeros(n, np.int32)
    off, by = np.zeros(n, np.uint64), np.zeros(n, np.uint64)
    rc = lib().kvo_handoff_plan(len(ob) + 1, _p(ob, C.c_int32), len(nb) + 1, _p(nb, C.c_int32),
                                row_bytes, n, _p(after, C.c_int32), _p(tokens, C.c_int32),
                                _p(cap, C.c_uint64), _p(ns, C.c_int32), _p(rl, C.c_int32),
                                _p(off, C.c_uint64), _p(by, C.c_uint64))
    return int(rc), ns, rl, off, by


def weights_plan(num_layers, layer_bytes, old_b, new_b):
    ob, nb = _i32(list(old_b)), _i32(list(new_b))
    ss, ds = np.zeros(num_layers, np.int32), np.zeros(num_layers, np.int32)
    so, do = np.zeros(num_layers, np.uint64), np.zeros(num_layers, np.uint64)
    lib().kvo_weights_plan(num_layers, layer_bytes, len(ob) + 1, _p(ob, C.c_int32), len(nb) + 1,
                           _p(nb, C.c_int32), _p(ss, C.c_int32), _p(so, C.c_uint64),
                           _p(ds, C.c_int32), _p(do, C.c_uint64))
    return ss, so, ds, do


def warm_start_ms(stage_bytes, cached, host_bw, storage_bw) -> float:
    b = np.ascontiguousarray(stage_bytes, dtype=np.float64)
    c = np.ascontiguousarray(cached, dtype=np.uint8)
    return float(lib().kvo_warm_start_ms(len(b), _p(b, C.c_double), _p(c, C.c_uint8), host_bw, storage_bw))


class StackBM:
    """Host restatement of the device block manager: a numpy free stack and
    its top (kvo_bm_init order: pops yield 0, 1, 2, ...)."""

    def __init__(self, capacity: int):
        self.stack = np.zeros(capacity, np.int32)
        self.capacity = capacity
        self.reset()

    def reset(self):
        lib().kvo_bm_init(_p(self.stack, C.c_int32), self.capacity)
        self.top = self.capacity

    def pop(self, n: int) -> np.ndarray:
        assert n <= self.top
        out = self.stack[self.top - n:self.top][::-1].copy()
        self.top -= n
        return out

    def push(self, ids) -> None:
        ids = np.asarray(ids, np.int32)
        self.stack[self.top:self.top + len(ids)] = ids
        self.top += len(ids)

    def snapshot(self) -> np.ndarray:
        return self.stack[:self.top].copy()
