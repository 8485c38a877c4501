"""C-ABI argument validation (CPU): malformed descriptors and arrays are
rejected with KVX_EINVAL (or KVX_ESTALE/ESTATE) before any CUDA call, never
by a crash -- the boundary never throws and never dereferences NULL."""
import ctypes as C

import numpy as np
import pytest

from paper_2510_11938_b200 import kvx

L = kvx.lib()


def desc(**over):
    d = kvx._Desc()
    d.geometry = kvx.geometry(4, 2, 64)
    ob = (C.c_int32 * 1)(2)
    nb = (C.c_int32 * 1)(1)
    pools = (C.c_void_p * 2)(None, None)
    d.old_plan = kvx._Plan(2, ob, C.cast(pools, C.POINTER(C.c_void_p)))
    d.new_plan = kvx._Plan(2, nb, C.cast(pools, C.POINTER(C.c_void_p)))
    d.max_requests, d.max_blocks, d.dst_num_blocks = 4, 4, 16
    bt = (C.c_int32 * 16)(*([-1] * 16))
    d.src_block_table = C.cast(bt, C.POINTER(C.c_int32))
    d.epoch = 1
    keep = (ob, nb, pools, bt)
    for k, v in over.items():
        setattr(d, k, v)
    return d, keep


def begin_rc(d):
    h = C.c_void_p()
    return L.kvx_begin(C.byref(d), C.byref(h))


def test_null_arguments():
    h = C.c_void_p()
    assert L.kvx_begin(None, C.byref(h)) == kvx.KVX_EINVAL
    assert L.kvx_wave(None, 1, 0, None, None, None) == kvx.KVX_EINVAL
    assert L.kvx_wait(None, 1, None) == kvx.KVX_EINVAL
    assert L.kvx_commit(None, 1, 0, None, None, None) == kvx.KVX_EINVAL
    assert L.kvx_abort(None) == kvx.KVX_EINVAL
    assert L.kvx_destroy(None) == kvx.KVX_OK
    assert L.kvx_pool_destroy(None) == kvx.KVX_OK
    assert L.kvx_bm_destroy(None) == kvx.KVX_OK
    assert L.kvx_handoff(None, 1, 16, 0, None, None, None, None) == kvx.KVX_EINVAL
    assert L.kvx_ctl_begin(None, 0, None, None, None) == kvx.KVX_EINVAL


@pytest.mark.parametrize("field,value", [
    ("max_requests", 0), ("max_blocks", 0), ("dst_num_blocks", 0),
])
def test_bad_sizes(field, value):
    d, keep = desc(**{field: value})
    assert begin_rc(d) == kvx.KVX_EINVAL


def test_bad_geometry_and_plans():
    d, keep = desc()
    d.geometry = kvx.geometry(4, 1, 4)           # token_bytes 8: not a 16-byte multiple
    assert begin_rc(d) == kvx.KVX_EINVAL
    d, keep = desc()
    bad = (C.c_int32 * 1)(4)                      # boundary == L
    d.old_plan = kvx._Plan(2, bad, d.old_plan.pools)
    assert begin_rc(d) == kvx.KVX_EINVAL
    d, keep = desc()
    d.new_plan = kvx._Plan(9, d.new_plan.boundaries, d.new_plan.pools)  # more stages than layers
    assert begin_rc(d) == kvx.KVX_EINVAL
    d, keep = desc()
    d.src_block_table = None
    assert begin_rc(d) == kvx.KVX_EINVAL


def test_missing_new_pool_rejected_in_push_mode():
    d, keep = desc()                               # new_plan pools are NULL
    assert begin_rc(d) == kvx.KVX_EINVAL
    assert b"new-stage pool" in L.kvx_last_error()


def test_negative_max_ctas_rejected():
    d, keep = desc(max_ctas=-1)
    assert begin_rc(d) == kvx.KVX_EINVAL


def test_error_message_is_thread_local_and_set():
    d, keep = desc(max_blocks=0)
    begin_rc(d)
    msg = L.kvx_last_error()
    assert isinstance(msg, bytes) and len(msg) > 0


def test_pool_wrap_validation():
    g = kvx.geometry(4, 2, 64)
    h = C.c_void_p()
    assert L.kvx_pool_wrap(0, None, 1 << 20, C.byref(g), 2, 4, C.byref(h)) == kvx.KVX_EINVAL
    assert L.kvx_pool_wrap(0, C.c_void_p(0x1001), 1 << 20, C.byref(g), 2, 4, C.byref(h)) == kvx.KVX_EINVAL  # misaligned
    assert L.kvx_pool_wrap(0, C.c_void_p(0x1000), 16, C.byref(g), 2, 4, C.byref(h)) == kvx.KVX_EINVAL      # too small


def test_layout_validation():
    g = kvx.geometry(4, 2, 64)
    h = C.c_void_p()
    assert L.kvx_pool_create_layout(0, C.byref(g), 2, 4, 7, C.byref(h)) == kvx.KVX_EINVAL   # unknown layout
    g8 = kvx.geometry(4, 4, 4)                                # 8-byte head rows: no head-major layout
    assert L.kvx_pool_create_layout(0, C.byref(g8), 2, 4, kvx.LAYOUT_HEADS, C.byref(h)) == kvx.KVX_EINVAL
    ok = (C.c_void_p * 2)(0x1000, 0x2000)
    bb = g.block_bytes
    W = L.kvx_pool_wrap_layers
    assert W(0, 2, None, 4 * bb, C.byref(g), 4, kvx.LAYOUT_KV_PLANES, C.byref(h)) == kvx.KVX_EINVAL
    assert W(0, 2, ok, 4 * bb, C.byref(g), 4, 9, C.byref(h)) == kvx.KVX_EINVAL               # unknown layout
    assert W(0, 2, ok, 4 * bb - 16, C.byref(g), 4, 1, C.byref(h)) == kvx.KVX_EINVAL          # layer too small
    assert W(0, 2, (C.c_void_p * 2)(0x1000, None), 4 * bb, C.byref(g), 4, 1, C.byref(h)) == kvx.KVX_EINVAL
    assert W(0, 2, (C.c_void_p * 2)(0x1000, 0x2008), 4 * bb, C.byref(g), 4, 1, C.byref(h)) == kvx.KVX_EINVAL
    # bookkeeping only: a valid per-layer wrap needs no GPU; it cannot be read or exported
    assert W(0, 2, ok, 4 * bb, C.byref(g), 4, kvx.LAYOUT_KV_PLANES, C.byref(h)) == kvx.KVX_OK
    lay = C.c_int32(-1)
    assert L.kvx_pool_layout(h, C.byref(lay)) == kvx.KVX_OK and lay.value == kvx.LAYOUT_KV_PLANES
    buf = (C.c_uint8 * 16)()
    assert L.kvx_pool_read(h, 0, 16, buf) == kvx.KVX_EINVAL
    assert L.kvx_pool_export(h, (C.c_char * 64)()) == kvx.KVX_EINVAL
    assert L.kvx_pool_destroy(h) == kvx.KVX_OK


def test_weights_validation():
    ob = (C.c_int32 * 1)(2)
    ptrs = (C.c_void_p * 2)(None, None)
    db, hb = C.c_uint64(), C.c_uint64()
    # layer_bytes not a 16-byte multiple
    assert L.kvx_weights_migrate(0, None, 4, 10, 2, ob, ptrs, 2, ob, ptrs, None, None,
                                 C.byref(db), C.byref(hb)) == kvx.KVX_EINVAL
    # missing new-stage buffer
    assert L.kvx_weights_migrate(0, None, 4, 16, 2, ob, ptrs, 2, ob, ptrs, None, None,
                                 C.byref(db), C.byref(hb)) == kvx.KVX_EINVAL


def _wrap(device, addrs, num_blocks=16):
    """A bookkeeping-only per-layer pool at fake addresses (no GPU needed)."""
    g = kvx.geometry(4, 2, 64)
    h = C.c_void_p()
    ptrs = (C.c_void_p * len(addrs))(*addrs)
    assert L.kvx_pool_wrap_layers(device, len(addrs), ptrs, num_blocks * g.block_bytes, C.byref(g), num_blocks,
                                  kvx.LAYOUT_BLOCKS, C.byref(h)) == kvx.KVX_OK
    return h


def _desc_with(old, new):
    d, keep = desc()
    op = (C.c_void_p * 2)(*old)
    np_ = (C.c_void_p * 2)(*new)
    d.old_plan = kvx._Plan(2, d.old_plan.boundaries, C.cast(op, C.POINTER(C.c_void_p)))
    d.new_plan = kvx._Plan(2, d.new_plan.boundaries, C.cast(np_, C.POINTER(C.c_void_p)))
    return d, keep + (op, np_)


def test_new_pool_overlapping_an_old_pool_rejected():
    """destination ids start at 0, so a new pool aliasing an old one
    would overwrite source blocks a later wave still reads."""
    span = 16 * kvx.geometry(4, 2, 64).block_bytes
    base = 1 << 32
    old = [_wrap(0, [base, base + span]), _wrap(0, [base + 2 * span, base + 3 * span])]
    alias = [_wrap(0, [base + 2 * span + 4096]), _wrap(0, [base + 8 * span, base + 9 * span, base + 10 * span])]
    d, keep = _desc_with(old, alias)
    assert begin_rc(d) == kvx.KVX_EINVAL
    assert b"overlaps" in L.kvx_last_error()
    for h in old + alias:
        L.kvx_pool_destroy(h)


def test_old_pool_on_another_device_rejected():
    span = 16 * kvx.geometry(4, 2, 64).block_bytes
    base = 1 << 32
    old = [_wrap(1, [base, base + span]), _wrap(0, [base + 2 * span, base + 3 * span])]
    new = [_wrap(0, [base + 8 * span]), _wrap(0, [base + 9 * span, base + 10 * span, base + 11 * span])]
    d, keep = _desc_with(old, new)
    assert begin_rc(d) == kvx.KVX_EINVAL
    assert b"old pool on another device" in L.kvx_last_error()
    for h in old + new:
        L.kvx_pool_destroy(h)


def test_null_boundaries_rejected():
    d, keep = desc()
    d.old_plan = kvx._Plan(2, None, d.old_plan.pools)
    assert begin_rc(d) == kvx.KVX_EINVAL
    assert b"boundaries is null" in L.kvx_last_error()


def test_stage_kv_bytes_host_only():
    """kvx_stage_kv_bytes (no GPU): per new stage, layers x blocks x block bytes --
    what the engine adds to the grant's binding (engine.cpp:584-619)."""
    g = kvx.geometry(40, 40, 128)                 # Llama-2-13B: 320 KiB per layer-block
    out = kvx.stage_kv_bytes(g, [10, 20, 30], 1300)
    assert out == [10 * 1300 * 327680] * 4
    assert kvx.stage_kv_bytes(g, [5], 7) == [5 * 7 * 327680, 35 * 7 * 327680]
    with pytest.raises(kvx.KvxError):
        kvx.stage_kv_bytes(g, [30, 20], 4)        # not increasing
    with pytest.raises(kvx.KvxError):
        kvx.stage_kv_bytes(kvx.geometry(4, 1, 4), [2], 4)   # token_bytes 8


def test_begin_accepts_a_device_table_without_a_host_one():
    """ABI 4: src_block_table may be NULL when src_block_table_dev is given; without
    either, kvx_begin rejects the descriptor."""
    d, keep = desc()
    d.src_block_table = None
    assert begin_rc(d) == kvx.KVX_EINVAL
    assert b"src_block_table is null" in L.kvx_last_error()
    d, keep = desc()
    d.src_block_table = None
    d.src_block_table_dev = C.cast(C.c_void_p(0x1000), C.POINTER(C.c_int32))
    assert begin_rc(d) == kvx.KVX_EINVAL                # fails later (no pools), not on the table
    assert b"src_block_table" not in L.kvx_last_error()
