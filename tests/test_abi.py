"""The C-ABI library loads and exports every symbol include/kvx.h declares
(no compute calls: this runs on the CPU-only build box too)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "kvx.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(kvx_\w+)\s*\(", src, re.M)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ("kvx_begin", "kvx_wave", "kvx_wait", "kvx_commit", "kvx_abort", "kvx_destroy",
                 "kvx_pool_create", "kvx_pool_export", "kvx_pool_import", "kvx_ctl_begin",
                 "kvx_ctl_sync_complete", "kvx_ctl_commit"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2510_11938_b200 import kvx
    lib = ctypes.CDLL(kvx.LIB_PATH)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert kvx.lib().kvx_abi_version() == 4


def test_library_is_sm100a():
    from paper_2510_11938_b200 import kvx
    out = subprocess.run(["cuobjdump", "--list-elf", kvx.LIB_PATH], capture_output=True, text=True)
    assert out.returncode == 0 and "sm_100a" in out.stdout


def test_no_gpu_is_reported_not_crashed():
    from paper_2510_11938_b200 import kvx
    n = kvx.device_count()
    assert n >= 0
    if n == 0:
        g = kvx.geometry(4, 2, 64)
        with pytest.raises(kvx.KvxError):
            kvx.Pool(0, g, 2, 8)


def test_invalid_geometry_rejected_before_cuda():
    from paper_2510_11938_b200 import kvx
    g = kvx.geometry(4, 1, 4)  # token_bytes = 8, not a multiple of 16
    with pytest.raises(kvx.KvxError) as e:
        kvx.Pool(0, g, 2, 8)
    assert e.value.code == kvx.KVX_EINVAL


def test_product_never_imports_the_oracle():
    """The product path has no CPU fallback and never touches oracle/."""
    pkg = os.path.join(ROOT, "paper_2510_11938_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "kvx_oracle" not in txt, f


def test_python_face_binds_every_declared_symbol():
    """kvx.py gives every header entry point a typed ctypes signature (a
    missing one would silently default to int arguments)."""
    src = open(os.path.join(ROOT, "paper_2510_11938_b200", "kvx.py")).read()
    bound = set(re.findall(r'"(kvx_\w+)":\s*\(', src))
    missing = [n for n in declared() if n not in bound]
    assert not missing, missing
