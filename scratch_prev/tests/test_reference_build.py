"""The oracle's reference build is faithful: the reference's OWN unit tests
(/root/reference/proj/tests/test_*.cpp, 104 doctest cases, unchanged, through
oracle/shim/doctest.h) and its acceptance binary (12 SPEC criteria) pass
against oracle/_ref/libpipesim.a -- the library the golden vectors are
extracted from.  Built by `make -C oracle reftests` (needs the reference
sources; __graft_entry__.build() does it in the build container)."""
import os
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = os.path.join(ROOT, "oracle", "_ref", "unit_tests")
ACCEPT = os.path.join(ROOT, "oracle", "_ref", "acceptance")


@pytest.mark.skipif(not os.path.exists(UNIT), reason="reference unit tests not built (no /root/reference here)")
def test_reference_unit_tests_pass():
    with tempfile.TemporaryDirectory() as d:
        out = subprocess.run([UNIT], capture_output=True, text=True, cwd=d, timeout=300)
    assert out.returncode == 0, out.stderr[-3000:]
    assert "104 passed | 0 failed" in out.stdout


@pytest.mark.skipif(not os.path.exists(ACCEPT), reason="reference acceptance not built (no /root/reference here)")
def test_reference_acceptance_passes():
    """Criterion 12 (acceptance_main.cpp:631-689) is the refactor-correctness
    gate whose scenario tests/golden/criterion12.jsonl pins."""
    with tempfile.TemporaryDirectory() as d:
        out = subprocess.run([ACCEPT], capture_output=True, text=True, cwd=d, timeout=600)
    assert out.returncode == 0, out.stdout[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("[PASS]") or l.startswith("[FAIL]")]
    assert len(lines) == 12 and all(l.startswith("[PASS]") for l in lines), out.stdout
    assert any("mid-decode refactor correctness" in l for l in lines)
