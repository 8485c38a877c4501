"""The reference engine with kvx in its own transition handlers
(integration/engine_kvx.patch, built by integration/Makefile from a scratch
copy of /root/reference/proj):

  * CPU: the patch applies to the reference as shipped, and with PIPESIM_KVX
    unset the patched engine IS the reference -- its own 104 unit tests and
    12 acceptance criteria pass unchanged;
  * GPU: the same unmodified test sources with PIPESIM_KVX=parity (every
    wave / commit / abort moves real paged KV through libkvx.so), the plane's
    report proving the data plane ran: device Eq. 10 == host Eq. 10 at every
    commit, every live destination word == the payload; and the patched-engine
    cases of tests/native/test_kvx_patched.cpp (measured-time scheduling, the
    KV hold at the grant).
"""
import json
import os
import shutil
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
B = os.path.join(ROOT, "integration", "_build")
REF = "/root/reference/proj"


def _bin(name):
    path = os.path.join(B, name)
    assert os.path.exists(path), f"{path} missing: build it with __graft_entry__.build() (needs the reference)"
    return path


def _run(name, env_extra=None, timeout=1800):
    env = dict(os.environ)
    env.pop("PIPESIM_KVX", None)
    env.update(env_extra or {})
    return subprocess.run([_bin(name)], capture_output=True, text=True, timeout=timeout, env=env, cwd=B)


def _report(path):
    with open(path) as f:
        lines = [json.loads(l) for l in f if l.strip()]
    assert lines, "the kvx plane wrote no report"
    return lines[-1]


@pytest.mark.skipif(not os.path.isdir(REF), reason="needs /root/reference (build container)")
def test_patch_applies_to_the_reference():
    with tempfile.TemporaryDirectory() as d:
        shutil.copytree(os.path.join(REF, "src"), os.path.join(d, "src"))
        shutil.copytree(os.path.join(REF, "include"), os.path.join(d, "include"))
        out = subprocess.run(["patch", "--dry-run", "-p2", "-i", os.path.join(ROOT, "integration", "engine_kvx.patch")],
                             cwd=d, capture_output=True, text=True)
        assert out.returncode == 0, out.stdout + out.stderr


def test_patched_engine_without_kvx_is_the_reference():
    out = _run("unit_tests_kvx")
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "104 passed | 0 failed" in out.stdout


def test_patched_engine_without_kvx_passes_acceptance():
    out = _run("acceptance_kvx")
    assert out.returncode == 0, out.stdout[-3000:]
    assert "ALL CRITERIA PASS" in out.stdout


@pytest.mark.gpu
def test_reference_unit_tests_with_kvx_live(gpu_count, tmp_path):
    rep = str(tmp_path / "unit.jsonl")
    out = _run("unit_tests_kvx", {"PIPESIM_KVX": "parity", "PIPESIM_KVX_REPORT": rep})
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "104 passed | 0 failed" in out.stdout
    r = _report(rep)
    assert r["mode"] == "parity" and r["engines"] > 0
    assert r["transitions"] >= 4 and r["commits"] >= 3 and r["aborts"] >= 1   # test_engine.cpp:194-263
    assert r["waves"] > 0 and r["tokens"] > 0 and r["kvx_launches"] > 0
    assert r["violation_mismatches"] == 0 and r["violations_device"] == r["violations_host"]
    assert r["mismatched_words"] == 0 and r["verified_tokens"] > 0


@pytest.mark.gpu
def test_reference_acceptance_with_kvx_live(gpu_count, tmp_path):
    rep = str(tmp_path / "acc.jsonl")
    out = _run("acceptance_kvx", {"PIPESIM_KVX": "parity", "PIPESIM_KVX_REPORT": rep}, timeout=3000)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    assert "ALL CRITERIA PASS" in out.stdout
    r = _report(rep)
    assert r["commits"] >= 2 and r["waves"] > 0 and r["tokens"] > 0
    assert r["violation_mismatches"] == 0 and r["violations_device"] == r["violations_host"]
    assert r["mismatched_words"] == 0


@pytest.mark.gpu
def test_patched_engine_cases(gpu_count):
    out = _run("test_kvx_patched")
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    assert "4 passed | 0 failed" in out.stdout


@pytest.mark.gpu
def test_measured_time_mode_c3_real_geometry(gpu_count):
    """C3 (13B 8->4) through the patched engine at the real KV geometry: in
    measured mode wave 0's KvSyncComplete fires at begin + the B200's measured
    wave time, well before the reference's modelled 18.67 ms (kv_sync_bw 900 GB/s)."""
    env = {"PIPESIM_KVX": "measured"}
    out = subprocess.run([_bin("engine_patched_run"), "llama13b_8to4"], capture_output=True, text=True,
                         timeout=900, env=dict(os.environ, **env), cwd=B)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["refactor_commits"] == 1 and r["kv_violations"] == 0 and r["mismatched_words"] == 0
    assert "40x128" in r["geometries"]
    w0 = r["waves"][0]
    assert w0["scheduled_ms"] == w0["measured_ms"] < w0["modelled_ms"]
    first_sync = r["kv_sync_complete_ms"][0][1][0]
    assert first_sync == w0["issued_ms"] + w0["measured_ms"]


@pytest.mark.gpu
def test_reference_acceptance_in_measured_time_mode(gpu_count, tmp_path):
    """The reference's acceptance criteria with the engine on B200 time: every
    KvSyncComplete / RefactorCommit at the measured device completion."""
    rep = str(tmp_path / "acc_measured.jsonl")
    out = _run("acceptance_kvx", {"PIPESIM_KVX": "measured", "PIPESIM_KVX_REPORT": rep}, timeout=3000)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    assert "ALL CRITERIA PASS" in out.stdout
    r = _report(rep)
    assert r["mode"] == "measured" and r["commits"] >= 2 and r["mismatched_words"] == 0
    assert r["violation_mismatches"] == 0
    assert all(w["scheduled_ms"] == w["measured_ms"] for w in r["wave_log"])
