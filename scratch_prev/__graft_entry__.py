"""Driver entry points.

build(): compiles the product (paper_2510_11938_b200/_lib/libkvx.so, sm_100a)
         and the CPU oracle (oracle/_build/libkvx_oracle.so); when the
         reference sources are present (build container only) also the
         reference library + golden extractor under oracle/_ref.  Building
         the checker is not using it.
smoke(): one small inflight refactor on cuda:0 through the C-ABI, checked
         byte for byte against the oracle.
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def build() -> None:
    from paper_2510_11938_b200 import build as B
    B.build()
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True)
    if os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref", "reftests", "-j8"], check=True)
        # reference engine <-> kvx integration harness (links both libraries)
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "native")], check=True)
    import paper_2510_11938_b200.kvx  # noqa: F401  (loads the .so: fails loudly if absent)


def smoke() -> None:
    import numpy as np

    from paper_2510_11938_b200 import kvx
    from paper_2510_11938_b200 import workload as W
    from tests.gpu_harness import SEED, GpuCase

    if kvx.device_count() < 1:
        raise RuntimeError("smoke(): no CUDA device visible to libkvx.so")
    before = kvx.launch_count()
    scn = W.load_golden("engine_mid_decode")  # test_engine.cpp:207-238, forced 4->16 mid-decode
    (t,) = scn.transitions
    case = GpuCase(scn, t, 2, 64)
    try:
        case.run_ctl()
        case.compare_tables()
        case.compare_bytes()
        res = case.tr.on_refactor_commit((t.live_req, t.live_kv))
        ov, row_ptr, blocks, free = case.dp.commit(t.live_req, t.live_kv)
        assert res.violations == ov == t.violations == 0
        assert np.array_equal(res.blocks, blocks) and np.array_equal(res.free_list, free)
        assert case.tr.verify_pattern(SEED, t.live_req, t.live_kv) == 0
    finally:
        case.close()
    launched = kvx.launch_count() - before
    print(f"smoke ok: {t.old_stages}->{t.new_stages} stages, {len(t.live_req)} live requests, "
          f"{launched} kvx kernels launched, bit-exact vs oracle")


if __name__ == "__main__":
    build()
    if "--smoke" in sys.argv:
        smoke()
