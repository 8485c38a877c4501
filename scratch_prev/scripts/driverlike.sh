#!/usr/bin/env bash
# What the round-end driver runs, in order, on one GPU.
o=gpurun_out/driverlike; mkdir -p $o
[ -z "${SKIP_TESTS:-}" ] && python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "smoke rc=$?" > $o/status.txt
[ -z "${SKIP_TESTS:-}" ] && timeout 1200 python -m pytest tests -x -q -m gpu > $o/pytest.log 2>&1; echo "pytest rc=$?" >> $o/status.txt
t0=$SECONDS; python bench.py --impl reference > $o/ref.jsonl 2> $o/ref.err; echo "ref rc=$? $((SECONDS-t0)) s" >> $o/status.txt
t0=$SECONDS; python bench.py > $o/bench.jsonl 2> $o/bench.err; echo "bench rc=$? $((SECONDS-t0)) s" >> $o/status.txt
