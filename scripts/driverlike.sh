#!/usr/bin/env bash
# What the round-end driver runs, in order, on one GPU.
o=gpurun_out/driverlike; mkdir -p $o
python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "smoke rc=$?" > $o/status.txt
timeout 1200 python -m pytest tests -x -q -m gpu > $o/pytest.log 2>&1; echo "pytest rc=$?" >> $o/status.txt
/usr/bin/time -f "%e s" python bench.py --impl reference > $o/ref.jsonl 2> $o/ref.err; echo "ref rc=$?" >> $o/status.txt
/usr/bin/time -f "%e s" python bench.py > $o/bench.jsonl 2> $o/bench.err; echo "bench rc=$?" >> $o/status.txt
