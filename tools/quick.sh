#!/usr/bin/env bash
# Box check: GPU tests, smoke, default bench line.
OUT=gpurun_out/${1:-quick}
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest.txt 2>&1; echo "pytest rc $?"
tail -5 $OUT/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc $?"; tail -2 $OUT/smoke.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc $?"
tail -1 $OUT/bench.json | cut -c1-3000
tail -5 $OUT/bench.err
