#!/bin/bash
# Quick GPU check of a change: focused parity tests (pytest -k EXPR) and C5 / C3 stage times (bench.py, 2 steps).
# Usage (GPU box, repo root): bash tools/exp_quick.sh TAG "pytest -k expression"
TAG=$1; K=$2; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -x -q -m gpu -k "$K" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.log
fi
bash tools/exp_opts.sh $TAG "C5:X=1" "C3:X=1" "C5:X=2"
