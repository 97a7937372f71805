#!/bin/bash
# inner-solve build variants: per-round cost and per-warp-group phase clocks (tools/bench_inner.py)
for v in "$@"; do
  MPJSVD_NVCC_FLAGS="$v" python -c "from paper_2209_04626_b200 import build as b; b.build(force=True)" > /tmp/b.log 2>&1 || { echo "build failed $v"; tail -3 /tmp/b.log; continue; }
  echo "== $v"; python tools/bench_inner.py; python tools/bench_inner.py phases 2>&1 | grep "inner timing"
done
python -c "from paper_2209_04626_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
