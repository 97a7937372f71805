#!/bin/bash
# Steady-state (warm L2, --cache-control none) DRAM read bytes per launch of the fp32 round kernels at C5, ONE metric
# so that ncu needs a single pass (no save / restore of the written buffers between passes, which would flush L2):
#   bash tools/l2probe.sh TAG [MPJSVD_BENCH_OPTS]
TAG=${1:-l2probe}; OPTS=${2:-}
mkdir -p gpurun_out/$TAG
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
MPJSVD_BENCH_OPTS=$OPTS timeout 900 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum -k regex:k_pair -s 4000 -c 12 --csv --log-file gpurun_out/$TAG/warm.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-profile > gpurun_out/$TAG/warm.log 2>&1
echo rc=$?
