#!/bin/bash
# One GPU session: parity tests, bench (C5 + C3), ncu launch list of the bench command.
# Usage (from the repo root, on the GPU box): bash tools/gpu_check.sh TAG [tests|bench|ncu ...]
set -u
TAG=${1:-run}; shift
WHAT=${*:-"tests bench ncu"}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $OUT/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -20 $OUT/build.log; exit 1; }
for w in $WHAT; do
  case $w in
  tests) timeout 1500 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log ;;
  smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke.log ;;
  bench) timeout 900 python bench.py > $OUT/bench_C5.json 2> $OUT/bench_C5.err; echo "bench C5 rc=$?"; cut -c1-400 $OUT/bench_C5.json
         timeout 600 python bench.py --config C3 --no-cpu-baseline > $OUT/bench_C3.json 2> $OUT/bench_C3.err; echo "bench C3 rc=$?"; cut -c1-300 $OUT/bench_C3.json ;;
  ncu)   timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_C5.csv \
            python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?" ;;
  esac
done
# ncu --set full of the Jacobi kernels on C3 (one launch each, round 11 of sweep 1)
if [[ " $WHAT " == *" ncufull "* ]]; then
  timeout 600 python bench.py --config C3 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $OUT/plain_C3.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_pair_(solve|update|gram)" -s 30 -c 3 \
     -o $OUT/prof_C3 python bench.py --config C3 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $OUT/ncu_full.log 2>&1
  echo "ncu full rc=$?"
fi
