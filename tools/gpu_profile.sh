#!/bin/bash
# Round profile: default bench line (C5) + C3 line, ncu launch list (first N launches of one C5 step),
# ncu --set full of the top kernels.  Usage: bash tools/gpu_profile.sh TAG
TAG=${1:-prof}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
timeout 900 python bench.py > $OUT/bench_C5.json 2> $OUT/bench_C5.err; echo "bench C5 rc=$?"
timeout 600 python bench.py --config C3 --no-cpu-baseline > $OUT/bench_C3.json 2> $OUT/bench_C3.err; echo "bench C3 rc=$?"
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 600 $CMD > $OUT/plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches_C5.csv $CMD > $OUT/ncu_launch.log 2>&1
echo "ncu launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"k_qrp_lazy|k_pair_solve|k_pair_update_tc|k_pair_update_dmma|k_pair_gram_tma|k_pair_gram_dmma" -s 60 -c 7 \
  -o $OUT/prof_C5 $CMD > $OUT/ncu_full.log 2>&1
echo "ncu full rc=$?"
# the QRP (one launch per step; the dominant single kernel): full set, first launch
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_qrp_lazy" -c 1 \
  -o $OUT/prof_qrp_C5 $CMD > $OUT/ncu_qrp.log 2>&1
echo "ncu qrp rc=$?"
