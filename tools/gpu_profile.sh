#!/bin/bash
# Round profile of the default path: ncu launch list of one C5 step and one C3 step, ncu --set full of the
# Jacobi-round kernels and of the QRP for both configs.  Usage (GPU box): bash tools/gpu_profile.sh TAG
# Then here: tools/ncu_summary.py launches/report/traffic on gpurun_out/TAG/* -> profiles/.
TAG=${1:-prof}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
for C in C5 C3; do
  CMD="python bench.py --config $C --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-profile --also ''"
  timeout 600 bash -c "$CMD" > $OUT/plain_$C.log 2>&1 || { echo "plain $C failed"; tail -3 $OUT/plain_$C.log; continue; }
  timeout 1500 bash -c "ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file $OUT/launches_$C.csv $CMD" > $OUT/ncu_launch_$C.log 2>&1
  echo "ncu launches $C rc=$?"
  timeout 1500 bash -c "ncu --set full --clock-control none --import-source on -k regex:'k_pair_solve|k_pair_update_tc|k_pair_update_dmma|k_pair_gram_tma|k_pair_gram_dmma' -s 60 -c 10 -o $OUT/prof_$C $CMD" > $OUT/ncu_full_$C.log 2>&1
  echo "ncu full $C rc=$?"
  timeout 1500 bash -c "ncu --set full --clock-control none --import-source on -k regex:'k_pair_gram_dmma|k_pair_update_dmma' -s 8 -c 4 -o $OUT/prof_f64_$C $CMD" > $OUT/ncu_f64_$C.log 2>&1
  echo "ncu f64 $C rc=$?"
  timeout 1500 bash -c "ncu --set full --clock-control none --import-source on -k regex:'k_qrp_lazy' -c 1 -o $OUT/prof_qrp_$C $CMD" > $OUT/ncu_qrp_$C.log 2>&1
  echo "ncu qrp $C rc=$?"
done
