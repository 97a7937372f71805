#!/bin/bash
# Round profile of the default path, summarised ON the GPU box (raw ncu reports stay there: gpurun copies
# back at most 64 MiB).  Per config (C5, C3): ncu launch list of one step, ncu --set full of the fp32 round
# kernels, of the fp64 round kernels and of the QRP; summaries (launch shares, key metrics, DRAM traffic per
# launch -> profiles/ncu_traffic.json entry, per-line stall samples) written to gpurun_out/TAG.
# Usage (GPU box): bash tools/gpu_profile.sh TAG
TAG=${1:-prof}; OUT=gpurun_out/$TAG; RAW=/tmp/ncu_$TAG; mkdir -p $OUT $RAW
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
for C in ${CONFIGS:-C5 C3}; do
  CMD="python bench.py --config $C --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-profile --also ''"
  timeout 600 bash -c "$CMD" > $OUT/plain_$C.log 2>&1 || { echo "plain $C failed"; tail -3 $OUT/plain_$C.log; continue; }
  timeout 1500 bash -c "ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file $RAW/launches_$C.csv $CMD" > $RAW/ncu_launch_$C.log 2>&1
  echo "ncu launches $C rc=$?"
  python tools/ncu_summary.py launches $RAW/launches_$C.csv > $OUT/ncu_launches_$C.txt 2>&1
  timeout 1500 bash -c "ncu --set full --clock-control none --import-source on -k regex:'k_pair_solve|k_pair_update_tc|k_pair_gram_sw|k_pair_gram_tma' -s 60 -c 9 -o $RAW/prof_$C $CMD" > $RAW/ncu_full_$C.log 2>&1
  echo "ncu full $C rc=$?"
  timeout 1500 bash -c "ncu --set full --clock-control none --import-source on -k regex:'k_pair_gram_dmma|k_pair_update_dmma' -s 8 -c 4 -o $RAW/prof_f64_$C $CMD" > $RAW/ncu_f64_$C.log 2>&1
  echo "ncu f64 $C rc=$?"
  timeout 1500 bash -c "ncu --set full --clock-control none --import-source on -k regex:'k_qrp_lazy' -c 1 -o $RAW/prof_qrp_$C $CMD" > $RAW/ncu_qrp_$C.log 2>&1
  echo "ncu qrp $C rc=$?"
  python tools/ncu_summary.py report $RAW/prof_$C.ncu-rep $RAW/prof_f64_$C.ncu-rep $RAW/prof_qrp_$C.ncu-rep > $OUT/ncu_full_$C.txt 2>&1
  python tools/ncu_summary.py traffic $C $RAW/prof_$C.ncu-rep $RAW/prof_f64_$C.ncu-rep $RAW/prof_qrp_$C.ncu-rep > $OUT/ncu_traffic_$C.json 2>&1
  for k in k_pair_gram_sw k_pair_update_tc k_pair_solve; do
    python tools/ncu_hotlines.py $RAW/prof_$C.ncu-rep $k 25 > $OUT/hot_${C}_$k.txt 2>&1
  done
  python tools/ncu_hotlines.py $RAW/prof_f64_$C.ncu-rep k_pair_update_dmma 25 > $OUT/hot_${C}_k_pair_update_dmma.txt 2>&1
  python tools/ncu_hotlines.py $RAW/prof_qrp_$C.ncu-rep k_qrp_lazy 40 > $OUT/hot_${C}_k_qrp_lazy.txt 2>&1
done
cp profiles/ncu_traffic.json $OUT/ncu_traffic.json
du -sh $OUT
