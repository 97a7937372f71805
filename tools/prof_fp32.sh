#!/bin/bash
# Targeted ncu capture of the fp32 round kernels (Gram + update) at one config, summarised on the box.
TAG=${1:-prof_fp32}; C=${2:-C5}; OUT=gpurun_out/$TAG; RAW=/tmp/ncu_$TAG; mkdir -p $OUT $RAW
CMD="python bench.py --config $C --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-profile --also ''"
timeout 600 bash -c "$CMD" > $OUT/plain.log 2>&1 || { tail -3 $OUT/plain.log; exit 1; }
timeout 1200 bash -c "ncu --set full --clock-control none --import-source on -k regex:'k_pair_gram_sw|k_pair_update_tc_ts' -s 40 -c 6 -o $RAW/prof $CMD" > $RAW/ncu.log 2>&1
echo "ncu rc=$?"
python tools/ncu_summary.py report $RAW/prof.ncu-rep > $OUT/ncu_full_$C.txt 2>&1
for k in k_pair_gram_sw k_pair_update_tc_ts; do python tools/ncu_hotlines.py $RAW/prof.ncu-rep $k 30 > $OUT/hot_${C}_$k.txt 2>&1; done
python tools/ncu_summary.py traffic $C $RAW/prof.ncu-rep > $OUT/traffic_$C.json 2>&1
