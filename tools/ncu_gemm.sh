#!/bin/bash
# ncu --set full of the library DMMA GEMM at the path's shapes (tools/time_gemm.py), per-line stall reasons
OUT=gpurun_out/${1:-ncu_gemm}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python tools/time_gemm.py > $OUT/time.txt 2>&1; cat $OUT/time.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm_f64 -s 1 -c 2 -o /tmp/gemm_prof python tools/time_gemm.py > $OUT/ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py report /tmp/gemm_prof.ncu-rep > $OUT/summary.txt 2>&1
python tools/ncu_stalls.py /tmp/gemm_prof.ncu-rep k_gemm_f64 k_linalg.cu 40 180 > $OUT/stalls.txt 2>&1
grep -E "Duration|Throughput|tensor|Occupancy|Registers|Warp Cycles" $OUT/summary.txt | head -30
sort -k2 -n -r $OUT/stalls.txt | head -20 | cut -c1-220
