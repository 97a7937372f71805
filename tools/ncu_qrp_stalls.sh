OUT=gpurun_out/ncu_qrp_stalls; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
CMD="python bench.py --config C5 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-profile --also ''"
timeout 600 bash -c "$CMD" > $OUT/plain.log 2>&1 || { echo plain failed; tail -3 $OUT/plain.log; exit 1; }
timeout 1200 bash -c "ncu --set full --clock-control none --import-source on -k regex:k_qrp_lazy -c 1 -o /tmp/qrp_prof $CMD" > $OUT/ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_stalls.py /tmp/qrp_prof.ncu-rep k_qrp_lazy k_qrp.cu 200 620 > $OUT/stalls.txt 2>&1
python tools/ncu_hotlines.py /tmp/qrp_prof.ncu-rep k_qrp_lazy 50 > $OUT/hot.txt 2>&1
python tools/ncu_summary.py report /tmp/qrp_prof.ncu-rep > $OUT/summary.txt 2>&1
tail -5 $OUT/stalls.txt | cut -c1-300
