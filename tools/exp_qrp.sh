#!/bin/bash
# QRP experiment: parity tests of the QRP kernels, then per option set (OPTS="a=1 b=2,c=3 ...", bench-option
# overrides) the C5/C3 step time and the QRP phase clocks.
OUT=gpurun_out/${1:-exp_qrp}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
python -m pytest tests -m gpu -q -x -k "qr_vs_oracle or qrp" > $OUT/tests.log 2>&1; tail -2 $OUT/tests.log
for o in ${OPTS:-qrp_panel_stages=-1}; do
for c in ${CONFIGS:-C5 C3}; do
  n=$(echo "$o" | tr ',=' '__')
  MPJSVD_BENCH_OPTS=$o timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --also "" --no-profile > $OUT/bench_${c}_$n.json 2>&1
  python -c "import json; d=json.loads(open('$OUT/bench_${c}_$n.json').read().strip().splitlines()[-1]); print('$c $o', round(d['value'],4), {k: round(v,1) for k,v in d['stage_ms'].items()})"
  MPJSVD_BENCH_OPTS=diag_timing=1,$o timeout 600 python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --also "" --no-profile > /dev/null 2> $OUT/qrp_timing_${c}_$n.txt
  grep "qrp timing" $OUT/qrp_timing_${c}_$n.txt | tail -2 | head -1
done
done
