#!/bin/bash
# QRP experiment: parity tests of the QRP kernels, then C5/C3 step time and the QRP phase clocks.
OUT=gpurun_out/${1:-exp_qrp}; mkdir -p $OUT
python -m pytest tests -m gpu -q -x -k "qr_vs_oracle or qrp" > $OUT/tests.log 2>&1; tail -2 $OUT/tests.log
for c in C5 C3; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --also "" --no-profile > $OUT/bench_$c.json 2>&1
  python -c "import json; d=json.loads(open('$OUT/bench_$c.json').read().strip().splitlines()[-1]); print('$c', round(d['value'],4), {k: round(v,1) for k,v in d['stage_ms'].items()})"
  MPJSVD_BENCH_OPTS=diag_timing=1 timeout 600 python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --also "" --no-profile > /dev/null 2> $OUT/qrp_timing_$c.txt
  grep "qrp timing" $OUT/qrp_timing_$c.txt | tail -2
done
