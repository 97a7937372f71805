#!/bin/bash
# E-in-registers inner solve: parity tests, per-round timing (ER vs smem E), C3/C5 stage times.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
mkdir -p gpurun_out/exp_er
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "inner or block_jacobi or factor_vs_oracle or ragged" 2>&1 | tail -3
for er in 1 0; do
  echo "== MPJSVD_INNER_EREG=$er"
  MPJSVD_INNER_EREG=$er MPJSVD_INNER_TIMING=1 timeout 300 python tools/bench_inner.py 2>&1 | grep -v "^\[inner" ; 
  MPJSVD_INNER_EREG=$er MPJSVD_INNER_TIMING=1 timeout 300 python tools/bench_inner.py 2>&1 | grep "^\[inner" | sort | uniq -c | sort -rn | head -4
done
for cfg in C3 C5; do
for o in "ER=1" "ER=0" "ER=1,mp_rrqr=1"; do
  er=${o:3:1}; extra=""; [[ "$o" == *mp_rrqr* ]] && extra="mp_rrqr=1"
  MPJSVD_INNER_EREG=$er MPJSVD_BENCH_OPTS="$extra" timeout 600 python bench.py --config $cfg --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/exp_er/${cfg}_$o.json 2>/dev/null
  python - "$cfg" "$o" <<'PY'
import json,sys
d=json.load(open(f"gpurun_out/exp_er/{sys.argv[1]}_{sys.argv[2]}.json"))
print(sys.argv[1], sys.argv[2], round(d['value'],4), d['sweeps32'], d['sweeps64'], {k:round(v,1) for k,v in d['stage_ms'].items()}, d['upd_trace64'], d['check'])
PY
done; done
