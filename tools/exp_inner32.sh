python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/exp1
for cfg in C3 C5; do
for o in "max_inner32=1" "max_inner32=2" "max_inner32=3"; do
  MPJSVD_BENCH_OPTS="$o" timeout 600 python bench.py --config $cfg --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/exp1/${cfg}_$o.json 2>/dev/null
  python - "$cfg" "$o" <<'PY'
import json,sys
d=json.load(open(f"gpurun_out/exp1/{sys.argv[1]}_{sys.argv[2]}.json"))
print(sys.argv[1], sys.argv[2], round(d['value'],4), d['sweeps32'], d['sweeps64'], {k:round(v,1) for k,v in d['stage_ms'].items() if k in ('fp32','fp64')}, d['upd_trace64'])
PY
done; done
