OUT=gpurun_out/r02_b; mkdir -p $OUT
MPJSVD_RECORD_DIR=$OUT/rec python -m pytest tests -m gpu -q -k "fullsize or warp_specialised or qrsvd or factor_vs_oracle or refine_v or auto or option_paths or ragged" > $OUT/tests.log 2>&1; tail -3 $OUT/tests.log
for v in 0 8 9; do
  for c in C5 C3; do
    MPJSVD_BENCH_OPTS=gram_variant=$v timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --also "" > $OUT/bench_gv${v}_$c.json 2>&1
    python -c "import json; d=json.loads(open('$OUT/bench_gv${v}_$c.json').read().strip().splitlines()[-1]); print('gv$v $c', round(d['value'],4), round(d['stage_ms']['fp32'],1), d['kernels'].get('pair_gram_f32'))"
  done
done
timeout 600 python tools/time_qrsvd.py 512 1024 2048 4096 > $OUT/qrsvd_time.log 2>&1; tail -1 $OUT/qrsvd_time.log
