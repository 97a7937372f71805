#!/bin/bash
# Build-flag experiment: rebuild libmpjsvd.so with each MPJSVD_NVCC_FLAGS variant, time C5 / C3 (bench.py, stage
# and kernel-bracket times), then restore the default build.  Usage: bash tools/exp_build_variants.sh TAG "flags" ...
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
for v in "$@"; do
  MPJSVD_NVCC_FLAGS="$v" python -c "from paper_2209_04626_b200 import build as b; b.build(force=True)" > $OUT/build.log 2>&1 || { echo "build failed: $v"; tail -3 $OUT/build.log; continue; }
  for c in ${CONFIGS:-C5 C3}; do
    n=$(echo "$v $c" | tr ' =' '__')
    timeout 600 python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/$n.json 2>$OUT/$n.err
    python - $OUT/$n.json "$v $c" <<'PY'
import json,sys
d=json.load(open(sys.argv[1]))
k={kk:round(v['ms_per_step'],1) for kk,v in d['kernels'].items() if 'pair' in kk}
print(sys.argv[2], round(d['value'],4), d['sweeps32'], d['sweeps64'], {kk:round(v,1) for kk,v in d['stage_ms'].items() if kk in ('fp32','fp64','lq','lift','assemble','qrp')}, k)
PY
  done
done
python -c "from paper_2209_04626_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
