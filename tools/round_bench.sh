#!/bin/bash
# Round record on the GPU box: default bench lines (C5 headline with C3 alongside), the reference arm, the ncu
# launch list of one C5 step and --set full of the round kernels (tools/gpu_profile.sh), all under gpurun_out/TAG.
TAG=${1:-round}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
timeout 1200 python bench.py --steps 20 --warmup 5 > $OUT/bench_C5.json 2> $OUT/bench_C5.err; echo "bench rc=$?"; cut -c1-300 $OUT/bench_C5.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?"; cut -c1-300 $OUT/bench_ref.json
[ -n "$NOPROF" ] || CONFIGS="${CONFIGS:-C5 C3}" bash tools/gpu_profile.sh $TAG/prof
