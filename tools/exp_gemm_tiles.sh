#!/bin/bash
# GEMM tile experiment: rebuild libmpjsvd.so with MPJSVD_NVCC_FLAGS variants and time tools/time_gemm.py
OUT=gpurun_out/${1:-exp_gemm_tiles}; mkdir -p $OUT
for v in "${@:2}"; do
  MPJSVD_NVCC_FLAGS="$v" python -c "from paper_2209_04626_b200 import build as b; b.build(force=True)" > $OUT/build.log 2>&1 || { echo "build failed: $v"; tail -3 $OUT/build.log; continue; }
  echo "== $v"; timeout 300 python tools/time_gemm.py 2>&1 | tee -a $OUT/time.txt
done
python -c "from paper_2209_04626_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
