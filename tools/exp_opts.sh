#!/bin/bash
# Experiment driver: bash tools/exp_opts.sh TAG "CFG:ENV=..;OPTS=.." ...   (stage times per setting)
TAG=$1; shift
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
mkdir -p gpurun_out/$TAG
for spec in "$@"; do
  cfg=${spec%%:*}; rest=${spec#*:}
  envs=$(echo "$rest" | sed 's/;/ /g')
  name=$(echo "$spec" | tr ':;=,' '____')
  env $envs timeout 600 python bench.py --config $cfg --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/$TAG/$name.json 2>gpurun_out/$TAG/$name.err
  python - gpurun_out/$TAG/$name.json "$spec" <<'PY'
import json,sys
d=json.load(open(sys.argv[1]))
k={kk:round(v['ms_per_step'],1) for kk,v in d['kernels'].items() if 'pair' in kk}
print(sys.argv[2], round(d['value'],4), d['sweeps32'], d['sweeps64'], {kk:round(v,1) for kk,v in d['stage_ms'].items() if kk in ('fp32','fp64','lq','lift','assemble','qr_tall')}, k)
PY
done
