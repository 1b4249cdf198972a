#!/bin/bash
# A/B of one config's bench line under env variants: tools/ab_cfg.sh <config> VAR=val[,VAR2=val] ...
mkdir -p gpurun_out
cfg=$1; shift
run() { # tag env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --config $cfg --no-per-config --no-cpu --no-e2e --steps 20 > gpurun_out/ab_${cfg}_$tag.json 2>gpurun_out/ab_${cfg}_$tag.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab_${cfg}_$tag.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$cfg $tag', d['ms_per_step'], r['kernel_ms'], r['bound'], r['frac'], r['hbm_frac'], d['clocks']['sm_mhz'], d['parity']['pass'])" || tail -5 gpurun_out/ab_${cfg}_$tag.err
}
run default X=1
for v in "$@"; do run "${v//[=,]/_}" ${v//,/ }; done
