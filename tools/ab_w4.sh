#!/bin/bash
# A/B of the C3 headline kernel: default vs env variants (bench lines, no per-config)
mkdir -p gpurun_out
run() { # tag env...
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --no-per-config --no-cpu --no-e2e --steps 10 > gpurun_out/ab_$tag.json 2>gpurun_out/ab_$tag.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$tag.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$tag', d['ms_per_step'], r['kernel_ms'], r['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'], d['parity']['pass'])" || tail -5 gpurun_out/ab_$tag.err
}
run default X=1
for v in "$@"; do run "${v//[=,]/_}" ${v//,/ }; done
