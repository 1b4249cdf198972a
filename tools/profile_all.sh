#!/bin/bash
# ncu evidence for every config (one GPU): a --set full capture of each
# config's dominant kernel(s) and the cold launch list of a short bench run.
mkdir -p gpurun_out/r02
cap() {  # cfg kernel-regex name [extra bench args]
  local cfg=$1 kre=$2 name=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$kre" -s 2 -c 1 \
    -o gpurun_out/r02/prof_$name -f python bench.py --config $cfg --steps 1 --warmup 2 --no-e2e --no-cpu --no-parity --no-per-config "$@" \
    > gpurun_out/r02/prof_$name.log 2>&1; echo "$name rc=$?"
  ncu -i gpurun_out/r02/prof_$name.ncu-rep --page raw --csv > gpurun_out/r02/prof_$name.raw.csv 2>/dev/null
}
launches() {  # cfg [extra]
  local cfg=$1; shift
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02/launches_$cfg.csv python bench.py --config $cfg --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity --no-per-config "$@" \
    > /dev/null 2>&1; echo "launches $cfg rc=$?"
}
cap options region_exact options
cap bonds mlp3_tc bonds
cap minibude w4_fused minibude_w4
cap particlefilter conv_pool particlefilter_conv
cap particlefilter dense_pair particlefilter_dense
cap miniweather region_exact miniweather
for c in options bonds minibude particlefilter miniweather; do launches $c; done
