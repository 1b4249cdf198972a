#!/bin/bash
# ncu evidence for the kernels added late in round 2 (the others' captures are in profiles/r02)
mkdir -p gpurun_out/r02
cap() {  # cfg kernel-regex name [extra bench args]
  local cfg=$1 kre=$2 name=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$kre" -s 2 -c 1 \
    -o gpurun_out/r02/prof_$name -f python bench.py --config $cfg --steps 1 --warmup 2 --no-e2e --no-cpu --no-parity --no-per-config "$@" \
    > gpurun_out/r02/prof_$name.log 2>&1; echo "$name rc=$?"
}
launches() {  # cfg [extra]
  local cfg=$1; shift
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02/launches_$cfg.csv python bench.py --config $cfg --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity --no-per-config "$@" \
    > /dev/null 2>&1; echo "launches $cfg rc=$?"
}
cap particlefilter_bf16 conv_pool particlefilter_bf16_conv
cap particlefilter_bf16 gemm_tc particlefilter_bf16_gemm
cap miniweather_bf16 stencil_mma miniweather_bf16
for c in ${LAUNCH_CONFIGS:-options bonds minibude particlefilter particlefilter_bf16 miniweather miniweather_bf16}; do launches $c; done
