#!/bin/bash
# usage: tools/prof.sh <config> <kernel-regex> <name> [extra bench args]
# one `ncu --set full` capture of the config's fused kernel (after warm-up)
mkdir -p gpurun_out
cfg=$1; kre=$2; name=$3; shift 3
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$kre" -s 2 -c 1 \
  -o gpurun_out/prof_$name -f python bench.py --config $cfg --steps 1 --warmup 2 --no-e2e --no-cpu "$@" \
  > gpurun_out/prof_$name.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/prof_$name.log
