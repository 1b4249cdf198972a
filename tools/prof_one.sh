#!/bin/bash
# usage: tools/prof_one.sh <config> <kernel-regex> <name> [extra bench args]
# one `ncu --set full` capture (source-annotated) of the config's kernel after warm-up,
# plus the raw-page CSV export read back in the build container
mkdir -p gpurun_out
cfg=$1; kre=$2; name=$3; shift 3
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$kre" -s 2 -c 1 \
  -o gpurun_out/prof_$name -f python bench.py --config $cfg --steps 1 --warmup 2 --no-e2e --no-cpu --no-parity --no-per-config "$@" \
  > gpurun_out/prof_$name.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/prof_$name.log
ncu -i gpurun_out/prof_$name.ncu-rep --page raw --csv > gpurun_out/prof_$name.raw.csv 2>/dev/null
ncu -i gpurun_out/prof_$name.ncu-rep --page details --csv > gpurun_out/prof_$name.details.csv 2>/dev/null
