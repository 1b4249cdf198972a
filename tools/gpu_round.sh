#!/bin/bash
# One gpurun call: GPU parity suite, every config's bench line, the launch list
# of the headline bench.  Output under gpurun_out/ (scratch; summaries go to profiles/).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
cp MEASURED_PEAKS.json gpurun_out/ 2>/dev/null
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
for c in ${CONFIGS:-options bonds minibude particlefilter miniweather}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 ${BENCH_FLAGS:---no-cpu} > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$?"; tail -1 gpurun_out/bench_$c.json | cut -c1-600
done
