#!/bin/bash
# One gpurun call: the GPU parity suite, smoke(), the default bench line (headline + per_config),
# the reference arm, and the small-MLP kernel's ncu capture + launch list.  Output under gpurun_out/.
mkdir -p gpurun_out/r02
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "ref rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:small_tc" -s 2 -c 1 \
    -o gpurun_out/r02/prof_options_bf16 -f python bench.py --config options_bf16 --steps 1 --warmup 2 --no-e2e --no-cpu --no-parity --no-per-config > gpurun_out/r02/prof_options_bf16.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02/launches_options_bf16.csv python bench.py --config options_bf16 --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity --no-per-config > /dev/null 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:w4_fused" -s 2 -c 1 \
    -o gpurun_out/r02/prof_minibude_w4 -f python bench.py --config minibude --steps 1 --warmup 2 --no-e2e --no-cpu --no-parity --no-per-config > gpurun_out/r02/prof_minibude_w4.log 2>&1; echo "ncu w4 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02/launches_minibude.csv python bench.py --config minibude --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity --no-per-config > /dev/null 2>&1; echo "launches minibude rc=$?"
