mkdir -p gpurun_out; : > gpurun_out/var.txt
timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_region.py -x -q 2>&1 | tail -3 >> gpurun_out/var.txt
for c in ${CFG:-bonds}; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['clocks'])" >> gpurun_out/var.txt
done
cat gpurun_out/var.txt
