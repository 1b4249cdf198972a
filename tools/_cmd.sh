mkdir -p gpurun_out; : > gpurun_out/var.txt
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 >> gpurun_out/var.txt
timeout 300 python tools/halo_run.py --steps 20 >> gpurun_out/var.txt 2>&1
for c in options bonds; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['e2e']['value'], d['value'], d['gpu_launches'])" >> gpurun_out/var.txt
done
cat gpurun_out/var.txt
