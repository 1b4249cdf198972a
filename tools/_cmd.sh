mkdir -p gpurun_out; : > gpurun_out/var.txt
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 >> gpurun_out/var.txt
for c in options miniweather; do
  timeout 200 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['roofline']['kernel_ms'], d['roofline']['frac'])" >> gpurun_out/var.txt
done
cat gpurun_out/var.txt
