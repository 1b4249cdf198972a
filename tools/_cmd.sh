mkdir -p gpurun_out; : > gpurun_out/var.txt
timeout 600 python -m pytest tests/test_gpu_cnn.py -x -q 2>&1 | tail -3 >> gpurun_out/var.txt
for c in particlefilter; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['clocks'])" >> gpurun_out/var.txt
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_pf.csv python bench.py --config particlefilter --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
cat gpurun_out/var.txt
