mkdir -p gpurun_out; : > gpurun_out/var.txt
for v in x3 x3l4; do
  if [ $v = default ]; then unset SMLRT_B200_LIB; else export SMLRT_B200_LIB=paper_2407_18352_b200/libsmlrt_b200_$v.so; fi
  for k in ss ts; do
  SMLRT_TC_KERNEL=$k timeout 300 python bench.py --config bonds --steps 20 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $k', d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'])" >> gpurun_out/var.txt
  done
done
cat gpurun_out/var.txt
