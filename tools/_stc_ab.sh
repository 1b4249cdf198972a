for lib in paper_2407_18352_b200/libsmlrt_b200.so paper_2407_18352_b200/libsmlrt_var_e1_32.so; do
for i in 1 2; do
SMLRT_B200_LIB=$PWD/$lib timeout 100 python bench.py --config options_bf16 --no-per-config --no-e2e --no-cpu --steps 30 --warmup 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', d['ms_per_step'], d['roofline']['kernel_ms'], d['parity']['pass'])"
done; done
