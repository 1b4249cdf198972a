cfg=$1; shift
for lib in "$@"; do
for i in 1 2; do
SMLRT_B200_LIB=$PWD/paper_2407_18352_b200/$lib timeout 100 python bench.py --config $cfg --no-per-config --no-e2e --no-cpu --steps 30 --warmup 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cfg $lib', d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['parity']['pass'])"
done; done
