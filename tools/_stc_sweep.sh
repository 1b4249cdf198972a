timeout 300 python -m pytest tests/test_gpu_small_mma.py -x -q 2>&1 | tail -3
SMLRT_STC_DEBUG=1 timeout 100 python bench.py --config options_bf16 --no-per-config --no-e2e --no-cpu --no-parity --steps 5 --warmup 3 2>&1 | grep small_tc | head -3
for n in 4 6 8; do
SMLRT_STC_PER_SM=$n timeout 100 python bench.py --config options_bf16 --no-per-config --no-e2e --no-cpu --no-parity --steps 20 --warmup 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('per_sm $n', d['ms_per_step'], d['roofline']['kernel_ms'])"
done
