mkdir -p gpurun_out
export SMLRT_TC_PAIR=${PAIRS:-1}
timeout 300 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -2
SMLRT_TC_PAIR=0 timeout 200 python bench.py --config bonds --steps 20 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-200
SMLRT_TC_PAIR=1 timeout 200 python bench.py --config bonds --steps 20 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-200
export SMLRT_B200_LIB=paper_2407_18352_b200/libsmlrt_b200_trace.so
SMLRT_TC_PAIR=0 timeout 120 python tools/tc_trace.py > gpurun_out/trace_single.txt 2>&1
SMLRT_TC_PAIR=1 timeout 120 python tools/tc_trace.py > gpurun_out/trace_pair.txt 2>&1
grep period gpurun_out/trace_*.txt
