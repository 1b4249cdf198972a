mkdir -p gpurun_out
export SMLRT_B200_LIB=paper_2407_18352_b200/libsmlrt_b200_trace.so
SMLRT_TC_PAIR=0 timeout 120 python tools/tc_trace.py > gpurun_out/trace_single.txt 2>&1
SMLRT_TC_PAIR=1 timeout 120 python tools/tc_trace.py > gpurun_out/trace_pair.txt 2>&1
tail -5 gpurun_out/trace_single.txt gpurun_out/trace_pair.txt
