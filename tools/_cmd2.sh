mkdir -p gpurun_out
timeout 300 compute-sanitizer --tool memcheck --show-backtrace device --print-limit 3 python -m pytest "tests/test_gpu_stencil_tc.py::test_stencil_tc_matches_oracle[fused-40-132]" -x -q > gpurun_out/san2.log 2>&1
grep -v "^=========     Host Frame" gpurun_out/san2.log | head -40
