bash scripts/gpu_quick.sh "c3 c5" "tests/test_golden.py tests/test_gpu_solver.py tests/test_gpu_bands.py"
timeout 600 python scripts/prof_run.py c3 2 --trace > gpurun_out/trace_c3.log 2>&1
tail -7 gpurun_out/trace_c3.log
