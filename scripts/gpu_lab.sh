#!/bin/bash
# Development call: new multi-GPU tests, the SpMV kernel lab, the forced
# 8-neighbour TMA case under memcheck.
mkdir -p gpurun_out
python -m pytest tests/test_gpu_bands.py -x -q -s -k "multi_gpu" > gpurun_out/pytest_multi.log 2>&1
echo "pytest multi rc=$?" >> gpurun_out/times.log
timeout 900 python scripts/spmv_lab.py > gpurun_out/spmv_lab.log 2>&1
echo "lab rc=$?" >> gpurun_out/times.log
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_cases.py tiled8tma > gpurun_out/tma8_memcheck.log 2>&1
echo "tma8 memcheck rc=$?" >> gpurun_out/times.log
