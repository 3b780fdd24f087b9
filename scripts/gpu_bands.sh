#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_bands.py tests/test_gpu_solver.py -x -q > gpurun_out/pytest_bands.log 2>&1
echo "pytest bands rc=$?" >> gpurun_out/times.log
