#!/bin/bash
# GPU tests + the C5 bench line (general-graph kernels) + C4 quick bench.
mkdir -p gpurun_out
T0=$(date +%s)
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$? wall=$(( $(date +%s) - T0 ))s" >> gpurun_out/times.log
python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
echo "bench c5 rc=$?" >> gpurun_out/times.log
