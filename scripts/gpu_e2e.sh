#!/bin/bash
# GPU tests + e2e breakdown + default bench (device-side grid topology build)
mkdir -p gpurun_out
T0=$(date +%s); python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$? wall=$(( $(date +%s) - T0 ))s" >> gpurun_out/times.log
PFE_SETUP_TIMING=1 PFE_E2E_TIMING=1 python scripts/e2e_breakdown.py c4 2 > gpurun_out/e2e_c4.txt 2>&1; echo "e2e rc=$?" >> gpurun_out/times.log
PFE_SETUP_TIMING=1 PFE_E2E_TIMING=1 python scripts/e2e_breakdown.py c3 2 > gpurun_out/e2e_c3.txt 2>&1
python bench.py --no-cpu-baseline > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?" >> gpurun_out/times.log
python bench.py --config c3 --steps 5 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench c3 rc=$?" >> gpurun_out/times.log
python bench.py --config c2 --steps 5 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench c2 rc=$?" >> gpurun_out/times.log
