#!/bin/bash
mkdir -p gpurun_out
PFE_SETUP_TIMING=1 PFE_E2E_TIMING=1 python scripts/e2e_breakdown.py c5 2 > gpurun_out/e2e_c5.txt 2>&1; echo "e2e rc=$?" >> gpurun_out/times.log
python bench.py --config c5 --steps 5 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench c5 rc=$?" >> gpurun_out/times.log
python -m pytest tests/test_gpu_full_parity.py -x -q -k c5 -s > gpurun_out/pytest_c5.log 2>&1; echo "parity c5 rc=$?" >> gpurun_out/times.log
