#!/bin/bash
mkdir -p gpurun_out
PFE_E2E_TIMING=1 PFE_SETUP_TIMING=1 python bench.py --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_e2e.json 2> gpurun_out/bench_c4_e2e.err
echo "bench rc=$?" >> gpurun_out/times.log
