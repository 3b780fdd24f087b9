#!/bin/bash
# Development round: staging bitwise tests, C4 with cp.async vs TMA tiles,
# C5 bench.
mkdir -p gpurun_out
python -m pytest tests/test_gpu_solver.py -x -q -k "tma_staging or persistent" > gpurun_out/pytest_tma.log 2>&1
echo "pytest tma rc=$?" >> gpurun_out/times.log
for t in 0 1; do
  PFE_TMA=$t python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_tma$t.json 2> gpurun_out/bench_c4_tma$t.err
  echo "bench c4 tma=$t rc=$?" >> gpurun_out/times.log
  PFE_TMA=$t timeout 600 python scripts/prof_run.py c4 2 --trace > gpurun_out/trace_c4_tma$t.txt 2>&1
done
python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
echo "bench c5 rc=$?" >> gpurun_out/times.log
