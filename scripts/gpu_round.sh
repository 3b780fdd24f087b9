#!/bin/bash
# Development round: TMA box probe (every case in its own process), GPU tests,
# C5 bench.
mkdir -p gpurun_out
n=$(./scripts/tma_probe count)
for i in $(seq 0 $((n - 1))); do
  timeout 30 ./scripts/tma_probe $i 2>&1 | head -1 >> gpurun_out/tma_probe_cases.log
done
echo "probe cases done" >> gpurun_out/times.log
T0=$(date +%s)
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$? wall=$(( $(date +%s) - T0 ))s" >> gpurun_out/times.log
for c in ${PFE_CONFIGS:-c5}; do
  python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "bench $c rc=$?" >> gpurun_out/times.log
done
