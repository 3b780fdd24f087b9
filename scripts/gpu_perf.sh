#!/bin/bash
# GPU tests, then bench lines of C3 / C4 / C5 and phase traces of the
# persistent kernels (development measurements).
mkdir -p gpurun_out
T0=$(date +%s)
python -m pytest tests -m gpu -x -q ${PFE_PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$? wall=$(( $(date +%s) - T0 ))s" >> gpurun_out/times.log
for c in ${PFE_CONFIGS:-c5 c3 c4}; do
  T0=$(date +%s)
  python bench.py --config $c --steps ${PFE_STEPS:-5} --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "bench $c rc=$? wall=$(( $(date +%s) - T0 ))s" >> gpurun_out/times.log
done
for c in ${PFE_TRACE_CONFIGS:-c3 c4}; do
  timeout 600 python scripts/prof_run.py $c 2 --trace > gpurun_out/trace_$c.txt 2>&1
  echo "trace $c rc=$?" >> gpurun_out/times.log
done
