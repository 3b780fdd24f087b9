#!/bin/bash
# GPU check used during development: GPU tests, the default bench line and the
# reference arm, with wall times.  Outputs under gpurun_out/.
mkdir -p gpurun_out
T0=$(date +%s)
python -m pytest tests -m gpu -x -q -s -k "${PFE_TEST_K:-}" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$? wall=$(( $(date +%s) - T0 ))s" >> gpurun_out/times.log
if [ -n "${PFE_BENCH:-1}" ]; then
  T0=$(date +%s)
  python bench.py ${PFE_BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench rc=$? wall=$(( $(date +%s) - T0 ))s" >> gpurun_out/times.log
fi
if [ -n "${PFE_REF:-}" ]; then
  T0=$(date +%s)
  python bench.py --impl reference ${PFE_REF_ARGS:-} > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
  echo "reference rc=$? wall=$(( $(date +%s) - T0 ))s" >> gpurun_out/times.log
fi
