#!/bin/bash
# Re-entry check: GPU tests, smoke, the default bench line.
mkdir -p gpurun_out
log() { echo "$1 rc=$2 wall=$(( $(date +%s) - T0 ))s" >> gpurun_out/times.log; }
T0=$(date +%s); python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; log pytest $?
T0=$(date +%s); python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; log smoke $?
T0=$(date +%s); python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; log bench_default $?
T0=$(date +%s); python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; log bench_c5 $?
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/times.log
