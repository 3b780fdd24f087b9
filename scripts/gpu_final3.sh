#!/bin/bash
# Round-2 closing measurements with the final build (what the driver runs,
# plus every configuration and the launch list of the default bench).
mkdir -p gpurun_out
log() { echo "$1 rc=$2 wall=$(( $(date +%s) - T0 ))s" >> gpurun_out/times.log; }
T0=$(date +%s); python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; log pytest $?
T0=$(date +%s); python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; log smoke $?
T0=$(date +%s); python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; log bench_default $?
for c in c1 c2 c3 c5; do
  T0=$(date +%s); python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; log bench_$c $?
done
T0=$(date +%s); python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; log reference $?
T0=$(date +%s)
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-warmup 0 > gpurun_out/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_c4_bench.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-warmup 0 > gpurun_out/ncu_launch.log 2>&1; log ncu_launches $?
T0=$(date +%s); PFE_SETUP_TIMING=1 PFE_E2E_TIMING=1 python scripts/e2e_breakdown.py c4 3 > gpurun_out/e2e_breakdown_c4.txt 2>&1; log e2e_c4 $?
cat gpurun_out/times.log; tail -2 gpurun_out/pytest_gpu.log
