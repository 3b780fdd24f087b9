#!/bin/bash
# GPU tests (+ new error / warning tests), the default C4 bench line, the
# partition statistics, the ncu launch list of the bench command and one
# ncu --set full capture of the C4 persistent kernel.
mkdir -p gpurun_out
T0=$(date +%s)
python -m pytest tests -m gpu -x -q --deselect "tests/test_gpu_full_parity.py::test_full_size_parity[c4]" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$? wall=$(( $(date +%s) - T0 ))s" >> gpurun_out/times.log
T0=$(date +%s)
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$? wall=$(( $(date +%s) - T0 ))s" >> gpurun_out/times.log
python scripts/partition_stats.py > gpurun_out/partition_stats.json 2> gpurun_out/partition_stats.err
echo "partition rc=$?" >> gpurun_out/times.log
T0=$(date +%s)
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_c4_bench.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-warmup 0 > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$? wall=$(( $(date +%s) - T0 ))s" >> gpurun_out/times.log
T0=$(date +%s)
ncu --set full --clock-control none --import-source on -k regex:k_sb_persistent --launch-skip 1 -c 1 \
  -o gpurun_out/ncu_k_sb_persistent_c4 python scripts/prof_run.py c4 1 > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$? wall=$(( $(date +%s) - T0 ))s" >> gpurun_out/times.log
