#!/bin/bash
# A/B: default library vs a variant (PFE_VARIANT), C4 bench + trace, bitwise tests on the variant.
mkdir -p gpurun_out
PFE_LIB_VARIANT=$PFE_VARIANT python -m pytest tests/test_gpu_solver.py -x -q -k "tma_staging or persistent" > gpurun_out/pytest_variant.log 2>&1
echo "pytest variant rc=$?" >> gpurun_out/times.log
for v in "" $PFE_VARIANT; do
  for c in ${PFE_CONFIGS:-c4}; do
    PFE_LIB_VARIANT=$v python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_${v:-base}.json 2> gpurun_out/bench_${c}_${v:-base}.err
    echo "bench $c ${v:-base} rc=$?" >> gpurun_out/times.log
    PFE_LIB_VARIANT=$v timeout 600 python scripts/prof_run.py $c 2 --trace > gpurun_out/trace_${c}_${v:-base}.txt 2>&1
  done
done
