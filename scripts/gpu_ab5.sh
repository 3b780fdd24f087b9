#!/bin/bash
# A/B on C5: default library vs a variant (PFE_VARIANT); C5 set-up breakdown.
mkdir -p gpurun_out
PFE_LIB_VARIANT=$PFE_VARIANT python -m pytest tests/test_gpu_primitives.py tests/test_gpu_bands.py -x -q > gpurun_out/pytest_variant.log 2>&1
echo "pytest variant rc=$?" >> gpurun_out/times.log
for v in "" $PFE_VARIANT; do
  PFE_LIB_VARIANT=$v python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_${v:-base}.json 2> gpurun_out/bench_c5_${v:-base}.err
  echo "bench c5 ${v:-base} rc=$?" >> gpurun_out/times.log
done
PFE_SETUP_TIMING=1 PFE_E2E_TIMING=1 python scripts/e2e_breakdown.py c5 2 > gpurun_out/e2e_c5.txt 2>&1
