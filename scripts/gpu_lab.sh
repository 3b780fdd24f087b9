#!/bin/bash
# Development call: one ncu --set full launch per chosen SpMV lab variant.
mkdir -p gpurun_out
LAB_REPS=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"v_regs|v_ring|v_stream" -c 4 \
  -o gpurun_out/ncu_lab python scripts/spmv_lab.py 0 5 14 9 > gpurun_out/ncu_lab.log 2>&1
echo "ncu lab rc=$?" >> gpurun_out/times.log
