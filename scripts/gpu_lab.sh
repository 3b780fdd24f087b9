#!/bin/bash
# Development call: SpMV lab timings under several storage orders.
mkdir -p gpurun_out
for o in bfs cluster32 cluster64 cluster128 cluster256; do
  LAB_ORDER=$o timeout 900 python scripts/spmv_lab.py 5 20 22 24 > gpurun_out/spmv_lab_$o.log 2>&1
  echo "lab $o rc=$?" >> gpurun_out/times.log
done
