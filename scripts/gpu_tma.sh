#!/bin/bash
# 8-neighbour TMA investigation: every box case of scripts/tma_probe in its
# own process (a fault kills the context).
mkdir -p gpurun_out
n=$(./scripts/tma_probe count)
for i in $(seq 0 $((n - 1))); do
  timeout 30 ./scripts/tma_probe $i 2>&1 | head -1 >> gpurun_out/tma_probe_cases.log
done
echo "probe cases done" >> gpurun_out/times.log
