#!/bin/bash
# ncu --set full of one C4 tiled persistent launch with the closing build
# (plain run of the same command first), per-line stall summary on the box.
mkdir -p gpurun_out
python scripts/prof_run.py c4 1 --persistent > gpurun_out/plain_prof_c4.log 2>&1 && \
SKIP=1 COUNT=1 bash scripts/gpu_prof.sh c4 "k_sb_persistent" "--persistent" > gpurun_out/gpu_prof.log 2>&1
python scripts/ncu_lines.py gpurun_out/ncu_c4_source.csv 40 > gpurun_out/ncu_c4_persist_lines.txt 2>&1
rm -f gpurun_out/ncu_c4_source.csv gpurun_out/ncu_c4_details.txt
ls -la gpurun_out
