set -x
SKIP=2 COUNT=4 bash scripts/gpu_prof.sh c3 "k_grid_sb_pass|k_grid_pcg_init" "--host"
timeout 600 python scripts/prof_run.py c3 2 --trace > gpurun_out/trace_c3.log 2>&1
timeout 600 python scripts/prof_run.py c4 1 --trace > gpurun_out/trace_c4.log 2>&1
rm -f gpurun_out/ncu_c3_source.csv
