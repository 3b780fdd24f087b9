bash scripts/gpu_quick.sh "c3" "tests/test_golden.py tests/test_gpu_solver.py"
SKIP=2 COUNT=3 bash scripts/gpu_prof.sh c4 "k_grid_pcg_spmv|k_grid_sb_pass|k_pcg_update" "--host"
python scripts/ncu_lines.py gpurun_out/ncu_c4_source.csv 40 > gpurun_out/ncu_c4_lines.txt 2>&1
rm -f gpurun_out/ncu_c4_source.csv
