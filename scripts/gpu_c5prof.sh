bash scripts/gpu_quick.sh "c5" "tests/test_golden.py"
SKIP=3 COUNT=1 bash scripts/gpu_prof.sh c5 "k_sb_pass" "--host"
python scripts/ncu_lines.py gpurun_out/ncu_c5_source.csv 40 > gpurun_out/ncu_c5_sb_lines.txt 2>&1
rm -f gpurun_out/ncu_c5_source.csv
