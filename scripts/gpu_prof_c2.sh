# ncu --set full of one k_sb_resident launch (C2, the bench default) + summary
set -x
mkdir -p gpurun_out
SKIP=2 COUNT=1 bash scripts/gpu_prof.sh c2 "k_sb_resident" "--persistent"
python scripts/ncu_lines.py gpurun_out/ncu_c2_source.csv 30 > gpurun_out/ncu_c2_lines.txt 2>&1
rm -f gpurun_out/ncu_c2_source.csv
