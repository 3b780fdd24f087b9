# ncu of one PCG direction pass + SpMV pair of C5 (the bench's pcg_spmv class)
set -x
SKIP=20 COUNT=2 bash scripts/gpu_prof.sh c5 "k_pcg_pdir|k_pcg_spmv" "--host"
python scripts/ncu_lines.py gpurun_out/ncu_c5_source.csv 30 > gpurun_out/ncu_c5_spmv_lines.txt 2>&1
rm -f gpurun_out/ncu_c5_source.csv
