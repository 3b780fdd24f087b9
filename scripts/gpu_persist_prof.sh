# ncu --set full of one tiled persistent launch (C3 and C4) + per-line stall summary
set -x
mkdir -p gpurun_out
for c in c3 c4; do
  SKIP=1 COUNT=1 bash scripts/gpu_prof.sh $c "k_sb_persistent" "--persistent"
  python scripts/ncu_lines.py gpurun_out/ncu_${c}_source.csv 50 > gpurun_out/ncu_${c}_persist_lines.txt 2>&1
  rm -f gpurun_out/ncu_${c}_source.csv
done
