# ncu captures of the weakest multi-kernel phases; reports are summarised on
# the box (details + raw csv + source csv) so gpurun_out stays small
# usage: bash scripts/gpu_prof.sh "c5 c3" [kernel-regex] [extra prof_run args]
set -x
mkdir -p gpurun_out
CFGS=${1:-"c5 c3"}
KRE=${2:-"k_pcg_pdir|k_pcg_spmv|k_sb_pass|k_grid_pcg_spmv|k_grid_sb_pass"}
EXTRA=${3:-"--host"}
for c in $CFGS; do
  rep=/tmp/ncu_$c
  timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"$KRE" --launch-skip ${SKIP:-12} -c ${COUNT:-4} -o $rep -f python scripts/prof_run.py $c 1 $EXTRA > gpurun_out/ncu_$c.log 2>&1
  echo "$c rc=$?"
  ncu -i $rep.ncu-rep --page details > gpurun_out/ncu_${c}_details.txt 2>&1
  ncu -i $rep.ncu-rep --page raw --csv > gpurun_out/ncu_${c}_raw.csv 2>&1
  ncu -i $rep.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/ncu_${c}_source.csv 2>&1
  ls -la gpurun_out/
done
