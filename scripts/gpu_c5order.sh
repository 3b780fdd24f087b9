#!/bin/bash
# A/B of the general-graph storage order on C5 (BFS vs reverse Cuthill-McKee)
# + ncu of the split-Bregman pass and SpMV for each (CSV exported on the box).
mkdir -p gpurun_out
for o in bfs rcm; do
  PFE_STORAGE_ORDER=$o python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_$o.json 2> gpurun_out/bench_c5_$o.err
  echo "bench c5 $o rc=$?" >> gpurun_out/times.log
  PFE_STORAGE_ORDER=$o timeout 900 ncu --set full --clock-control none -k regex:"k_sb_pass|k_pcg_spmv" --launch-skip 30 -c 2 \
    -o /tmp/ncu_c5_$o python scripts/prof_run.py c5 1 --host > gpurun_out/ncu_c5_$o.log 2>&1
  ncu -i /tmp/ncu_c5_$o.ncu-rep --page raw --csv > gpurun_out/ncu_c5_${o}_raw.csv 2>/dev/null
  rm -f /tmp/ncu_c5_$o.ncu-rep
done
