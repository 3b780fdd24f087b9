#!/bin/bash
# 8-neighbour TMA investigation: the standalone box probe, then the tiled
# persistent kernel on an 8-neighbour grid with TMA forced per phase (each in
# its own process, bounded by timeout).  Then ncu captures for profiles/,
# exported to CSV on the box (the .ncu-rep files are too big to bring back).
mkdir -p gpurun_out
timeout 120 ./scripts/tma_probe > gpurun_out/tma_probe.log 2>&1
echo "probe rc=$?" >> gpurun_out/times.log
for m in 1 2 4 8 16 31; do
  for d in 8 4; do
    r=$(PFE_TMA_MASK=$m PFE_SAN_D=$d timeout 120 python scripts/sanitize_cases.py tiled8tma 2>&1 | tail -1 | cut -c1-160)
    echo "mask $m d $d: $r" >> gpurun_out/tma_masks.log
  done
done
echo "masks done" >> gpurun_out/times.log
export_rep() {  # $1 = report base name
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/$1_src.csv 2>/dev/null
  gzip -f gpurun_out/$1_src.csv
  rm -f /tmp/$1.ncu-rep
}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sb_persistent --launch-skip 1 -c 1 \
  -o /tmp/ncu_k_sb_persistent_c3 python scripts/prof_run.py c3 1 > gpurun_out/ncu_c3.log 2>&1
echo "ncu c3 rc=$?" >> gpurun_out/times.log
export_rep ncu_k_sb_persistent_c3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pcg_spmv|k_sb_pass|k_pcg_init" --launch-skip 30 -c 3 \
  -o /tmp/ncu_c5 python scripts/prof_run.py c5 1 --host > gpurun_out/ncu_c5.log 2>&1
echo "ncu c5 rc=$?" >> gpurun_out/times.log
export_rep ncu_c5
du -sh gpurun_out >> gpurun_out/times.log
