#!/bin/bash
# Round-2 closing measurements (what the driver runs, plus profiles):
# GPU tests, smoke, the default bench line, every config's bench line, the
# reference arm, the ncu launch list of the default bench and full captures
# of the C4 persistent kernel and the C5 split-Bregman pass (CSV on the box).
mkdir -p gpurun_out
log() { echo "$1 rc=$2 wall=$(( $(date +%s) - T0 ))s" >> gpurun_out/times.log; }
T0=$(date +%s); python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; log pytest $?
T0=$(date +%s); python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; log smoke $?
T0=$(date +%s); python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; log bench_default $?
for c in c1 c2 c3 c5; do
  T0=$(date +%s); python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; log bench_$c $?
done
T0=$(date +%s); python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; log reference $?
T0=$(date +%s)
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_c4_bench.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-warmup 0 > gpurun_out/ncu_launch.log 2>&1; log ncu_launches $?
export_rep() {
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
  ncu -i /tmp/$1.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | gzip > gpurun_out/$1_src.csv.gz
  rm -f /tmp/$1.ncu-rep
}
T0=$(date +%s)
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_sb_persistent --launch-skip 1 -c 1 \
  -o /tmp/ncu_k_sb_persistent_c4 python scripts/prof_run.py c4 1 > gpurun_out/ncu_c4.log 2>&1; log ncu_c4 $?
export_rep ncu_k_sb_persistent_c4
T0=$(date +%s)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sb_pass" --launch-skip 10 -c 1 \
  -o /tmp/ncu_c5_sb python scripts/prof_run.py c5 1 --host > gpurun_out/ncu_c5_sb.log 2>&1; log ncu_c5_sb $?
export_rep ncu_c5_sb
T0=$(date +%s); python scripts/e2e_breakdown.py c4 3 > gpurun_out/e2e_breakdown_c4.txt 2>&1; log e2e_c4 $?
T0=$(date +%s); PFE_SETUP_TIMING=1 PFE_E2E_TIMING=1 python scripts/e2e_breakdown.py c4 1 > gpurun_out/e2e_timing_c4.txt 2>&1; log e2e_timing_c4 $?
du -sh gpurun_out >> gpurun_out/times.log
