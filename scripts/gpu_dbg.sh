mkdir -p gpurun_out
run() { timeout 120 python scripts/repro_tma.py $1 $2 2>&1 | tail -1 | cut -c1-40; }
( for m in 17 17 17 31 31 31 1 1; do echo "r1d4 mask $m: $(PFE_TMA=$m run 1 4)"; done
  for m in 31 31; do echo "r1d8 mask $m: $(PFE_TMA=$m run 1 8)"; done
  for m in 31 31; do echo "r1d4 1cta mask $m: $(PFE_PERSIST_ONE_CTA=1 PFE_TMA=$m run 1 4)"; done
  for m in 31 31 31; do echo "r2d4 mask $m: $(PFE_TMA=$m run 2 4)"; done ) > gpurun_out/dbg.log 2>&1
cat gpurun_out/dbg.log
