#!/bin/bash
# GPU tests, then e2e stage timings under bench conditions (stderr of pfe_solve / pfe_solver_create)
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
PFE_E2E_TIMING=1 PFE_SETUP_TIMING=1 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_e2e_c4.json 2> gpurun_out/bench_e2e_c4.err
grep -h "pfe_solve:" gpurun_out/bench_e2e_c4.err | tail -8
for c in c2 c3 c5; do
PFE_E2E_TIMING=1 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_e2e_$c.json 2> gpurun_out/bench_e2e_$c.err
grep -h "pfe_solve:" gpurun_out/bench_e2e_$c.err | tail -3
done
python - <<'P'
import json
for c in ('c4','c2','c3','c5'):
    j=json.loads(open(f'gpurun_out/bench_e2e_{c}.json').read().strip().splitlines()[-1])
    print(c, 'value', round(j['value'],2), 'e2e', round(j['e2e']['value'],2), j['clocks']['sm_mhz'], j['clocks']['reasons'])
P
