#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for c in c5 c1; do
PFE_E2E_TIMING=1 PFE_SETUP_TIMING=1 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_e2e_$c.json 2> gpurun_out/bench_e2e_$c.err
grep -h "pfe_solve:\|topology\|pfe_solver_create" gpurun_out/bench_e2e_$c.err | tail -6
done
python - <<'P'
import json
for c in ('c5','c1'):
    j=json.loads(open(f'gpurun_out/bench_e2e_{c}.json').read().strip().splitlines()[-1])
    print(c, 'value', round(j['value'],2), 'e2e', round(j['e2e']['value'],2), j['clocks']['sm_mhz'], j['clocks']['reasons'])
P
