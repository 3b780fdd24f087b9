#!/bin/bash
# C5 A/B: split-Bregman pass with / without the L2 prefetch of b_old rows
mkdir -p gpurun_out
for p in 0 1; do
PFE_SB_PREFETCH=$p python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_pf$p.json 2> gpurun_out/bench_c5_pf$p.err
done
python - <<'P'
import json
for p in (0,1):
    j=json.loads(open(f'gpurun_out/bench_c5_pf{p}.json').read().strip().splitlines()[-1])
    k=j['roofline']['kernels']
    print('prefetch', p, 'value', round(j['value'],2), 'e2e', round(j['e2e']['value'],2), {n:(round(v['avg_us'],1), round(v['frac'],3)) for n,v in k.items()}, j['clocks']['sm_mhz'])
P
