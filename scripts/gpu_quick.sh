# quick GPU check: parity tests + benches of the given configs
# usage: bash scripts/gpu_quick.sh "c5 c2" "tests/test_golden.py tests/test_gpu_solver.py"
set -x
mkdir -p gpurun_out
CFGS=${1:-"c5"}
TESTS=${2:-"tests/test_golden.py tests/test_gpu_solver.py tests/test_gpu_primitives.py tests/test_gpu_bands.py"}
timeout 1200 python -m pytest $TESTS -m gpu -x -q > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
tail -3 gpurun_out/pytest_quick.log
for c in $CFGS; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -2 gpurun_out/bench_$c.err; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/bench_c*.json')):
    try: d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e: print(f, 'ERR', e); continue
    r=d['roofline']; ks=r.get('kernels') or r.get('kernels_multi_kernel_path') or {}
    print(f, round(d['value'],1), 'e2e', round(d['e2e']['value'],1), r['kernel'], round(r['frac'],3), {k:(round(v['avg_us'],1), round(v['frac'],3)) for k,v in ks.items()})
PY
