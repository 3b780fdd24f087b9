set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_solver.py -m gpu -x -q -k "tma or persistent or resident" > gpurun_out/pytest_tma.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tma.log
tail -15 gpurun_out/pytest_tma.log
bash scripts/gpu_quick.sh "c3 c4" "tests/test_golden.py"
for c in c3 c4; do PFE_TMA=0 timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_notma.json 2>/dev/null; done
python - <<'PY'
import json
for c in ('c3','c4'):
    for suf in ('','_notma'):
        try:
            d=json.loads(open(f'gpurun_out/bench_{c}{suf}.json').read().strip().splitlines()[-1]); print(c, suf or 'tma', round(d['value'],1), round(d['roofline']['frac'],3))
        except Exception as e: print(c, suf, 'ERR', e)
PY
