set -x
mkdir -p gpurun_out
timeout 600 python scripts/repro_tma.py 1 4 > gpurun_out/repro.log 2>&1; echo "repro rc=$?" >> gpurun_out/repro.log; tail -2 gpurun_out/repro.log
timeout 900 python -m pytest tests/test_gpu_solver.py -m gpu -x -q -k "tma or persistent or resident" > gpurun_out/pytest_tma.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tma.log
tail -5 gpurun_out/pytest_tma.log
bash scripts/gpu_quick.sh "c4" "tests/test_golden.py"
PFE_BULK=0 timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_nobulk.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/bench_c4_nobulk.json').read().strip().splitlines()[-1]); print('nobulk', d['value'], d['roofline']['frac'])"
