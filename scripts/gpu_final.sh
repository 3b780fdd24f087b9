# Round-end measurement: GPU tests, smoke, bench of every config (+ reference
# arm), ncu launch list of the default bench command, IC(0) / GMM timings.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
for c in c3 c4 c5; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 600 python scripts/time_ic0.py > gpurun_out/time_ic0.txt 2>&1
timeout 300 python scripts/time_gmm.py c2 > gpurun_out/time_gmm.txt 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -5 gpurun_out/smoke.log; cat gpurun_out/time_ic0.txt
