# build, GPU tests, then per-layer live timings of cfg4 and cfg5
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 120 python scripts/run_step.py --workload cfg2 > gpurun_out/quick_cfg2.log 2>&1; echo quick_cfg2 $? >> gpurun_out/status.txt
grep -q "quick_cfg2 0" gpurun_out/status.txt || exit 1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests $? >> gpurun_out/status.txt
for w in cfg4 cfg5; do timeout 300 python bench.py --workload $w --steps 5 --no-e2e --no-cpu-baseline --profile-json gpurun_out/prof_$w.json > gpurun_out/bench_$w.log 2>&1; echo bench_$w $? >> gpurun_out/status.txt; done
