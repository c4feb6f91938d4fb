# quick GPU validation: smoke, parity tests, bench on the three big configs (live per-kernel tables)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $? >> gpurun_out/status.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests $? >> gpurun_out/status.txt
for w in cfg4 cfg5 cfg3; do timeout 600 python bench.py --workload $w --no-cpu-baseline --profile-json gpurun_out/prof_$w.json > gpurun_out/bench_$w.log 2>&1; echo bench_$w $? >> gpurun_out/status.txt; done
