# build, then per-layer live timings of cfg4 and cfg5 (no tests)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for w in cfg4 cfg5; do timeout 300 python bench.py --workload $w --steps 5 --no-e2e --no-cpu-baseline --profile-json gpurun_out/prof_$w.json > gpurun_out/bench_$w.log 2>&1; echo bench_$w $? >> gpurun_out/status.txt; done
