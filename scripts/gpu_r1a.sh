set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $? >> gpurun_out/status.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests $? >> gpurun_out/status.txt
timeout 900 python bench.py --profile-json gpurun_out/prof_cfg4.json > gpurun_out/bench_cfg4.log 2>&1; echo bench $? >> gpurun_out/status.txt
for w in cfg3 cfg5; do timeout 600 python bench.py --workload $w --no-cpu-baseline --profile-json gpurun_out/prof_$w.json > gpurun_out/bench_$w.log 2>&1; echo bench_$w $? >> gpurun_out/status.txt; done
timeout 600 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_cfg4.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu.log 2>&1; echo ncu $? >> gpurun_out/status.txt
