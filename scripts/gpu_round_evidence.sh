# full round evidence in one call: GPU tests, smoke, default bench line (cfg4), per-workload
# bench lines and live per-kernel tables (cfg3/cfg4/cfg5), the reference arm, the ncu
# launch list of the default bench command and full ncu captures of one cfg4 / cfg5 step
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests $? >> gpurun_out/status.txt
bash scripts/gpu_evidence.sh
for w in cfg3 cfg5; do
  timeout 600 python bench.py --workload $w > gpurun_out/bench_$w.log 2>&1; echo bench_$w $? >> gpurun_out/status.txt
done
for w in cfg3 cfg4 cfg5; do
  timeout 600 python bench.py --workload $w --steps 5 --no-e2e --no-cpu-baseline --profile-json gpurun_out/live_$w.json > gpurun_out/live_$w.log 2>&1; echo live_$w $? >> gpurun_out/status.txt
done
timeout 300 python scripts/api_tour.py > gpurun_out/api_tour.log 2>&1; echo api_tour $? >> gpurun_out/status.txt
