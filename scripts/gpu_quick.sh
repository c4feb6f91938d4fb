# Quick iteration on the GPU box: selected GPU tests (-k expr, printouts kept) and live
# per-kernel tables of cfg4 / cfg5 (bench.py --profile-json).
# Usage: gpurun -- bash scripts/gpu_quick.sh "<pytest -k expr>" [tag]
mkdir -p gpurun_out
TAG=${2:-q}
if [ -n "$1" ]; then
  timeout 1800 python -m pytest tests -m gpu -q -s -rA -k "$1" > gpurun_out/tests_$TAG.log 2>&1; echo tests $? >> gpurun_out/status_$TAG.txt
fi
for w in cfg4 cfg5; do
  timeout 600 python bench.py --workload $w --steps 5 --no-e2e --no-cpu-baseline --profile-json gpurun_out/live_${w}_$TAG.json > gpurun_out/live_${w}_$TAG.log 2>&1; echo live_$w $? >> gpurun_out/status_$TAG.txt
done
