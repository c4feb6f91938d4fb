# GPU suite with the per-test printouts (-s: per-tensor errors, argmax flips), smoke(), and
# one default bench line.  Usage: gpurun -- bash scripts/gpu_tests.sh [pytest -k expr]
mkdir -p gpurun_out
{ nproc; free -g; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; } > gpurun_out/box.txt 2>&1
K=${1:+-k "$1"}
eval timeout 2400 python -m pytest tests -m gpu -q -s -rA $K > gpurun_out/gpu_tests.log 2>&1; echo tests $? >> gpurun_out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $? >> gpurun_out/status.txt
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench $? >> gpurun_out/status.txt
