# A/B of kernel flags on the GPU box: bash scripts/gpu_ab.sh "<flags>" "<match>" [tag] [pytest -k]
mkdir -p gpurun_out
TAG=${3:-ab}
if [ -n "$4" ]; then
  timeout 1800 python -m pytest tests -m gpu -q -s -rA -k "$4" > gpurun_out/tests_$TAG.log 2>&1; echo tests $? >> gpurun_out/status_$TAG.txt
fi
for w in cfg4 cfg5; do
  timeout 600 python scripts/kernel_ab.py --workload $w --flags $1 --match $2 --json gpurun_out/ab_${w}_$TAG.json > gpurun_out/ab_${w}_$TAG.log 2>&1; echo ab_$w $? >> gpurun_out/status_$TAG.txt
done
