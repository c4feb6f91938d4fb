# fixed per-step costs of small per-GPU batches: per-kernel tables of cfg5 at 1 and 8 images,
# graph-replayed step times of the strong-scaling shares, and the cfg3 bench line
# (64 one-image SGD steps).  Usage: gpurun -- bash scripts/gpu_small.sh [pytest -k expr]
mkdir -p gpurun_out
if [ -n "$1" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -rA -k "$1" > gpurun_out/small_tests.log 2>&1; echo tests $? >> gpurun_out/small_status.txt
fi
for n in 1 8; do
  timeout 600 python scripts/kernel_ab.py --workload cfg5 --images $n --flags 0 --json gpurun_out/small_cfg5_n$n.json > gpurun_out/small_cfg5_n$n.log 2>&1
done
for w in cfg5 cfg4; do
  timeout 600 python scripts/strong_scaling_probe.py --workload $w --graph > gpurun_out/small_probe_$w.txt 2>&1; echo probe_$w $? >> gpurun_out/small_status.txt
done
timeout 600 python bench.py --workload cfg3 --no-cpu-baseline > gpurun_out/small_bench_cfg3.log 2>&1; echo bench_cfg3 $? >> gpurun_out/small_status.txt
