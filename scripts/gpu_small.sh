# per-kernel tables of cfg5 at 1 and 8 images (fixed per-kernel costs of small per-GPU batches)
mkdir -p gpurun_out
for n in 1 8; do
  timeout 600 python scripts/kernel_ab.py --workload cfg5 --images $n --flags 0 --json gpurun_out/small_cfg5_n$n.json > gpurun_out/small_cfg5_n$n.log 2>&1
done
