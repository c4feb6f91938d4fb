# strong-scaling probe (eager and CUDA graph) + an A/B of flags: bash scripts/gpu_probe.sh "<flags>" "<match>" <tag>
mkdir -p gpurun_out
for w in cfg5 cfg4; do
  timeout 600 python scripts/strong_scaling_probe.py --workload $w > gpurun_out/probe_${w}_$3.log 2>&1
  timeout 600 python scripts/strong_scaling_probe.py --workload $w --graph >> gpurun_out/probe_${w}_$3.log 2>&1
done
for w in cfg4 cfg5; do
  timeout 600 python scripts/kernel_ab.py --workload $w --flags $1 --match $2 > gpurun_out/ab_${w}_$3.log 2>&1
done
