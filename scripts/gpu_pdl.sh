# PDL A/B: the step time (no per-kernel events) with and without MPF_FLAG_NO_PDL, eager and graph
mkdir -p gpurun_out
T=${1:-pdl}
if [ -n "$2" ]; then
  timeout 1800 python -m pytest tests -m gpu -q -s -rA -k "$2" > gpurun_out/tests_$T.log 2>&1; echo tests $? >> gpurun_out/status_$T.txt
fi
for w in cfg5 cfg4 cfg3; do
  for fl in 0 0x200; do
    timeout 600 python scripts/strong_scaling_probe.py --workload $w --flags $fl >> gpurun_out/pdl_${w}_$T.log 2>&1
    timeout 600 python scripts/strong_scaling_probe.py --workload $w --flags $fl --graph >> gpurun_out/pdl_${w}_$T.log 2>&1
  done
done
