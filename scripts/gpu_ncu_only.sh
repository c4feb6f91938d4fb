# The ncu part of scripts/gpu_evidence_r2.sh alone (launch list of the default bench command,
# full captures of one cfg4 / cfg5 step), each right after the same command exited 0 without
# ncu.  Usage: bash scripts/gpu_ncu_only.sh <tag>
mkdir -p gpurun_out
T=${1:-r2}
S=gpurun_out/status_$T.txt
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph"
timeout 600 $B > gpurun_out/plain_bench_$T.log 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4_$T.csv $B > gpurun_out/ncu_launch_$T.log 2>&1; echo launches $? >> $S
for w in cfg4 cfg5; do
  timeout 300 python scripts/run_step.py --workload $w --order-json gpurun_out/order_${w}_$T.json > gpurun_out/order_${w}_$T.log 2>&1
  timeout 300 python scripts/run_step.py --workload $w > gpurun_out/plain_${w}_$T.log 2>&1 &&
  timeout 1500 ncu -f --set full --clock-control none --profile-from-start off -o /tmp/ncu_${w}_$T python scripts/run_step.py --workload $w > gpurun_out/ncu_${w}_$T.log 2>&1; echo ncu_$w $? >> $S
  ncu -i /tmp/ncu_${w}_$T.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/ncu_${w}_raw_$T.csv.gz
done
