# Round-2 evidence in one call: GPU suite, smoke, bench lines (cfg4 default, cfg5, cfg3), live
# per-kernel tables, the reference arm, then ncu (the only profiling tool of this call): the
# launch list of the default bench command and a full capture of one cfg4 / cfg5 step, each
# right after the same command exited 0 without ncu.  Usage: bash scripts/gpu_evidence_r2.sh <tag>
mkdir -p gpurun_out
T=${1:-r2}
S=gpurun_out/status_$T.txt
timeout 2400 python -m pytest tests -m gpu -q -s -rA > gpurun_out/gpu_tests_$T.log 2>&1; echo tests $? >> $S
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo smoke $? >> $S
timeout 900 python bench.py > gpurun_out/bench_cfg4_$T.log 2>&1; echo bench $? >> $S
for w in cfg5 cfg3; do
  timeout 600 python bench.py --workload $w > gpurun_out/bench_${w}_$T.log 2>&1; echo bench_$w $? >> $S
done
for w in cfg4 cfg5 cfg3; do
  timeout 600 python bench.py --workload $w --steps 5 --no-e2e --no-cpu-baseline --profile-json gpurun_out/live_${w}_$T.json > gpurun_out/live_${w}_$T.log 2>&1; echo live_$w $? >> $S
done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference_$T.log 2>&1; echo ref $? >> $S
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-graph"
timeout 600 $B > gpurun_out/plain_bench_$T.log 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4_$T.csv $B > gpurun_out/ncu_launch_$T.log 2>&1; echo launches $? >> $S
for w in cfg4 cfg5; do
  timeout 300 python scripts/run_step.py --workload $w --order-json gpurun_out/order_${w}_$T.json > gpurun_out/order_${w}_$T.log 2>&1
  timeout 300 python scripts/run_step.py --workload $w > gpurun_out/plain_${w}_$T.log 2>&1 &&
  timeout 1500 ncu -f --set full --clock-control none --profile-from-start off -o /tmp/ncu_${w}_$T python scripts/run_step.py --workload $w > gpurun_out/ncu_${w}_$T.log 2>&1; echo ncu_$w $? >> $S
  ncu -i /tmp/ncu_${w}_$T.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/ncu_${w}_raw_$T.csv.gz
done
