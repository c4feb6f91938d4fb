# bench, then full ncu captures of one step (cfg5 and cfg4); only text summaries come back
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for w in cfg4 cfg5 cfg3; do timeout 600 python bench.py --workload $w --no-cpu-baseline --profile-json gpurun_out/prof_$w.json > gpurun_out/bench_$w.log 2>&1; echo bench_$w $? >> gpurun_out/status.txt; done
for w in cfg5 cfg4; do
  timeout 300 python scripts/run_step.py --workload $w > gpurun_out/plain_$w.log 2>&1 &&
  timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -f -o /tmp/ncu_$w python scripts/run_step.py --workload $w > gpurun_out/ncu_$w.log 2>&1; echo ncu_$w $? >> gpurun_out/status.txt
  ncu -i /tmp/ncu_$w.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/ncu_${w}_raw.csv.gz
  ncu -i /tmp/ncu_$w.ncu-rep --page details --csv 2>/dev/null | gzip > gpurun_out/ncu_${w}_details.csv.gz
done
ls -la gpurun_out
