# tuning sweep: per-layer live timings of cfg4/cfg5 under different knobs
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for n in 4 2 1; do
  for w in cfg4 cfg5; do
    MPF_TC_NACC_MAX=$n timeout 600 python bench.py --workload $w --steps 3 --no-e2e --no-cpu-baseline --profile-json gpurun_out/sweep_${w}_nacc$n.json > gpurun_out/sweep_${w}_nacc$n.log 2>&1
  done
done
