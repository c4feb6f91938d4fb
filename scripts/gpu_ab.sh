# A/B of environment knobs on per-layer live timings (cfg4, cfg5)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in "$@"; do
  for w in cfg4 cfg5; do
    env $v timeout 300 python bench.py --workload $w --steps 3 --no-e2e --no-cpu-baseline --profile-json "gpurun_out/ab_${w}_${v}.json" > "gpurun_out/ab_${w}_${v}.log" 2>&1
  done
done
