# MPF_TC_PROF role timings of one cfg4 step under forced CTA-pair / single modes
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for m in 0 1; do
  MPF_TC_PAIR=$m MPF_TC_PROF=1 timeout 300 python scripts/run_step.py --workload ${1:-cfg4} --warmup 1 > gpurun_out/tcprof_pair$m.log 2>&1
done
