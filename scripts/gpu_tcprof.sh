set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
MPF_TC_PROF=1 timeout 300 python scripts/run_step.py --workload cfg5 --warmup 1 > gpurun_out/tcprof_cfg5.log 2>&1
MPF_TC_PROF=1 timeout 300 python scripts/run_step.py --workload cfg4 --warmup 1 > gpurun_out/tcprof_cfg4.log 2>&1
