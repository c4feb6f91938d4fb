# build, GPU tests, then per-layer live timings of cfg4/cfg5 for each env variant given
# usage: bash scripts/gpu_tb_ab.sh "<pytest -k expr or empty>" VAR=val ...
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 120 python scripts/run_step.py --workload cfg2 > gpurun_out/quick_cfg2.log 2>&1; echo quick_cfg2 $? >> gpurun_out/status.txt
grep -q "quick_cfg2 0" gpurun_out/status.txt || exit 1
KEXPR="$1"
timeout 900 python -m pytest tests -m gpu -x -q ${KEXPR:+-k "$KEXPR"} > gpurun_out/gpu_tests.log 2>&1; echo tests $? >> gpurun_out/status.txt
shift
for v in NONE=1 "$@"; do
  for w in cfg4 cfg5; do
    env $v timeout 300 python bench.py --workload $w --steps 5 --no-e2e --no-cpu-baseline --profile-json "gpurun_out/ab_${w}_${v}.json" > "gpurun_out/ab_${w}_${v}.log" 2>&1; echo "bench_${w}_${v} $?" >> gpurun_out/status.txt
  done
done
