# ncu --set full of selected kernels of one step; exports raw + source pages as text
# usage: bash scripts/gpu_ncu1.sh <workload> <kernel-regex> <count> [skip]
set -x
w=$1; rx=$2; cnt=$3; skip=${4:-0}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python scripts/run_step.py --workload $w > gpurun_out/plain_$w.log 2>&1 &&
rm -f /tmp/ncu_k.ncu-rep; timeout 1200 ncu -f --set full --clock-control none --import-source on --profile-from-start off -k regex:"$rx" -s $skip -c $cnt -o /tmp/ncu_k python scripts/run_step.py --workload $w > gpurun_out/ncu_k.log 2>&1; echo ncu $? >> gpurun_out/status.txt
ncu -i /tmp/ncu_k.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/ncu_k_raw.csv.gz
for i in $(seq 0 $((cnt-1))); do
  ncu -i /tmp/ncu_k.ncu-rep --page source --csv --print-source sass --launch-skip $i --launch-count 1 2>/dev/null | gzip > gpurun_out/ncu_k_src$i.csv.gz
done
