# ncu --set full of one kernel (name regex $2) of a kernel_ab.py run: bash scripts/gpu_ncu_kernel.sh <workload> <regex> [tag] [flags]
mkdir -p gpurun_out
TAG=${3:-k}
FL=${4:-0}
timeout 900 ncu -f --set full --import-source on --clock-control none -k "regex:$2" -c 1 -o /tmp/ncu_$TAG python scripts/kernel_ab.py --workload $1 --flags $FL --steps 1 > gpurun_out/ncu_$TAG.log 2>&1; echo ncu $? >> gpurun_out/status_$TAG.txt
ncu -i /tmp/ncu_$TAG.ncu-rep --page details --csv > gpurun_out/ncu_${TAG}_details.csv 2>/dev/null
ncu -i /tmp/ncu_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_${TAG}_raw.csv 2>/dev/null
ncu -i /tmp/ncu_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_${TAG}_sass.csv 2>/dev/null
cp /tmp/ncu_$TAG.ncu-rep gpurun_out/ 2>/dev/null
