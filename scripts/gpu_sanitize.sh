# ONE compute-sanitizer tool per gpurun call (the profiling guide: never several tools, nor
# ncu, in one call), after the same program exited 0 without it.
# Usage: bash scripts/gpu_sanitize.sh <memcheck|racecheck|synccheck|initcheck>
mkdir -p gpurun_out
timeout 300 python scripts/sanitize_step.py > gpurun_out/sanitize_plain_$1.log 2>&1 &&
timeout 1500 compute-sanitizer --tool $1 --print-limit 20 python scripts/sanitize_step.py > gpurun_out/sanitizer_$1.log 2>&1; echo sanitizer_$1 $? >> gpurun_out/status_san.txt
