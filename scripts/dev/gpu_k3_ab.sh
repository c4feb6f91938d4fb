mkdir -p gpurun_out
T=$1
timeout 900 python -m pytest tests -m gpu -q -s -rA -k "band_matches_blocks or k3_scatter or bench_step_cfg5" > gpurun_out/tests_$T.log 2>&1; echo tests $? >> gpurun_out/status_$T.txt
timeout 600 python scripts/kernel_ab.py --workload cfg5 --flags 0 0x800 0 0x800 --match mpf_bwd --steps 5 > gpurun_out/ab_cfg5_$T.log 2>&1; echo ab $? >> gpurun_out/status_$T.txt
timeout 600 python scripts/step_ab.py --workload cfg5 --flags 0 0x800 --rounds 4 --steps 5 > gpurun_out/step_cfg5_$T.log 2>&1; echo step $? >> gpurun_out/status_$T.txt
