#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/bench_algo.py --bits 4096 --count 65536 --algos 0 --redc 1 --reps 3 --check 4 > gpurun_out/k_c4.jsonl 2>&1
timeout 300 python tools/bench_algo.py --bits 4096 --count 65536 --algos 0 --redc 0 --reps 2 --check 4 >> gpurun_out/k_c4.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "config4 or theorem2 or modexp" > gpurun_out/k_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/k_pytest.log
echo done
