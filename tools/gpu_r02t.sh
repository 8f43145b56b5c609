#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/bench_algo.py --bits 1024 --count 1048576 --algos 0 --redc 2 --reps 3 --check 8 > gpurun_out/t_reg.jsonl
timeout 300 python tools/bench_suite.py --configs 6 --reps 3 > gpurun_out/t_crt.jsonl 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "cios_register or rsa" > gpurun_out/t_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t_pytest.log
echo done
