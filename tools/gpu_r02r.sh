#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "radix52" > gpurun_out/r_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r_pytest.log
timeout 300 python tools/bench_algo.py --bits 1024 --count 1048576 --algos 4 --redc 2 --reps 3 --check 8 | sed 's|}|, "kernel": "radix-2^52 register CIOS"}|' > gpurun_out/r_d52r.jsonl
timeout 300 python tools/bench_algo.py --bits 1024 --count 1048576 --algos 0 --redc 2 --reps 3 --check 2 | sed 's|}|, "kernel": "radix-2^32 register CIOS"}|' >> gpurun_out/r_d52r.jsonl
echo done
