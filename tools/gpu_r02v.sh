#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "karatsuba or config4 or one_thread_and" > gpurun_out/v_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/v_pytest.log
timeout 600 python tools/bench_algo.py --bits 4096 --count 65536 --algos 1,2,3 --redc 1 --reps 2 --check 4 > gpurun_out/v_kara.jsonl 2>&1
echo done
