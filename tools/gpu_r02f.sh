#!/bin/bash
mkdir -p gpurun_out
./tools/microbench_kara16 1965 > gpurun_out/f_kara16.txt 2>&1
B="timeout 300 python tools/bench_algo.py --bits 2048 --count 262144 --redc 1 --reps 3 --check 4 --algos 4"
MPB_LIB=tune/libmpb_d52c4m4.so $B > gpurun_out/f_d52.jsonl 2>&1
MPB_LIB=tune/libmpb_d52c4m5.so $B >> gpurun_out/f_d52.jsonl 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu --durations=5 > gpurun_out/f_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/f_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
echo done
