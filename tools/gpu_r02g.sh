#!/bin/bash
mkdir -p gpurun_out
for bits in 2048 1024 3072 4096; do
  case $bits in 1024) n=1048576;; 2048) n=262144;; 3072) n=131072;; 4096) n=65536;; esac
  timeout 300 python tools/bench_algo.py --bits $bits --count $n --algos 0 --redc 1 --reps 3 --check 4 | sed 's/}/, "lib": "kara-block"}/' >> gpurun_out/g_ab.jsonl 2>&1
  MPB_LIB=tune/libmpb_kb0.so timeout 300 python tools/bench_algo.py --bits $bits --count $n --algos 0 --redc 1 --reps 3 --check 4 | sed 's/}/, "lib": "schoolbook-block"}/' >> gpurun_out/g_ab.jsonl 2>&1
done
timeout 1500 python -m pytest tests -x -q -m gpu --durations=5 > gpurun_out/g_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g_pytest.log
echo done
