#!/bin/bash
mkdir -p gpurun_out
for lib in "" tune/libmpb_m4.so; do
  MPB_LIB=$lib timeout 300 python tools/bench_algo.py --bits 4096 --count 65536 --algos 0 --redc 1 --reps 2 --check 2 | sed "s|}|, \"lib\": \"$lib\"}|" >> gpurun_out/j_m4.jsonl
  MPB_LIB=$lib timeout 300 python tools/bench_algo.py --bits 2048 --count 262144 --algos 0 --redc 1 --reps 2 --check 2 | sed "s|}|, \"lib\": \"$lib\"}|" >> gpurun_out/j_m4.jsonl
done
echo done
