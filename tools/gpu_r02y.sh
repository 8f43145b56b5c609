#!/bin/bash
mkdir -p gpurun_out
for lib in "" tune/libmpb_pu2.so "" tune/libmpb_pu2.so; do
  MPB_LIB=$lib timeout 300 python tools/bench_algo.py --bits 2048 --count 262144 --algos 0 --redc 1 --reps 3 --check 2 | sed "s|}|, \"lib\": \"$lib\"}|" >> gpurun_out/y_pu.jsonl
done
for lib in "" tune/libmpb_pu2.so; do
  MPB_LIB=$lib timeout 300 python tools/bench_algo.py --bits 4096 --count 65536 --algos 0 --redc 1 --reps 2 --check 2 | sed "s|}|, \"lib\": \"$lib\"}|" >> gpurun_out/y_pu.jsonl
done
echo done
