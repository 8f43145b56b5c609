#!/bin/bash
mkdir -p gpurun_out
for lib in "" tune/libmpb_mov0.so "" tune/libmpb_mov0.so; do
  MPB_LIB=$lib timeout 300 python tools/bench_algo.py --bits 2048 --count 262144 --algos 0 --redc 1 --reps 3 --check 2 | sed "s|}|, \"lib\": \"$lib\"}|" >> gpurun_out/o_mov.jsonl
done
for lib in "" tune/libmpb_mov0.so; do
  MPB_LIB=$lib timeout 300 python tools/bench_algo.py --bits 4096 --count 65536 --algos 0 --redc 1 --reps 2 --check 2 | sed "s|}|, \"lib\": \"$lib\"}|" >> gpurun_out/o_mov.jsonl
  MPB_LIB=$lib timeout 300 python tools/bench_algo.py --bits 1024 --count 1048576 --algos 0 --redc 1 --reps 2 --check 2 | sed "s|}|, \"lib\": \"$lib\"}|" >> gpurun_out/o_mov.jsonl
done
echo done
