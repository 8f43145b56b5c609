#!/bin/bash
mkdir -p gpurun_out
for lib in "" tune/libmpb_c12k.so tune/libmpb_c12w.so tune/libmpb_c12kw.so; do
  MPB_LIB=$lib timeout 300 python tools/bench_algo.py --bits 4108 --count 65536 --algos 0 --redc 1 --reps 2 --check 4 | sed "s|}|, \"lib\": \"$lib\"}|" >> gpurun_out/u_4108.jsonl
done
echo done
