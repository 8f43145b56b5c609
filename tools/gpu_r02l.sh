#!/bin/bash
mkdir -p gpurun_out
for blk in 16 8; do
  MPB_BLOCK=$blk timeout 300 python tools/bench_algo.py --bits 1024 --count 1048576 --algos 0 --redc 1 --reps 3 --check 4 | sed "s|}|, \"block\": $blk}|" >> gpurun_out/l_1024.jsonl
  MPB_BLOCK=$blk timeout 300 python tools/bench_algo.py --bits 1024 --count 1048576 --algos 0 --redc 0 --reps 2 --check 2 | sed "s|}|, \"block\": $blk}|" >> gpurun_out/l_1024.jsonl
done
echo done
