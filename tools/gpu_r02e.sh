#!/bin/bash
mkdir -p gpurun_out
B="timeout 300 python tools/bench_algo.py --bits 2048 --count 262144 --redc 1 --reps 3 --check 4"
$B --algos 0 > gpurun_out/e_l2.jsonl 2>&1
MPB_LIB=tune/libmpb_l2a.so $B --algos 0 >> gpurun_out/e_l2.jsonl 2>&1
MPB_LIB=tune/libmpb_l2b.so $B --algos 0 >> gpurun_out/e_l2.jsonl 2>&1
$B --algos 0 >> gpurun_out/e_l2.jsonl 2>&1
$B --algos 4 > gpurun_out/e_d52.jsonl 2>&1
MPB_LIB=tune/libmpb_d52m2.so $B --algos 4 >> gpurun_out/e_d52.jsonl 2>&1
MPB_LIB=tune/libmpb_d52m4.so $B --algos 4 >> gpurun_out/e_d52.jsonl 2>&1
for n in 2048 8192; do for c in 0 1 4 8; do MPB_COOP=$c timeout 300 python tools/bench_algo.py --bits 4096 --count $n --algos 0 --redc 1 --reps 2 --check 2 | sed "s/}/, \"coop\": $c}/" >> gpurun_out/e_coop.jsonl 2>&1; done; done
echo done
