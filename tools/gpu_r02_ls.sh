#!/bin/bash
# warp-scheduler fairness: 384-thread CTAs (one per SM), with / without a CTA barrier every 6 ops;
# 128-thread CTAs with the barrier.  2048 bits, one wave (56 832) and config 3 (2^18).
mkdir -p gpurun_out
for r in 1 2; do
for lib in paper_2410_18129_b200/libmpb.so tune/libmpb_t384.so tune/libmpb_t384ls.so tune/libmpb_ls128.so; do
for n in 56832 262144; do
echo "$lib $n" >> gpurun_out/ls_bench.log
MPB_LIB=$lib timeout 300 python tools/bench_algo.py --bits 2048 --count $n --algos 0 --redc 1 --check 4 >> gpurun_out/ls_bench.log 2>&1
done; done; done
echo done >> gpurun_out/ls_bench.log
