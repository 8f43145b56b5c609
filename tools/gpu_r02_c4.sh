#!/bin/bash
# config 4 (4096 bits, 2^16, one wave): 4 x 128-thread CTAs per SM (shipped) vs one 448-thread CTA
# per SM vs 2 x 224 (same 128-register code; warp-scheduler fairness across CTAs)
mkdir -p gpurun_out
for r in 1 2; do
for lib in paper_2410_18129_b200/libmpb.so tune/libmpb_t448.so tune/libmpb_t224.so; do
echo "$lib" >> gpurun_out/c4_bench.log
MPB_LIB=$lib timeout 300 python tools/bench_algo.py --bits 4096 --count 65536 --algos 0 --redc 1 --check 4 >> gpurun_out/c4_bench.log 2>&1
done; done
echo done >> gpurun_out/c4_bench.log
