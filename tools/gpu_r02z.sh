#!/bin/bash
# 2048-bit tail experiments at 2^18: 224-thread CTAs x 2; cooperative 2/4-lane tail
mkdir -p gpurun_out
for r in 1 2; do
echo "base" >> gpurun_out/z_bench.log
python tools/bench_algo.py --bits 2048 --count 262144 --algos 0 --redc 1 >> gpurun_out/z_bench.log 2>&1
echo "t224" >> gpurun_out/z_bench.log
MPB_LIB=tune/libmpb_t224.so python tools/bench_algo.py --bits 2048 --count 262144 --algos 0 --redc 1 >> gpurun_out/z_bench.log 2>&1
for tl in 2 4; do
echo "tail$tl" >> gpurun_out/z_bench.log
MPB_COOP_TAIL=$tl python tools/bench_algo.py --bits 2048 --count 262144 --algos 0 --redc 1 >> gpurun_out/z_bench.log 2>&1
done; done
