#!/bin/bash
# L2 bulk prefetch of the window table ahead of the CT scan: A/B (pf1..3: 32 lanes x 1/32 of the
# table, 1..3 squarings ahead; pfo32 / pfo8: one lane, the whole table / its first quarter)
mkdir -p gpurun_out
for r in 1 2; do
for lib in paper_2410_18129_b200/libmpb.so tune/libmpb_pfo32.so tune/libmpb_pfo8.so; do
echo "$lib" >> gpurun_out/pf_bench.log
MPB_LIB=$lib timeout 300 python tools/bench_algo.py --bits 2048 --count 262144 --algos 0 --redc 1 --check 8 >> gpurun_out/pf_bench.log 2>&1
done; done
echo done >> gpurun_out/pf_bench.log
