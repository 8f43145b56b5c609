#!/bin/bash
# config 4 on the 448-thread one-wave instance: register-Karatsuba blocks (shipped) vs schoolbook blocks
# vs a 16-load table-scan group (fewer live registers)
mkdir -p gpurun_out
for r in 1 2; do
for lib in paper_2410_18129_b200/libmpb.so tune/libmpb_w448nk.so tune/libmpb_w448g4.so; do
echo "$lib" >> gpurun_out/c4b_bench.log
MPB_LIB=$lib timeout 300 python tools/bench_algo.py --bits 4096 --count 65536 --algos 0 --redc 1 --check 2 >> gpurun_out/c4b_bench.log 2>&1
done; done
echo done >> gpurun_out/c4b_bench.log
