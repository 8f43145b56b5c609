#!/bin/bash
# CT scan variants of the 1024-bit register CIOS (tools/build_variant.py scan_*)
mkdir -p gpurun_out
for r in 1 2; do
for lib in paper_2410_18129_b200/libmpb.so tune/libmpb_scan_u2.so tune/libmpb_scan_u4g4.so tune/libmpb_scan_ldg.so tune/libmpb_scan_u2ldg.so tune/libmpb_scan_u4g4ldg.so; do
echo "$lib" >> gpurun_out/z_bench.log
MPB_LIB=$lib python tools/bench_algo.py --bits 1024 --count 1048576 --algos 0 --redc 2 >> gpurun_out/z_bench.log 2>&1
done; done
