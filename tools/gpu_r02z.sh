#!/bin/bash
# block-engine CIOS squaring rows: parity subset + A/B (tune/libmpb_csq0.so = multiplication rows)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "cios or mont_mul_sqr or modexp or crt" > gpurun_out/z_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/z_tests.log
for r in 1 2; do
for lib in paper_2410_18129_b200/libmpb.so tune/libmpb_csq0.so; do
echo "$lib" >> gpurun_out/z_bench.log
MPB_LIB=$lib python tools/bench_algo.py --bits 2048 --count 262144 --algos 0 --redc 2 >> gpurun_out/z_bench.log 2>&1
MPB_LIB=$lib python tools/bench_algo.py --bits 4096 --count 65536 --algos 0 --redc 2 >> gpurun_out/z_bench.log 2>&1
MPB_LIB=$lib python tools/bench_algo.py --bits 3072 --count 131072 --algos 0 --redc 2 >> gpurun_out/z_bench.log 2>&1
done; done
