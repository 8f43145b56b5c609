#!/bin/bash
# persistent exponentiation (fixed workspace slots) with / without an L2 persisting window: A/B + parity
mkdir -p gpurun_out
nvidia-smi -q | grep -i -B1 -A3 "persist" | head -20 > gpurun_out/ps_attr.log
MPB_PERSIST=1 timeout 900 python -m pytest tests -m gpu -x -q -k "modexp and not radix52 and not hybrid" > gpurun_out/ps_tests.log 2>&1
echo "rc=$?" >> gpurun_out/ps_tests.log
for r in 1 2; do
echo base >> gpurun_out/ps_bench.log
timeout 300 python tools/bench_algo.py --bits 2048 --count 262144 --algos 0 --redc 1 --check 8 >> gpurun_out/ps_bench.log 2>&1
echo persist >> gpurun_out/ps_bench.log
MPB_PERSIST=1 timeout 300 python tools/bench_algo.py --bits 2048 --count 262144 --algos 0 --redc 1 --check 8 >> gpurun_out/ps_bench.log 2>&1
for mb in 32 64 96; do
echo "persist l2win $mb" >> gpurun_out/ps_bench.log
MPB_PERSIST=1 MPB_L2WIN=$mb timeout 300 python tools/bench_algo.py --bits 2048 --count 262144 --algos 0 --redc 1 --check 8 >> gpurun_out/ps_bench.log 2>&1
done; done
echo done >> gpurun_out/ps_bench.log
