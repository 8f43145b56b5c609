#!/bin/bash
# one-wave instances incl. 4108 bits (C = 12): new parity tests + A/B
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "onewave or one_thread or config4 or modexp_karatsuba" > gpurun_out/ow2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ow2_pytest.log
for ow in 1 0; do
for spec in "4108 65536" "4108 50000" "4096 65536"; do
set -- $spec
echo "onewave=$ow bits=$1 count=$2" >> gpurun_out/ow2_bench.log
MPB_ONEWAVE=$ow timeout 300 python tools/bench_algo.py --bits $1 --count $2 --algos 0 --redc 1 --check 2 >> gpurun_out/ow2_bench.log 2>&1
done; done
echo done >> gpurun_out/ow2_bench.log
