#!/bin/bash
# one-wave instances (inst_W384 / inst_W448): parity suite + A/B against MPB_ONEWAVE=0
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ow_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ow_pytest.log
for ow in 1 0; do
for spec in "4096 65536" "2048 56832" "2048 32768" "2048 16384" "3072 40000" "1024 100000" "2048 262144"; do
set -- $spec
echo "onewave=$ow bits=$1 count=$2" >> gpurun_out/ow_bench.log
MPB_ONEWAVE=$ow timeout 300 python tools/bench_algo.py --bits $1 --count $2 --algos 0 --redc 1 --check 4 >> gpurun_out/ow_bench.log 2>&1
done; done
echo done >> gpurun_out/ow_bench.log
