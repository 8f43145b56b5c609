#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "truncated_register or cios_register" > gpurun_out/p_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/p_pytest.log
for reg in 2 1; do
  MPB_REG=$reg timeout 300 python tools/bench_algo.py --bits 1024 --count 1048576 --algos 0 --redc 1 --reps 3 --check 8 | sed "s|}|, \"MPB_REG\": $reg}|" >> gpurun_out/p_rtr.jsonl
done
echo done
