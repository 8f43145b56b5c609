#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "hybrid or radix52" > gpurun_out/d_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/d_pytest.log
timeout 300 python tools/bench_algo.py --bits 2048 --count 262144 --algos 0,5 --redc 1 --reps 3 > gpurun_out/d_hybrid.jsonl 2>&1
for f in 0.5 0.6 0.75 0.8; do MPB_HYBRID_FRAC=$f timeout 300 python tools/bench_algo.py --bits 2048 --count 262144 --algos 5 --redc 1 --reps 2 --check 2 >> gpurun_out/d_hybrid.jsonl 2>&1; done
echo done
