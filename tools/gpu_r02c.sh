#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/hybrid_probe.py --bits 2048 > gpurun_out/c_hybrid.jsonl 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "fault_injection or one_thread_and" > gpurun_out/c_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c_pytest.log
timeout 300 python tools/bench_algo.py --bits 2048 --count 56832 --algos 4 --redc 1 --reps 1 --check 0 > gpurun_out/c_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_modexp_d52 -c 1 -o gpurun_out/c_d52 python tools/bench_algo.py --bits 2048 --count 56832 --algos 4 --redc 1 --reps 1 --check 0 > gpurun_out/c_ncu.log 2>&1
echo done
