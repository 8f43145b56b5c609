#!/bin/bash
# round-2 GPU check b: new parity tests, radix-2^52 and cooperative-tail A/B, full suite
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "theorem2 or radix52 or one_thread_and or redc_adversarial" --durations=10 > gpurun_out/b_pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/b_pytest_new.log
timeout 300 python tools/bench_algo.py --bits 2048 --count 262144 --algos 0,4 --redc 1 --reps 3 > gpurun_out/b_ab2048.jsonl 2>&1
timeout 300 python tools/bench_algo.py --bits 2048 --count 262144 --algos 0,4 --redc 0 --reps 2 >> gpurun_out/b_ab2048.jsonl 2>&1
timeout 300 python tools/bench_algo.py --bits 1024 --count 1048576 --algos 0,4 --redc 1 --reps 2 > gpurun_out/b_ab1024.jsonl 2>&1
for t in 0 2 4 8; do MPB_COOP_TAIL=$t timeout 300 python tools/bench_algo.py --bits 4096 --count 65536 --algos 0 --redc 1 --reps 2 --check 4 > gpurun_out/b_c4_tail$t.jsonl 2>&1; done
timeout 300 python tools/bench_algo.py --bits 4096 --count 65536 --algos 4 --redc 1 --reps 2 --check 4 > gpurun_out/b_c4_d52.jsonl 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu --durations=15 > gpurun_out/b_pytest_all.log 2>&1; echo "rc=$?" >> gpurun_out/b_pytest_all.log
echo done
