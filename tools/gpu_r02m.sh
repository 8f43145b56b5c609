#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "cios_register or modexp or fuzz or rsa" > gpurun_out/m_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/m_pytest.log
timeout 300 python tools/bench_algo.py --bits 1024 --count 1048576 --algos 0 --redc 2 --reps 3 --check 8 | sed 's|}|, "kernel": "register CIOS"}|' > gpurun_out/m_reg.jsonl
MPB_REG=0 timeout 300 python tools/bench_algo.py --bits 1024 --count 1048576 --algos 0 --redc 2 --reps 3 --check 4 | sed 's|}|, "kernel": "block-engine CIOS"}|' >> gpurun_out/m_reg.jsonl
timeout 300 python tools/bench_algo.py --bits 1024 --count 1048576 --algos 0 --redc 1 --reps 3 --check 4 | sed 's|}|, "kernel": "block-engine truncated"}|' >> gpurun_out/m_reg.jsonl
timeout 600 python tools/bench_suite.py --configs 6 --reps 3 > gpurun_out/m_crt.jsonl 2>&1
echo done
