#!/bin/bash
# round-2 GPU check: parity suite, bench, DFMA v2 microbenchmark
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_smi.txt
./tools/microbench_dfma2 1965 > gpurun_out/a_dfma2.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/a_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/a_bench.json 2> gpurun_out/a_bench.err
echo done
