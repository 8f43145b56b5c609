#!/bin/bash
mkdir -p gpurun_out
MPB_BENCH_SHARE_GPU=1 timeout 1500 python bench.py --gpus 2 --workload config5 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/x_c5g2.json 2> gpurun_out/x_c5g2.err; echo "rc=$?" >> gpurun_out/x_c5g2.err
MPB_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 4 --workload config5 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/x_c5g4.json 2> gpurun_out/x_c5g4.err; echo "rc=$?" >> gpurun_out/x_c5g4.err
echo done
