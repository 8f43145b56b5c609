#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python tools/bench_suite.py --configs 1,2,3,4,5,6,7,8,9 --reps 3 > gpurun_out/f_suite.jsonl 2> gpurun_out/f_suite.err
echo done
