#!/bin/bash
# round-2 closing collection on the final kernels: smoke, all-config suite (configs 1-6, 9)
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/h_smoke.log
timeout 3000 python tools/bench_suite.py --configs 1,2,3,4,5,6,9 --reps 3 > gpurun_out/h_suite.jsonl 2> gpurun_out/h_suite.err
echo "rc=$?" >> gpurun_out/h_suite.err
