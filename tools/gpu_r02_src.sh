#!/bin/bash
# source-level ncu capture of the headline kernel (128-thread k_modexp<16,1,4,0,3>, 2 waves)
mkdir -p gpurun_out
P="python tools/prof_modexp.py --count 113664"
$P > /dev/null 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_modexp -c 1 -f -o gpurun_out/s_modexp2048 $P > gpurun_out/s_ncu.log 2>&1
ncu -i gpurun_out/s_modexp2048.ncu-rep --page source --csv --print-source sass > gpurun_out/s_sass.csv 2>/dev/null
MPB_TESTS=1 timeout 600 python -m pytest tests -m gpu -x -q -k "register_truncated" > gpurun_out/s_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s_tests.log
echo done
