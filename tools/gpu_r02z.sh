#!/bin/bash
# squaring rows: focused tests, config 1/2 suite lines, one ncu --set full of the 1024-bit CIOS launch
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "sqr_rows or cios_register or mont_mul_sqr or crt" > gpurun_out/z_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/z_tests.log
python tools/bench_suite.py --configs 1,2 > gpurun_out/z_suite12.jsonl 2>&1
P="python tools/prof_modexp.py --bits 1024 --count 56832 --redc 2"
$P > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_modexp -c 1 -f -o gpurun_out/z_cios_sqr $P > gpurun_out/z_ncu.log 2>&1
echo done
