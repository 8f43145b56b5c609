#!/bin/bash
mkdir -p gpurun_out
P="python tools/prof_modexp.py --bits 1024 --count 56832"
MPB_REG=2 $P > /dev/null 2>&1 && MPB_REG=2 ncu --set full --clock-control none --import-source on -k regex:k_modexp -c 1 -f -o gpurun_out/q_rtr $P > gpurun_out/q_ncu1.log 2>&1
MPB_REG=1 $P --redc 2 > /dev/null 2>&1 && MPB_REG=1 ncu --set full --clock-control none --import-source on -k regex:k_modexp -c 1 -f -o gpurun_out/q_cios $P --redc 2 > gpurun_out/q_ncu2.log 2>&1
echo done
