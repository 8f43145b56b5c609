#!/bin/bash
mkdir -p gpurun_out
S="--section SpeedOfLight --section MemoryWorkloadAnalysis --section InstructionStats --section WarpStateStats --section ComputeWorkloadAnalysis --section LaunchStats --section Occupancy"
P="python tools/prof_modexp.py --bits 4096 --count 18944"
$P --algo 2 > /dev/null 2>&1 && ncu $S --clock-control none -k regex:k_modexp -c 1 -f -o gpurun_out/w_kara2 $P --algo 2 > gpurun_out/w_ncu1.log 2>&1
$P --algo 1 > /dev/null 2>&1 && ncu $S --clock-control none -k regex:k_modexp -c 1 -f -o gpurun_out/w_sb $P --algo 1 > gpurun_out/w_ncu2.log 2>&1
ls -la gpurun_out
echo done
