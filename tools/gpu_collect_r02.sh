#!/bin/bash
# round-2 ncu evidence: full captures of the headline (2048-bit, 2^18) and config-4 (4096-bit, 2^16,
# register-Karatsuba blocks) exponentiations, and constant-time counts for the shipped 32-bit kernel,
# the 4096-bit Karatsuba-block kernel, the 8-lane cooperative kernel and the radix-2^52 kernel.
mkdir -p gpurun_out
P="python tools/prof_modexp.py"
$P --count 262144 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_modexp -c 1 -f -o gpurun_out/r02_modexp2048 $P --count 262144 > gpurun_out/r02_ncu_2048.log 2>&1
$P --bits 4096 --count 65536 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_modexp -c 1 -f -o gpurun_out/r02_modexp4096 $P --bits 4096 --count 65536 > gpurun_out/r02_ncu_4096.log 2>&1
M=smsp__inst_executed.sum,smsp__sass_inst_executed.sum,smsp__sass_inst_executed_op_branch.sum,smsp__sass_inst_executed_op_global_ld.sum,smsp__sass_inst_executed_op_global_st.sum,smsp__sass_inst_executed_op_ldgsts.sum,smsp__sass_inst_executed_op_shared_ld.sum,gpu__time_duration.sum
for spec in "2048 0 18944 k32" "4096 0 18944 k4096" "4096 0 1024 coop8" "2048 4 18944 d52"; do
  set -- $spec
  for c in zero ones random; do
    python tools/ct_check.py --cls $c --bits $1 --algo $2 --count $3 > /dev/null 2>&1 && \
    ncu --metrics $M --clock-control none -k regex:k_modexp -c 1 --csv --log-file gpurun_out/r02_ct_$4_$c.csv python tools/ct_check.py --cls $c --bits $1 --algo $2 --count $3 > /dev/null 2>&1
  done
done
echo done
