#!/bin/bash
# constant-time counts for the squaring-row CIOS kernels (1024-bit register, 2048-bit block engine)
mkdir -p gpurun_out
M=smsp__inst_executed.sum,smsp__sass_inst_executed.sum,smsp__sass_inst_executed_op_branch.sum,smsp__sass_inst_executed_op_global_ld.sum,smsp__sass_inst_executed_op_global_st.sum,smsp__sass_inst_executed_op_ldgsts.sum,smsp__sass_inst_executed_op_shared_ld.sum,gpu__time_duration.sum
for spec in "1024 2 18944 reg1024" "2048 2 18944 cios2048"; do
  set -- $spec
  for c in zero ones random; do
    python tools/ct_check.py --cls $c --bits $1 --redc $2 --count $3 > /dev/null 2>&1 && \
    ncu --metrics $M --clock-control none -k regex:k_modexp -c 1 --csv --log-file gpurun_out/r02_ct_$4_$c.csv python tools/ct_check.py --cls $c --bits $1 --redc $2 --count $3 > /dev/null 2>&1
  done
done
timeout 900 python -m pytest tests -m gpu -x -q -k "sqr_rows" > gpurun_out/ct2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ct2_tests.log
echo done
