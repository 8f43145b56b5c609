#!/bin/bash
# round-2 final collection (current kernels): bench line, launch list, ncu full of the config-4
# one-wave (448-thread) launch, constant-time counts of the one-wave instances
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/g_clocks.csv &
SMI=$!
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err
kill $SMI
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/g_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/g_ncu_launch.log 2>&1
P="python tools/prof_modexp.py"
$P --bits 4096 --count 65536 > /dev/null 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_modexp -c 1 -f -o gpurun_out/g_modexp4096_w448 $P --bits 4096 --count 65536 > gpurun_out/g_ncu_4096.log 2>&1
M=smsp__inst_executed.sum,smsp__sass_inst_executed.sum,smsp__sass_inst_executed_op_branch.sum,smsp__sass_inst_executed_op_global_ld.sum,smsp__sass_inst_executed_op_global_st.sum,smsp__sass_inst_executed_op_ldgsts.sum,smsp__sass_inst_executed_op_shared_ld.sum,gpu__time_duration.sum
for spec in "2048 18944 w384" "4096 65536 w448"; do
  set -- $spec
  for c in zero ones random; do
    python tools/ct_check.py --cls $c --bits $1 --count $2 > /dev/null 2>&1 && \
    timeout 600 ncu --metrics $M --clock-control none -k regex:k_modexp -c 1 --csv --log-file gpurun_out/r02_ct_$3_$c.csv python tools/ct_check.py --cls $c --bits $1 --count $2 > /dev/null 2>&1
  done
done
echo done
