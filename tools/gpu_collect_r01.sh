set -x
python bench.py > gpurun_out/bench_final.log 2>&1; echo bench rc=$?
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python tools/prof_modexp.py --count 262144 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_modexp -c 1 -f -o gpurun_out/modexp_bench python tools/prof_modexp.py --count 262144 > gpurun_out/ncu_full.log 2>&1
M=smsp__inst_executed.sum,smsp__sass_inst_executed.sum,smsp__sass_inst_executed_op_branch.sum,smsp__sass_inst_executed_op_global_ld.sum,smsp__sass_inst_executed_op_global_st.sum,smsp__sass_inst_executed_op_ldgsts.sum,smsp__sass_inst_executed_op_shared_ld.sum,gpu__time_duration.sum
for c in zero ones random; do python tools/ct_check.py --cls $c > /dev/null 2>&1 && ncu --metrics $M --clock-control none -k regex:k_modexp -c 1 --csv --log-file gpurun_out/ct_$c.csv python tools/ct_check.py --cls $c > /dev/null 2>&1; done
ls -la gpurun_out
