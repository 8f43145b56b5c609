#!/bin/bash
mkdir -p gpurun_out
M=smsp__sass_inst_executed.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second
for c in random ones zero random zero ones; do
  python tools/ct_check.py --cls $c --bits 1024 --redc 2 --count 18944 > /dev/null 2>&1 && \
  ncu --metrics $M --clock-control none -k regex:k_modexp -c 1 --csv python tools/ct_check.py --cls $c --bits 1024 --redc 2 --count 18944 2>/dev/null | grep -E "duration|inst_executed|per_second" | sed "s/^/$c,/" >> gpurun_out/ct3.csv
done
echo done
