#!/bin/bash
# round-2 final collection: parity suite, smoke, bench (+ launch list under ncu), all-config suite
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/f_smoke.log
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/f_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/f_pytest.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 500 > gpurun_out/f_clocks.csv &
SMI=$!
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
kill $SMI
timeout 2400 python tools/bench_suite.py --configs 1,2,3,4,5,6,7,8,9 --reps 3 > gpurun_out/f_suite.jsonl 2> gpurun_out/f_suite.err
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/f_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/f_ncu_launch.log 2>&1
echo done
