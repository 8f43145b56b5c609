#!/bin/bash
# round-2 final collection: parity suite, bench, all-config suite
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu --durations=10 > gpurun_out/s_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/s_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/s_bench.json 2> gpurun_out/s_bench.err
timeout 2400 python tools/bench_suite.py --configs 1,2,3,4,5,6,7,8,9 --reps 3 > gpurun_out/s_suite.jsonl 2> gpurun_out/s_suite.err
echo done
