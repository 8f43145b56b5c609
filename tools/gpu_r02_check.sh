#!/bin/bash
# re-entry check: smoke, GPU parity suite, bench line at HEAD
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/c_smoke.log
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/c_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/c_bench.json 2> gpurun_out/c_bench.err
echo done
