#!/bin/bash
# round-2 closing validation at HEAD: smoke, full GPU parity suite, default bench line
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/z_smoke.log
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/z_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/z_pytest.log
timeout 900 python bench.py > gpurun_out/z_bench.json 2> gpurun_out/z_bench.err
echo done
