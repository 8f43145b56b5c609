#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/n_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/n_smoke.log
timeout 1200 python bench.py --workload config5 --steps 3 --warmup 3 > gpurun_out/n_c5.json 2> gpurun_out/n_c5.err; echo "rc=$?" >> gpurun_out/n_c5.err
timeout 300 python bench.py --gpus 2 --steps 1 > gpurun_out/n_g2.log 2>&1; echo "rc=$?" >> gpurun_out/n_g2.log
echo done
