#!/bin/bash
# stand-alone 1024-bit truncated MontMul / MontSqr: block engine vs register-resident truncated kernel
mkdir -p gpurun_out
for r in 1 2; do for p in 0 1; do
MPB_REG_TRUNC=$p timeout 300 python tools/ab_montop.py --bits 1024 --redc 1 >> gpurun_out/rtr_ab.jsonl 2>&1
done; done
MPB_REG_TRUNC=1 timeout 900 python -m pytest tests -m gpu -x -q -k "mont_mul_sqr or config2 or fuzz or empty" > gpurun_out/rtr_tests.log 2>&1; echo "rc=$?" >> gpurun_out/rtr_tests.log
echo done >> gpurun_out/rtr_ab.jsonl
