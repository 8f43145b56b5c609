#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/cta_times.py 56832 113664 262144 > gpurun_out/cta_times.jsonl 2>&1
echo rc=$? >> gpurun_out/cta_times.jsonl
