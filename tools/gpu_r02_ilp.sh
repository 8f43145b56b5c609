#!/bin/bash
mkdir -p gpurun_out
timeout 300 ./tools/mb_ilp2 > gpurun_out/ilp2.jsonl 2>&1
echo rc=$? >> gpurun_out/ilp2.jsonl
