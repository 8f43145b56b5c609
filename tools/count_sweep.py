"""Throughput of the 2048-bit, w = 5, truncated CT modexp against the batch size (whole and partial
waves of the 56 832 resident operands: 148 SMs x 3 CTAs x 128 threads), one sampled operand per
size checked against the oracle.  Output: JSON lines (profiles/r01_v7_count_sweep.jsonl)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import bench_suite as B  # noqa: E402

SLOTS = 148 * 3 * 128
for cnt in (1 << 14, 1 << 15, 1 << 16, SLOTS, 1 << 17, 2 * SLOTS, 1 << 18, 5 * SLOTS, 1 << 19, 1 << 20, 1 << 21,
            1 << 22):
    B.modexp_run(3, 2048, cnt, 2, redcs=((1, "truncated"),), check=1)
