"""One launch of each stand-alone product / Montgomery kernel at 2048 bits (56 832 operands) for
`ncu --metrics smsp__inst_executed.sum` -- the source of profiles/r01_instr_per_product.txt."""
import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2410_18129_b200 import inputs as I, mpb
import os
bits, count = int(os.environ.get("BITS", "2048")), 56832
a, b = I.mul_inputs(config=4, count=count, bits=bits)
da, db = mpb.to_device(a), mpb.to_device(b)
N, x, y = I.montmul_inputs(config=2, count=count, bits=bits)
dN, dx, dy = (mpb.to_device(v) for v in (N, x, y))
Np, _ = mpb.mont_batch_setup(dN, bits)
mpb.mp_batch_mul(da, db, bits, 1)
mpb.mp_batch_sqr(da, bits, 1)
for r in (1, 0, 2):
    mpb.mont_batch_mul(dx, dy, dN, Np, bits, redc=r)
    mpb.mont_batch_sqr(dx, dN, Np, bits, redc=r)
torch.cuda.synchronize()
print("ok")
