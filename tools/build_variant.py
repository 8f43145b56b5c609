"""Build a tuning variant of libmpb.so into tune/ (git-ignored): recompile the listed translation
units with extra nvcc flags, link them with the other up-to-date objects of the main build.

  python tools/build_variant.py NAME "-DMPB_L2HINT=1" inst_C16.cu [inst_D52.cu ...]
  MPB_LIB=tune/libmpb_NAME.so python tools/bench_algo.py ...
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as g  # noqa: E402

name, flags, units = sys.argv[1], sys.argv[2].split(), sys.argv[3:]
g.build_cuda()
objdir = os.path.join(g.PKG, "build")
tdir = os.path.join(ROOT, "tune", name)
os.makedirs(tdir, exist_ok=True)
objs, procs = [], []
for src in g._sources():
    b = os.path.basename(src)[:-3]
    if os.path.basename(src) in units:
        o = os.path.join(tdir, b + ".o")
        procs.append(subprocess.Popen([os.environ.get("NVCC", "nvcc"), *g.NVCC_FLAGS, *flags, "-c", src, "-o", o],
                                      stdout=open(o + ".log", "w"), stderr=subprocess.STDOUT))
        objs.append(o)
    else:
        objs.append(os.path.join(objdir, b + ".o"))
for p in procs:
    assert p.wait() == 0, "nvcc failed"
lib = os.path.join(ROOT, "tune", f"libmpb_{name}.so")
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib, *objs, "-lcudart"])
print(lib)
