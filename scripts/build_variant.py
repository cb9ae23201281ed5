"""Build a tuning/instrumentation variant of libbpt.so with extra nvcc flags (not the product):
  python scripts/build_variant.py <out.so> -DBPT_HIST -DBPT_WIN_IC=4 ...
Load it with BPT_LIB=<out.so>."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as ge  # noqa: E402

out, extra = sys.argv[1], sys.argv[2:]
bdir = os.path.join(ROOT, "variants", "obj", os.path.basename(out))
os.makedirs(bdir, exist_ok=True)
objs = []
for src in ge.SOURCES:
    obj = os.path.join(bdir, os.path.splitext(src)[0] + ".o")
    subprocess.run([ge.NVCC, *ge.NVCC_FLAGS, *extra, "-c", os.path.join(ge.CSRC, src), "-o", obj], check=True,
                   capture_output=True)
    objs.append(obj)
subprocess.run([ge.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out, *objs,
                *ge._nccl_link_flags()], check=True)
print(out)
