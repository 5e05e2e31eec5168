#!/usr/bin/env python
"""Build libdqmc.so with extra nvcc -D flags into tools/variants/libdqmc_<tag>.so
(A/B timing of compile-time alternatives; the product build is __graft_entry__.build).
Usage: python tools/build_variant.py TAG [-DNAME=VALUE ...]"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import __graft_entry__ as ge  # noqa: E402

tag, defs = sys.argv[1], sys.argv[2:]
obj = os.path.join(REPO, "build", "var_" + tag)
out = os.path.join(REPO, "tools", "variants", f"libdqmc_{tag}.so")
os.makedirs(obj, exist_ok=True)
os.makedirs(os.path.dirname(out), exist_ok=True)


def one(src):
    o = os.path.join(obj, os.path.splitext(src)[0] + ".o")
    if src.endswith(".cpp"):  # host-only unit
        cmd = ["g++", "-O3", "-std=c++17", "-fPIC", "-fvisibility=hidden", "-pthread", *defs, "-c", "-o", o,
               os.path.join(ge.CSRC, src)]
    else:
        cmd = [ge._nvcc(), *ge.NVCC_FLAGS, *defs, "-c", "-o", o, os.path.join(ge.CSRC, src)]
    r = subprocess.run(cmd, cwd=ge.CSRC, capture_output=True, text=True)
    if r.returncode:
        sys.stderr.write(r.stdout + r.stderr)
        raise SystemExit(f"nvcc failed on {src}")
    return o


with ThreadPoolExecutor(len(ge.SOURCES)) as ex:
    objs = list(ex.map(one, ge.SOURCES))
subprocess.run([ge._nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out, *objs], check=True)
print(out)
