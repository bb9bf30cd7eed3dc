"""Build (here, nvcc cross-compiles) and run one of the scripts/*.cu microbenchmarks that
export `extern "C" void run_all()`:  python scripts/run_microbench.py ring_bench"""
import ctypes
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
name = sys.argv[1]
so = os.path.join(HERE, name + ".so")
if "--build" in sys.argv or not os.path.exists(so):
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared",
                    "-Xcompiler", "-fPIC", "-o", so, os.path.join(HERE, name + ".cu")], check=True)
if "--build" in sys.argv:
    sys.exit(0)
fn = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else "run_all"
getattr(ctypes.CDLL(so), fn)()
