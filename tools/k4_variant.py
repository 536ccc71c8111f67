"""Link a variant of the library whose policy_mlp.cu object is compiled with
extra flags (the other objects from the normal build): quick K4 experiments.
usage: python tools/k4_variant.py NAME "-DFLAG=1 ..."  -> tools/exp/lib_NAME.so"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1810_05762_b200 import build as B  # noqa: E402

B.build()
name, flags = sys.argv[1], sys.argv[2].split()
obj = os.path.join(B.BUILD, f"policy_mlp_{name}.o")
subprocess.run([B.NVCC] + B.ARCH + B.FLAGS + flags + ["-c", os.path.join(B.CSRC, "policy_mlp.cu"), "-o", obj],
               check=True, capture_output=True)
objs = [os.path.join(B.BUILD, s + ".o") for s in B.SOURCES if s != "policy_mlp.cu"] + [obj]
out = os.path.join(ROOT, "tools", "exp", f"lib_{name}.so")
subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-o", out] + objs + ["-lcudart"], check=True)
print("built", out)
