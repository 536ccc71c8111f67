"""In-tree build of the CUDA extension libstampede_b200.so (sm_100a).

Each translation unit is compiled by nvcc in parallel, then linked with
``nvcc -shared``.  The result lives next to this file so it travels with the
repo snapshot to the GPU box (it is git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
OUT = os.path.join(PKG, "libstampede_b200.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
EXTRA = os.environ.get("STP_NVCC_EXTRA", "").split()
FLAGS = EXTRA + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         f"-I{os.path.join(ROOT, 'include')}", f"-I{CSRC}"]
# fp32 step kernel: IEEE-approximate division / sqrt (<= 2 ulp, no slow-path
# branches) and flush-to-zero — its parity is a stated fp32 envelope against
# the reference, and the f64 instantiation (the exact parity instrument) is
# not affected by these single-precision flags
FP32_FLAGS = ["-ftz=true", "-prec-div=false", "-prec-sqrt=false"]
# sim_aux.cu holds the fp32 math self-test, compiled like the step kernel
PER_SOURCE = {"sim_step_f32.cu": FP32_FLAGS, "sim_aux.cu": FP32_FLAGS}
SOURCES = ["sim_step_f32.cu", "sim_step_f64.cu", "sim_host.cu", "sim_aux.cu", "sim_pairs.cu", "models.cpp", "policy_mlp.cu"]
DEPS = ["sim_device.cuh", "sim_kernels.cuh", "sim_step.cuh", "sim_launch.h", "stp_rng.h", "stp_error.h"]


def _mtime(p):
    return os.path.getmtime(p) if os.path.exists(p) else 0.0


def _compile(src: str) -> tuple[str, str]:
    path = os.path.join(CSRC, src)
    obj = os.path.join(BUILD, src + ".o")
    newest = max([_mtime(path), _mtime(os.path.join(ROOT, "include", "stampede_sim.h"))] +
                 [_mtime(os.path.join(CSRC, d)) for d in DEPS])
    if _mtime(obj) >= newest:
        return obj, ""
    cmd = [NVCC] + ARCH + FLAGS + PER_SOURCE.get(src, []) + ["-c", path, "-o", obj]
    if src.endswith(".cpp"):
        cmd = [NVCC] + ARCH + FLAGS + ["-x", "cu", "-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    stamp = os.path.join(BUILD, "flags.txt")  # objects built with other flags are stale
    flags = " ".join(ARCH + FLAGS) + repr(sorted(PER_SOURCE.items()))
    if not os.path.exists(stamp) or open(stamp).read() != flags:
        for f in os.listdir(BUILD):
            if f.endswith(".o"):
                os.remove(os.path.join(BUILD, f))
        with open(stamp, "w") as fh:
            fh.write(flags)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(_compile, SOURCES))
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            if log:
                print(log, file=sys.stderr)
    if not os.path.exists(OUT) or _mtime(OUT) < max(_mtime(o) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", OUT] + objs + ["-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
