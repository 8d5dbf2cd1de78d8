"""Build libpentarag.so (the C-ABI + sm_100a kernels) in-tree with nvcc.

    python -m paper_2506_21593_b200.build [--force]

The shared object lands next to this file so it travels to the GPU box with
the repo snapshot; nothing is installed into site-packages.
"""
from __future__ import annotations

import argparse
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libpentarag.so")
STAMP = os.path.join(HERE, ".libpentarag.stamp")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
    *([f"-DPR_MBAR_SUSPEND_NS={os.environ['PR_MBAR_SUSPEND_NS']}u"] if os.environ.get("PR_MBAR_SUSPEND_NS") else []),
]


def sources() -> list[str]:
    return sorted(
        os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh", ".h"))
    ) + [os.path.join(INCLUDE, "pentarag.h")]


def _digest() -> str:
    h = hashlib.sha256()
    for p in sources():
        with open(p, "rb") as fh:
            h.update(p.encode())
            h.update(fh.read())
    h.update(" ".join(NVCC_FLAGS).encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False) -> str:
    digest = _digest()
    if not force and os.path.exists(OUT) and os.path.exists(STAMP):
        with open(STAMP) as fh:
            if fh.read().strip() == digest:
                return OUT
    cus = [p for p in sources() if p.endswith(".cu")]
    objs = []
    build_dir = os.path.join(HERE, "_build")
    os.makedirs(build_dir, exist_ok=True)
    procs = []
    for cu in cus:
        obj = os.path.join(build_dir, os.path.basename(cu) + ".o")
        objs.append(obj)
        cmd = ["nvcc", *NVCC_FLAGS, "-I", INCLUDE, "-c", cu, "-o", obj]
        procs.append((cu, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    failed = False
    logs = []
    for cu, p in procs:
        out, _ = p.communicate()
        logs.append(f"== {os.path.basename(cu)}\n{out}")
        if p.returncode != 0:
            failed = True
    log_text = "\n".join(logs)
    with open(os.path.join(build_dir, "ptxas.log"), "w") as fh:
        fh.write(log_text)
    if failed or verbose:
        sys.stderr.write(log_text)
    if failed:
        raise RuntimeError("nvcc failed building libpentarag (see paper_2506_21593_b200/_build/ptxas.log)")
    # the driver API (cuTensorMapEncodeTiled) is reached through
    # cudaGetDriverEntryPoint, so there is no link-time dependency on libcuda
    link = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", OUT, *objs]
    r = subprocess.run(link, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout)
        raise RuntimeError("nvcc link failed")
    with open(STAMP, "w") as fh:
        fh.write(digest)
    return OUT


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose))
