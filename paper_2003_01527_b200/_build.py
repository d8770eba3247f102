"""Build libgsm.so in-tree with nvcc for sm_100a (the only target)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libgsm.so")
SO_CHECKED = os.path.join(HERE, "libgsm_checked.so")  # -DGSM_DEVICE_CHECKS (tests only)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    c = os.path.join(HERE, "csrc")
    return sorted(glob.glob(os.path.join(c, "*.cu")) + glob.glob(os.path.join(c, "*.cpp")))


def deps():
    c = os.path.join(HERE, "csrc")
    return sources() + glob.glob(os.path.join(c, "*.h")) + [os.path.join(ROOT, "include", "gsm.h")]


def up_to_date(so: str = SO) -> bool:
    if not os.path.exists(so):
        return False
    t = os.path.getmtime(so)
    return all(os.path.getmtime(p) <= t for p in deps())


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """libgsm.so; checked=True: libgsm_checked.so with the device index checks compiled in
    (GSM_DEVICE_CHECKS, gsm_common.h) — a test build, selected by GSM_LIB=checked."""
    so = SO_CHECKED if checked else SO
    if not force and up_to_date(so):
        return so
    objdir = os.path.join(HERE, "build_checked" if checked else "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    common = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
              "-I", os.path.join(ROOT, "include"), "-I", os.path.join(HERE, "csrc")]
    if checked:
        common.append("-DGSM_DEVICE_CHECKS")
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *ARCH, *common, "-Xptxas", "-v" if verbose else "-O3", "-c", src, "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    failed = False
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            failed = True
            sys.stderr.write(" ".join(cmd) + "\n" + out + "\n")
        elif verbose and out:
            sys.stderr.write(out)
    if failed:
        raise RuntimeError("libgsm build failed")
    tmp = so + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-Xcompiler", "-fPIC"])
    os.replace(tmp, so)
    return so


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(SO)
