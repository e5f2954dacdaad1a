"""Build libdynscreen.so in-tree with nvcc for sm_100a.

    python -m paper_1412_4080_b200.build

The shared library lands in ``paper_1412_4080_b200/_lib/`` (git-ignored, but
it travels to GPU boxes with the repo snapshot).
"""

from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB_DIR = os.path.join(HERE, "_lib")
LIB_PATH = os.path.join(LIB_DIR, "libdynscreen.so")
# bounds-checked variant (device asserts on list / slot / support indices, -DDSCR_CHECKS); loaded
# instead of the default library when DSCR_LIB=checked -- the substitute for compute-sanitizer,
# which this GPU pool does not allow
CHECKED_PATH = os.path.join(LIB_DIR, "libdynscreen_checked.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_path():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def needs_build(path=LIB_PATH):
    if not os.path.exists(path):
        return True
    t = os.path.getmtime(path)
    deps = sources() + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + [os.path.join(ROOT, "include", "dynscreen.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force=False, verbose=False, checked=False):
    out_path = CHECKED_PATH if checked else LIB_PATH
    if not force and not needs_build(out_path):
        return out_path
    os.makedirs(LIB_DIR, exist_ok=True)
    objs = []
    cmd_base = [nvcc_path(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
                "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"),
                "-I", os.path.join(HERE, "csrc")]
    if verbose:
        cmd_base += ["-Xptxas", "-v"]
    cmd_base += os.environ.get("DSCR_NVCC_EXTRA", "").split()   # experiment knobs (-D...), empty by default
    if checked:
        cmd_base += ["-DDSCR_CHECKS"]
    build_dir = os.path.join(LIB_DIR, "obj_checked" if checked else "obj")
    os.makedirs(build_dir, exist_ok=True)
    procs = []
    for src in sources():
        obj = os.path.join(build_dir, os.path.basename(src) + ".o")
        objs.append(obj)
        procs.append((src, subprocess.Popen(cmd_base + ["-c", src, "-o", obj],
                                            stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out.decode())
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose and out:
            sys.stderr.write(out.decode())
    tmp = out_path + ".tmp"
    link = [nvcc_path(), *ARCH, "-shared", "-o", tmp, *objs, "-ldl"]
    p = subprocess.run(link, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    if p.returncode != 0:
        sys.stderr.write(p.stdout.decode())
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, out_path)
    return out_path


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, checked="--checked" in sys.argv))
