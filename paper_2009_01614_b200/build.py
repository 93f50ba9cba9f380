"""Build the in-tree shared libraries for sm_100a (no torch extension machinery, plain nvcc).

  paper_2009_01614_b200/libisax.so   the product: csrc/*.cu behind include/isax.h
  paper_2009_01614_b200/libisax_bounds.so   the same with device-side bounds checks (-DISAX_BOUNDS; tests only)
  datagen/libisaxgen.so              the seeded input generator (harness; no method arithmetic)

python -m paper_2009_01614_b200.build [--force]
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v,-warn-spills"]

TARGETS = {
    "isax": (os.path.join(PKG, "csrc"), os.path.join(PKG, "libisax.so")),
    # the same sources with the device-side bounds checks compiled in (ISAX_BOUND, isax_internal.cuh);
    # tests/test_bounds.py runs the GPU parity suite against it
    "isax_bounds": (os.path.join(PKG, "csrc"), os.path.join(PKG, "libisax_bounds.so")),
    "isaxgen": (os.path.join(ROOT, "datagen"), os.path.join(ROOT, "datagen", "libisaxgen.so")),
}


def _stale(out: str, srcs: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs)


def build_one(name: str, force: bool = False, verbose: bool = False) -> str:
    src_dir, out = TARGETS[name]
    srcs = sorted(glob.glob(os.path.join(src_dir, "*.cu")))
    deps = srcs + glob.glob(os.path.join(src_dir, "*.cuh")) + glob.glob(os.path.join(src_dir, "*.inc"))
    deps += glob.glob(os.path.join(src_dir, "*.h"))
    deps += glob.glob(os.path.join(ROOT, "include", "*.h"))
    if not force and not _stale(out, deps):
        return out
    tmp = out + f".tmp{os.getpid()}"
    objdir = os.path.join(ROOT, "build", name)
    os.makedirs(objdir, exist_ok=True)
    inc = ["-I", os.path.join(ROOT, "include")] + (["-DISAX_BOUNDS"] if name == "isax_bounds" else [])
    objs = [os.path.join(objdir, os.path.basename(s)[:-3] + ".o") for s in srcs]
    cmds = [[NVCC, *ARCH, *FLAGS, *inc, "-c", s, "-o", o] for s, o in zip(srcs, objs)]
    with ThreadPoolExecutor(max_workers=min(8, len(cmds))) as ex:
        results = list(ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), cmds))
    link = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", *objs, "-ldl", "-o", tmp]
    results.append(subprocess.run(link, capture_output=True, text=True) if all(r.returncode == 0 for r in results) else None)
    log = os.path.join(os.path.dirname(out), f"build_{name}.log")
    text = ""
    for c, r in zip(cmds + [link], results):
        if r is not None:
            text += " ".join(c) + "\n" + r.stdout + r.stderr
    with open(log, "w") as f:
        f.write(text)
    if any(r is None or r.returncode != 0 for r in results):
        sys.stderr.write(text[-6000:])
        raise RuntimeError(f"nvcc failed for {name}; see {log}")
    if verbose:
        sys.stdout.write(text)
    os.replace(tmp, out)
    return out


def build_all(force: bool = False, verbose: bool = False) -> list[str]:
    return [build_one(n, force, verbose) for n in TARGETS]


if __name__ == "__main__":
    for p in build_all(force="--force" in sys.argv, verbose="-v" in sys.argv):
        print(p)
