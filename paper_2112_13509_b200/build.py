"""Build libautobyte.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo)."""
from __future__ import annotations

import concurrent.futures
import glob
import os
import shutil
import subprocess
import sys
import tempfile

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libautobyte.so")
STATS_LIB = os.path.join(PKG, "libautobyte_stats.so")   # -DAB_STATS cycle-accounting variant (tools only)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def nccl_dirs():
    import nvidia.nccl  # the NCCL that ships with torch (2.28.x)
    base = list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))) + \
        sorted(glob.glob(os.path.join(ROOT, "include", "*.h")))


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in deps())


def build(force: bool = False, verbose: bool = False, stats: bool = False, exp: int = 0,
          defines: tuple = (), name: str = "") -> str:
    """exp > 0 builds libautobyte_exp<exp>.so with -DAB_EXP=<exp>: timing experiments of K2 that
    deliberately skip work (wrong results; tools only, never loaded by the package).
    defines / name build a tuning variant libautobyte_<name>.so (e.g. AB_NS_MAX=4) for tools."""
    lib_path = STATS_LIB if stats else LIB
    if exp:
        lib_path = os.path.join(PKG, f"libautobyte_exp{exp}.so")
    if name:
        lib_path = os.path.join(PKG, f"libautobyte_{name}.so")
    if not force and not stats and not exp and not name and up_to_date():
        return LIB
    inc, lib = nccl_dirs()
    flags = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
             "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
             "-I", os.path.join(ROOT, "include"), "-I", inc,
             *(["-DAB_STATS"] if stats else []), *([f"-DAB_EXP={exp}"] if exp else []),
             *[f"-D{d}" for d in defines]]
    if verbose:
        flags.insert(1, "-Xptxas=-v")
    # one object per translation unit, compiled in parallel, then one shared-library link
    objdir = tempfile.mkdtemp(prefix="ab_build_")
    objs = [os.path.join(objdir, os.path.basename(src) + ".o") for src in sources()]
    cmds = [[*flags, "-c", src, "-o", obj] for src, obj in zip(sources(), objs)]
    if verbose:
        for c in cmds:
            print(" ".join(c), file=sys.stderr)
    with concurrent.futures.ThreadPoolExecutor(max_workers=len(cmds)) as ex:
        for r in ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), cmds):
            if verbose or r.returncode:
                sys.stderr.write(r.stdout + r.stderr)
            if r.returncode:
                raise subprocess.CalledProcessError(r.returncode, r.args)
    subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *objs, "-o", lib_path + ".tmp",
                    "-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={lib}"], check=True)
    shutil.rmtree(objdir, ignore_errors=True)
    os.replace(lib_path + ".tmp", lib_path)
    return lib_path


if __name__ == "__main__":
    exp = int(sys.argv[sys.argv.index("--exp") + 1]) if "--exp" in sys.argv else 0
    defs = tuple(a.split("=", 1)[1] for a in sys.argv if a.startswith("-D="))
    name = sys.argv[sys.argv.index("--name") + 1] if "--name" in sys.argv else ""
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, stats="--stats" in sys.argv, exp=exp,
                defines=defs, name=name))
