"""Build libfde.so in-tree with nvcc for sm_100a (the .so travels to the GPU
box with the repo snapshot). Each translation unit (csrc/*.cu) is compiled
to an object in parallel, then the objects are linked into one shared
library."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
UNITS = ["fde.cu", "sop.cu"]
OUT = os.path.join(HERE, "libfde.so")
DEPS = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
DEPS.append(os.path.join(os.path.dirname(HERE), "include", "fde.h"))

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                 "-diag-suppress", "128,177"]


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(d) <= t for d in DEPS)


def build(force: bool = False, log: str = None, out: str = None, extra=()) -> str:
    """Compile libfde.so (or `out` with extra nvcc flags, for A/B variants)."""
    if out is None and not force and up_to_date():
        return OUT
    out = out or OUT
    nvcc = os.environ.get("NVCC", "nvcc")
    objdir = os.path.join(HERE, "build_obj")
    os.makedirs(objdir, exist_ok=True)
    tag = os.path.splitext(os.path.basename(out))[0]

    def compile_unit(u):
        obj = os.path.join(objdir, "%s_%s.o" % (tag, os.path.splitext(u)[0]))
        cmd = [nvcc] + CFLAGS + list(extra) + ["-c", "-o", obj, os.path.join(CSRC, u)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        return u, obj, r

    with ThreadPoolExecutor(max_workers=len(UNITS)) as ex:
        results = list(ex.map(compile_unit, UNITS))
    text = "".join(r.stdout + r.stderr for _, _, r in results)
    failed = [u for u, _, r in results if r.returncode != 0]
    if not failed:
        cmd = [nvcc] + ARCH + ["-shared", "-o", out] + [o for _, o, _ in results]
        r = subprocess.run(cmd, capture_output=True, text=True)
        text += r.stdout + r.stderr
        if r.returncode != 0:
            failed.append("link")
    if log:
        with open(log, "w") as f:
            f.write(text)
    if failed:
        sys.stderr.write(text[-6000:])
        raise RuntimeError("nvcc failed building %s (%s)" % (out, ", ".join(failed)))
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, log=os.path.join(HERE, "..", "build_ptxas.log")))
