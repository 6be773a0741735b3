"""Build libfde.so in-tree with nvcc for sm_100a (the .so travels to the GPU
box with the repo snapshot)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc", "fde.cu")
OUT = os.path.join(HERE, "libfde.so")
DEPS = [os.path.join(HERE, "csrc", f) for f in os.listdir(os.path.join(HERE, "csrc"))]
DEPS.append(os.path.join(os.path.dirname(HERE), "include", "fde.h"))

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v", "-diag-suppress", "128,177"]


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
    cmd = [nvcc] + NVCC_FLAGS + list(extra) + ["-o", out, SRC]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if log:
        with open(log, "w") as f:
            f.write(r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stderr[-4000:])
        raise RuntimeError("nvcc failed building %s" % out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, log=os.path.join(HERE, "..", "build_ptxas.log")))
