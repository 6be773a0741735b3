"""Per-CTA phase timing of the unit kernels from a -DFDE_PROBES build
(paper_1912_13304_b200/libfde_probe.so): marker 0 = start, 1 = inputs loaded,
2 = forward FFT done, 3 = transform done, 4 = stores issued (%globaltimer, ns)."""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["FDE_LIB"] = os.path.join(ROOT, "paper_1912_13304_b200", "libfde_probe.so")
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1912_13304_b200 import fde  # noqa: E402

fde.lib.fde_debug_probes.argtypes = [ctypes.c_void_p, ctypes.c_int64]
p = W.config(int(sys.argv[1]) if len(sys.argv) > 1 else 5, n=int(sys.argv[2]) if len(sys.argv) > 2 else 1023)
h = fde.Fde.from_problem(p, stream=torch.cuda.current_stream().cuda_stream)
x = torch.from_numpy(p.rhs.copy()).cuda()
y, z = torch.empty_like(x), torch.empty_like(x)
buf = np.zeros((8, 2048, 8), dtype=np.uint64)
for _ in range(3):
    h.matvec(x, y)
    h.tau_apply(x, z)
    torch.cuda.synchronize()
    fde.lib.fde_debug_probes(buf.ctypes.data, buf.nbytes)
names = ["toeplitz_rows", "toeplitz_cols", "dst_rows", "tau_cols", "dst_rows(post)"]
for s in range(5):
    b = buf[s].astype(np.int64)
    used = b[:, 0] > 0
    b = b[used]
    t0 = b[:, 0].min()
    rel = (b - t0) / 1e3
    print("%-15s CTAs %4d  start spread %.2f us  end (max marker4) %.2f us" % (names[s], used.sum(), rel[:, 0].max(), rel[:, 4].max()))
    for i in range(4):
        d = rel[:, i + 1] - rel[:, i]
        print("   phase %d->%d  median %.2f  max %.2f us" % (i, i + 1, np.median(d), d.max()))
