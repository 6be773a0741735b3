"""Per-CTA phase timing of the sine-domain PCG line kernels (-DFDE_PROBES
build, FDE_GRAPH=0): markers 0 start, 1 staged, 2 DST#1, 3 Toeplitz,
4 DST#2, 5 end (%globaltimer)."""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["FDE_LIB"] = os.path.join(ROOT, "paper_1912_13304_b200", "libfde_probe.so")
os.environ["FDE_GRAPH"] = "0"
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1912_13304_b200 import fde  # noqa: E402

fde.lib.fde_debug_probes.argtypes = [ctypes.c_void_p, ctypes.c_int64]
CFG = int(os.environ.get("PROBE_CFG", "5"))
NN = int(os.environ.get("PROBE_N", "1023"))
p = W.config(CFG, n=NN)
h = fde.Fde.from_problem(p, stream=torch.cuda.current_stream().cuda_stream)
b = torch.from_numpy(p.rhs.copy()).cuda()
x = torch.zeros_like(b)
buf = np.zeros((8, 2048, 8), dtype=np.uint64)
for _ in range(2):
    fde.lib.fde_debug_probes(buf.ctypes.data, buf.nbytes)
    h.pcg(b, x, 1e-10, 2)
    torch.cuda.synchronize()
    fde.lib.fde_debug_probes(buf.ctypes.data, buf.nbytes)
# every probed launch slot of the last iteration; a concurrent-body launch
# (sine_op_rc) is split into its column CTAs [0, gc) and row CTAs [gc, ...)
gc = (p.n + 1) // 2
for s in range(8):
    bb_all = buf[s].astype(np.int64)
    used_all = bb_all[:, 0] > 0
    if used_all.sum() == 0:
        continue
    t0 = bb_all[used_all, 0].min()
    ranges = [("all", np.arange(2048))]
    if used_all.sum() > gc:
        ranges = [("cols", np.arange(gc)), ("rows", np.arange(gc, 2048))]
    for nm, idx in ranges:
        bb = bb_all[idx]
        used = bb[:, 0] > 0
        bb = bb[used]
        rel = (bb - t0) / 1e3
        print("slot %d %-5s CTAs %4d start spread %.2f us end %.2f us" % (s, nm, used.sum(), rel[:, 0].max(), rel[:, 5].max()))
        for i in range(5):
            d = rel[:, i + 1] - rel[:, i]
            print("   phase %d->%d  median %.2f  max %.2f us" % (i, i + 1, np.median(d), d.max()))
