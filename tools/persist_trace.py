"""Phase timeline of the persistent 2D sine PCG kernel (trace build,
-DFDE_SOP_TRACE=1, via FDE_LIB): per CTA of the LAST iteration, globaltimer at
iteration start, end of phase A (units), after barrier 1, after the α sums,
end of phase B, after barrier 2, iteration end. Prints min/mean/max over CTAs
relative to the earliest iteration start (µs)."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1912_13304_b200 import fde  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1023
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 1
p = W.config(5, n=n, batch=batch)
h = fde.Fde.from_problem(p)
b = torch.from_numpy(p.rhs.copy()).cuda()
x = torch.zeros_like(b)
for _ in range(3):
    h.pcg(b, x, p.rtol, p.maxit)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (8192 * 8))()
assert fde.lib.fde_debug_sop_trace(buf, 8192 * 8) == 0
a = np.frombuffer(buf, dtype=np.uint64).reshape(8192, 8).astype(np.int64)
a = a[a[:, 0] > 0]
t0 = a[:, 0].min()
names = ["start", "A_end", "bar1", "alpha", "B_end", "bar2", "end"]
out = {"n": n, "batch": batch, "ctas": int(len(a))}
for i, nm in enumerate(names):
    v = (a[:, i] - t0) / 1e3
    out[nm] = [round(float(v.min()), 2), round(float(v.mean()), 2), round(float(v.max()), 2)]
print(json.dumps(out))
h.close()
