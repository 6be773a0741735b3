"""Per-step timeline of one GMRES(30) cycle's DCGS2 orthogonalisation (trace
build -DFDE_SOP_TRACE=1 via FDE_LIB): for every Arnoldi step j of the FIRST
cycle of a cfg-4 solve, pass A's first block start, last element-loop end, the
finalising block's Givens step done, and pass B's last block end (µs)."""
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
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 4
p = W.config(cfg, n=n)
h = fde.Fde.from_problem(p)
b = torch.from_numpy(p.rhs.copy()).cuda()
x = torch.zeros_like(b)
h.gmres(b, x, p.rtol, p.restart, 30)   # warm-up
torch.cuda.synchronize()
assert fde.lib.fde_debug_xr_trace_reset() == 0
h.gmres(b, x, p.rtol, p.restart, 30)   # one cycle
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 4096)()
assert fde.lib.fde_debug_xr_trace(buf, 4096) == 0
a = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
t = a[3000:3000 + 4 * 31].reshape(31, 4)
t0 = t[0, 0]
rows = []
prev = None
for j in range(30):
    s0, le, sd, be = [(v - t0) / 1e3 for v in t[j]]
    rows.append({"j": j, "A_start": round(s0, 1), "A_loop": round(le - s0, 1), "A_tail": round(sd - le, 1),
                 "B": round(be - sd, 1), "op_gap": None if prev is None else round(s0 - prev, 1)})
    prev = be
for r in rows:
    print(json.dumps(r))
h.close()
