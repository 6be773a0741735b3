"""Per-CTA trace of the sop operator kernel (measurement build with
-DFDE_SOP_TRACE=1, loaded through FDE_LIB): which SM ran which unit, when,
and the clock cycles of its phases (load, T1+T2, T3+T4, store). Runs one
fde_pcg solve of BASELINE cfg 5 and reads the LAST k_sop launch's trace.
usage: FDE_LIB=.../libfde_trace.so python tools/sop_trace.py [n] [batch]"""
import collections
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
m = n + 1
units = m * batch
buf = (ctypes.c_ulonglong * (8192 * 8))()
rc = fde.lib.fde_debug_sop_trace(buf, 8192 * 8)
assert rc == 0, rc
a = np.frombuffer(buf, dtype=np.uint64).reshape(8192, 8)[:units].astype(np.int64)
g0, sm, c2, c3, c4, c5, c6, g7 = a.T
t0 = g0.min()
start, end = (g0 - t0) / 1e3, (g7 - t0) / 1e3   # µs
u = np.arange(units) % m
col = u < m // 2
out = {"n": n, "batch": batch, "units": units, "span_us": float(end.max()),
       "sms_used": int(len(set(sm.tolist())))}
for name, sel in (("col", col), ("row", ~col)):
    out[name] = {"dur_us_mean": float((end - start)[sel].mean()), "dur_us_max": float((end - start)[sel].max()),
                 "start_us_max": float(start[sel].max()),
                 "cyc_load": float((c3 - c2)[sel].mean()), "cyc_t12": float((c4 - c3)[sel].mean()),
                 "cyc_t34": float((c5 - c4)[sel].mean()), "cyc_store": float((c6 - c5)[sel].mean()),
                 "cyc_total": float((c6 - c2)[sel].mean())}
per_sm = collections.defaultdict(list)
for i in range(units):
    per_sm[int(sm[i])].append(i)
spans = {s: (max(end[v]) - min(start[v]), sum(col[v]), len(v)) for s, v in per_sm.items()}
sp = np.array([v[0] for v in spans.values()])
out["sm_span_us"] = {"min": float(sp.min()), "mean": float(sp.mean()), "max": float(sp.max())}
mix = collections.Counter((v[2], int(v[1])) for v in spans.values())
out["sm_mix(units,cols)"] = {"%d,%d" % k: c for k, c in sorted(mix.items())}
slow = sorted(spans.items(), key=lambda kv: -kv[1][0])[:5]
out["slowest_sms"] = [{"sm": s, "span": round(v[0], 2), "cols": int(v[1]), "units": v[2]} for s, v in slow]
out["first_blocks_sm"] = [int(s) for s in sm[:24]]
xb = (ctypes.c_ulonglong * 4096)()
if fde.lib.fde_debug_xr_trace(xb, 4096) == 0:
    xa = np.frombuffer(xb, dtype=np.uint64).astype(np.int64)
    xt = xa[:4092].reshape(1023, 4)
    xt = xt[xt[:, 0] > 0]
    rel = lambda v: [round(float((v.min() - t0) / 1e3), 2), round(float((v.mean() - t0) / 1e3), 2),
                     round(float((v.max() - t0) / 1e3), 2)]
    out["timeline_us"] = {"sop_last_end": float((g7.max() - t0) / 1e3), "xr_ctas": int(len(xt)),
                          "xr_start": rel(xt[:, 0]), "xr_alpha": rel(xt[:, 1]), "xr_loop_end": rel(xt[:, 2]),
                          "xr_end": rel(xt[:, 3]), "ctrl": float((xa[4095] - t0) / 1e3)}
print(json.dumps(out))
h.close()
