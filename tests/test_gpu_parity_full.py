"""Oracle parity of full solves at the sizes the bench measures (SURVEY
§8(a) a3/a4, BASELINE north_star tolerances: iterations within ±1 of the
oracle's, final solution within 1e-9 relative), plus the paper's own tables
reproduced with every solve on the GPU.

What these check is τ and S applied through eq:tau and eq:sine_transform
 inside the production launch configuration: cfg 5 at n = 1023 is
the bench workload (the r02 sine-domain body), n = 2047 the second
north_star size, cfg 4 at n = 1023 the GMRES(30) workload. The oracle's dense
products cost ~17 GFlop per iteration at n = 1023, so each oracle solve runs
once per module (cached) and is shared by the GPU variants.
"""
import numpy as np
import pytest

import oracle as O
import workloads as W
from conftest import load_golden
from test_gpu_ops import oracle_system, oracle_weights, relerr

pytestmark = pytest.mark.gpu

_ORACLE = {}


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def oracle_cached(cfg, n, batch, solver):
    key = (cfg, n, batch, solver)
    if key not in _ORACLE:
        p = W.config(cfg, n=n, batch=batch)
        s = oracle_system(p)
        cx, cy = oracle_weights(p, s)
        Pinv = lambda v: s.prec_solve(v, p.prec, cx, cy)
        res = []
        for b in range(batch):
            if solver == "pcg":
                res.append(O.pcg(s.matvec, Pinv, p.rhs[b], p.rtol, p.maxit))
            else:
                res.append(O.gmres(s.matvec, Pinv, p.rhs[b], p.rtol, p.restart, p.maxit))
        _ORACLE[key] = (p, s, res)
    return _ORACLE[key]


def gpu_solve_env(torch, monkeypatch, p, solver, env):
    from paper_1912_13304_b200 import fde
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    h = fde.Fde.from_problem(p)
    b = torch.from_numpy(p.rhs.copy()).cuda()
    x = torch.zeros_like(b)
    if solver == "pcg":
        st, stats = h.pcg(b, x, p.rtol, p.maxit)
    else:
        st, stats = h.gmres(b, x, p.rtol, p.restart, p.maxit)
    torch.cuda.synchronize()
    out = x.cpu().numpy()
    h.close()
    return stats, out


def check(stats, x, p, s, res):
    for b in range(p.batch):
        xo, it_o, conv_o, _ = res[b]
        assert conv_o and stats[b]["converged"]
        assert abs(stats[b]["iters"] - it_o) <= 1, (b, stats[b]["iters"], it_o)
        assert relerr(x[b], xo) <= 1e-9, (b, relerr(x[b], xo))
        r = p.rhs[b] - s.matvec(x[b])
        assert np.linalg.norm(r) / np.linalg.norm(p.rhs[b]) <= 2e-10


# the sine-domain PCG body variants the library can run at these sizes
PCG_BODIES = [{}, {"FDE_SOP": "0"}]   # the r02 body (default) and the r01 concurrent body


@pytest.mark.parametrize("env", PCG_BODIES, ids=lambda e: ",".join("%s=%s" % kv for kv in e.items()) or "default")
@pytest.mark.parametrize("batch", [1, 2])
def test_cfg5_n1023_pcg_matches_oracle(torch_cuda, monkeypatch, batch, env):
    """The bench workload (BASELINE cfg 5, n = 1023, batch 1) and batch 2,
    every sine-domain body, against the oracle's dense PCG."""
    p, s, res = oracle_cached(5, 1023, batch, "pcg")
    stats, x = gpu_solve_env(torch_cuda, monkeypatch, p, "pcg", env)
    check(stats, x, p, s, res)


def test_cfg5_n2047_pcg_matches_oracle(torch_cuda, monkeypatch):
    """The second north_star size (cfg 5, n = 2047)."""
    p, s, res = oracle_cached(5, 2047, 1, "pcg")
    stats, x = gpu_solve_env(torch_cuda, monkeypatch, p, "pcg", {})
    check(stats, x, p, s, res)


def test_cfg4_n1023_gmres_matches_oracle(torch_cuda, monkeypatch):
    """BASELINE cfg 4 at full size: GMRES(30) right-preconditioned by the
    mean-coefficient τ (R9, R12) against the oracle's CGS2 GMRES (SURVEY
    App. A forecast: 466 iterations)."""
    p, s, res = oracle_cached(4, 1023, 1, "gmres")
    stats, x = gpu_solve_env(torch_cuda, monkeypatch, p, "gmres", {})
    check(stats, x, p, s, res)
    assert abs(res[0][1] - 466) <= 2


# ------------------------------------------------------------ paper tables --

TABLE12 = load_golden("table1_table2.txt")
PTRI = load_golden("table2_ptri.txt")
TABLE34 = load_golden("table3_table4.txt")


def example1_gpu(alpha, n, prec):
    """Example 1 time loop (b = ν u^{(m-1)} + h^α f(t_m))
    with every GMRES solve on the GPU: left-preconditioned, unrestarted,
    tol 1e-7, x0 = 0 (R8). Returns the average iterations per step."""
    from paper_1912_13304_b200 import fde
    ex = W.example1(alpha, n)
    h = fde.Fde(n, 1, alpha, nu=ex["nu"], dp_field=ex["dp"], dm_field=ex["dm"], prec=prec)
    u = ex["u0"].copy()
    its = 0
    for m in range(1, ex["M"] + 1):
        b = (ex["nu"] * u + ex["h"] ** alpha * ex["f"](m * ex["ht"]))[None, :]
        x = np.zeros_like(b)
        st, stats = h.gmres(np.ascontiguousarray(b), x, 1e-7, 64, 64, left=True)
        assert stats[0]["converged"]
        its += stats[0]["iters"]
        u = x[0]
    h.close()
    return its / ex["M"]


@pytest.mark.parametrize("row", TABLE12, ids=lambda r: "a%.1f-n%d" % (r[0], r[1]))
def test_paper_table1_table2_all_sizes_on_gpu(torch_cuda, row):
    """Table 1's P_F column (P_F = τ·D, R6) and Table 2's P̃
    column (R7) at every printed size n1+1 = 64..512, within
    ±0.15 of the printed average iteration count."""
    alpha, n1 = row[0], int(row[1])
    itF = example1_gpu(alpha, n1 - 1, W.PREC_TAU_D)
    assert abs(itF - row[4]) <= 0.15, ("P_F", alpha, n1, itF, row[4])
    itT = example1_gpu(alpha, n1 - 1, W.PREC_TILDE)
    assert abs(itT - row[6]) <= 0.15, ("P~", alpha, n1, itT, row[6])


@pytest.mark.parametrize("row", PTRI, ids=lambda r: "a%.1f-n%d" % (r[0], r[1]))
def test_paper_table2_ptri_all_sizes_on_gpu(torch_cuda, row):
    """Table 2's P_tri column (R19) at every printed size."""
    alpha, n1, printed = row[0], int(row[1]), row[2]
    it = example1_gpu(alpha, n1 - 1, W.PREC_TRI)
    assert abs(it - printed) <= 0.15, (alpha, n1, it, printed)


def example2_gpu(alpha, beta, n):
    """Examples 2/3 Crank-Nicolson loop on the GPU
    direct path (n+1 is not a power of two): WSGD stencil, P = τ(q_α +
    (s/r)q_β)·D_N (R4-R6, R14, R15), left/unrestarted GMRES tol 1e-7."""
    from paper_1912_13304_b200 import fde
    ex = W.example2(alpha, beta, n)
    s, inv_r, s_over_r = O.example2_matrices(ex, alpha, beta, n)
    h = fde.Fde(n, 2, alpha, beta, nu=inv_r, dp_field=ex["dp"], dm_field=ex["dm"], ep_field=ex["ep"],
                em_field=ex["em"], prec=W.PREC_TAU_D, cx=1.0, cy=s_over_r, ywt=s_over_r, stencil=2)
    u = ex["u0"].copy()
    its = 0
    for m_ in range(1, ex["M"] + 1):
        mu = np.zeros((1, n * n))
        h.matvec(np.ascontiguousarray(u[None, :]), mu)
        b = (2.0 * inv_r * u - mu[0] + 2.0 * ex["h"] ** alpha * ex["f"]((m_ - 0.5) * ex["ht"]))[None, :]
        x = np.zeros_like(b)
        st, stats = h.gmres(np.ascontiguousarray(b), x, 1e-7, 64, 64, left=True)
        assert stats[0]["converged"]
        its += stats[0]["iters"]
        u = x[0]
    h.close()
    return its / ex["M"]


@pytest.mark.parametrize("row", [r for r in TABLE34 if r[2] <= 32], ids=lambda r: "b%.1f-n%d" % (r[1], r[2]))
def test_paper_table3_table4_on_gpu(torch_cuda, row):
    """Table 3 (Example 2, β = 1.6) and Table 4 (Example 3,
    β = 1.2) at n = 16 and 32: the GPU's average iterations per
    step within ±0.25 of the oracle's loop under the same readings, and within
    ±0.5 of the printed P_F count — except Table 3 at n = 32, where the
    readings themselves give 8.63 against the printed 8.0, so
    the printed-value bar there is ±0.75."""
    alpha, beta, n, printed = row[0], row[1], int(row[2]), row[5]
    avg = example2_gpu(alpha, beta, n)
    ref = O.example2_run(W.example2(alpha, beta, n), alpha, beta, n, O.PREC_TAU_D)
    assert abs(avg - ref) <= 0.25, (avg, ref)
    bar = 0.75 if (beta == 1.6 and n == 32) else 0.5
    assert abs(avg - printed) <= bar, (avg, printed)
