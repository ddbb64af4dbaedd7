"""CP-ALS on the exact-rank device epilogue (R = 16 / 32) against the
unmodified reference (proj/src/cpals.cpp:66-111, dense_kernels.cpp:68-92).

The golden runs (tests/golden/cpals_exact_rank.npz, made by
tests/golden/gen_cpals_golden.py from oracle/_ref/libblco_ref.so) cover the
path BASELINE configs[3] runs: a Delicious-shaped 4-mode power-law tensor
(78-bit layout, 14 stripped bits, thousands of keyed blocks) at R = 16, and a
3-mode tensor at R = 32.  Tolerances: fit within 1e-10 per
iteration, factors within 1e-9 relative Frobenius after 10 iterations,
lambda within 1e-9.
"""
import ctypes as C
import json
from pathlib import Path

import numpy as np
import pytest

from conftest import rel_frobenius

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden" / "cpals_exact_rank.npz"


@pytest.fixture(scope="module")
def cgold():
    z = np.load(GOLDEN)
    return z, json.loads(bytes(z["meta"]).decode())


@pytest.mark.parametrize("name", ["n32", "d16"])
def test_cp_als_exact_rank_matches_reference(gpu, cgold, name):
    z, meta = cgold
    c = meta[name]
    dims = c["dims"]
    dt = gpu.DeviceTensor.synthetic_draws(dims, c["nnz"], c["seed"], c["skew"], 64, 1 << 27, 0)
    assert dt.nnz == c["nnz"]
    if name == "d16":
        assert dt.nblocks > 1000  # 14 stripped bits: the multi-key path
    opts = gpu.CpAlsOptions(rank=c["rank"], max_iters=c["iters"], tol=c["tol"], seed=c["fseed"])
    model = gpu.cp_als(dt, opts)
    want_fit = z[f"{name}_fit"]
    assert len(model.fit_history) == want_fit.size == c["iters"]
    assert np.max(np.abs(np.array(model.fit_history) - want_fit)) <= 1e-10
    assert rel_frobenius(model.lambda_, z[f"{name}_lambda"]) <= 1e-9
    for m in range(len(dims)):
        a = model.factors.factors[m]
        got = a if c["full"] else a[z[f"{name}_rows{m}"]]
        assert rel_frobenius(got, z[f"{name}_f{m}"]) <= 1e-9, (name, m)
        # whole-factor checks for the sampled case: column sums and norms
        assert rel_frobenius(a.sum(axis=0), z[f"{name}_colsum{m}"]) <= 1e-9, (name, m)
        assert rel_frobenius((a * a).sum(axis=0), z[f"{name}_colsq{m}"]) <= 1e-9, (name, m)


def _solve_device(gpu, grams, order, mode, m):
    """blco_als_solve on device copies of grams (order x R x R) and M."""
    import torch
    R = m.shape[1]
    dg = torch.from_numpy(np.ascontiguousarray(grams)).cuda()
    dm = torch.from_numpy(np.ascontiguousarray(m)).cuda()
    da = torch.empty_like(dm)
    dgram = torch.empty((R, R), dtype=torch.float64, device="cuda")
    dstat = torch.zeros(1, dtype=torch.int32, device="cuda")
    st = gpu._lib.lib.blco_als_solve(C.c_void_p(dg.data_ptr()), order, mode, R, C.c_void_p(dm.data_ptr()),
                                     m.shape[0], C.c_void_p(da.data_ptr()), C.c_void_p(dgram.data_ptr()),
                                     C.c_void_p(dstat.data_ptr()), C.c_void_p(0))
    assert st == 0
    torch.cuda.synchronize()
    return da.cpu().numpy(), int(dstat.item())


@pytest.mark.parametrize("R", [8, 16, 32])
def test_solve_escalation_with_large_trace(gpu, oracle, R):
    """solve_normal's Tikhonov escalation (dense_kernels.cpp:72-80) on a
    singular V whose trace/R is far above 1, so the first shift 1e-12 * unit
    is itself above 1e-3: every thread of k_small_prep must apply the same
    stop test (a per-thread `unit` once made the other threads quit early and
    left L half-written).  V = 1e12 * blockdiag(SPD, 0); order 2, mode 0, so
    V = grams[1]."""
    rng = np.random.default_rng(R)
    B = rng.uniform(-1, 1, size=(R - 1, R - 1))
    spd = B @ B.T / R + np.eye(R - 1)
    V = np.zeros((R, R))
    V[: R - 1, : R - 1] = spd
    V *= 1e12
    grams = np.stack([np.eye(R), V])
    M = rng.uniform(-1, 1, size=(1000, R))
    want = oracle.solve_normal(M, V)
    got, status = _solve_device(gpu, grams, 2, 0, M)
    assert status == 0
    assert rel_frobenius(got, want) <= 1e-12
    assert np.isfinite(got).all() and np.abs(got[:, R - 1]).max() > 0
