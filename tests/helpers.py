"""Shared test helpers (reference idioms)."""
import numpy as np


def per_species_rel_err(y, ref, ncomp):
    """max over species of max|y - ref| / max|ref| -- the idiom of
    proj/tests/test_mri.cpp:255 with max_norm_component per species."""
    y = np.asarray(y).reshape(ncomp, -1)
    ref = np.asarray(ref).reshape(ncomp, -1)
    worst = 0.0
    for k in range(ncomp):
        scale = np.abs(ref[k]).max()
        d = np.abs(y[k] - ref[k]).max()
        worst = max(worst, d / scale if scale > 0 else d)
    return worst


# LinearTwoRateOde::default_problem (proj/src/models.cpp:65-73)
A_FAST = np.array([[0.0, 4.0], [-4.0, 0.0]])
A_SI = np.array([[-1.0, 0.2], [0.3, -0.7]])
A_SE = np.array([[0.1, 0.4], [-0.3, -0.1]])
Y0_LIN = np.array([1.0, 0.6])


def expm_taylor(A, t):
    """analytic_solution (proj/src/models.cpp:75-100) in numpy."""
    a = np.array(A, dtype=float) * t
    sq = 0
    while np.abs(a).sum(axis=1).max() > 0.25:
        a *= 0.5
        sq += 1
    res = np.eye(len(a))
    term = np.eye(len(a))
    for k in range(1, 25):
        term = term @ a / k
        res = res + term
        if np.abs(term).sum(axis=1).max() < 1e-20:
            break
    for _ in range(sq):
        res = res @ res
    return res
