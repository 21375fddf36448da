"""Pick the slow step H for each workload from the chemistry's stiffness
(test/bench infrastructure; run once, results frozen in
paper_2211_03293_b200/configs.py and DESIGN.md).

lambda_max = max |eig(d f_fast / d y)| over a sample of cells of the workload's
own seeded initial condition (a one-plane slab through the hotspot centre of
the full grid, generated with the counter-based IC so it equals the full-grid
field), Jacobian by central differences.  H = m * theta / lambda_max with
h*lambda_max = theta = 1 for the inner RK4 (real-axis limit 2.785), rounded
down to 2 significant digits.
"""
import math
import sys

import numpy as np

import oracle as O


def lambda_max(S, R, mech_seed, ic_seed, n, rho, n_sample=48):
    mech = O.mechanism(mech_seed, S, R)
    i0 = n // 2
    sysm = O.System(1, n, n, S + 1, fast="chem", mech=mech, S=S, R=R, rho=rho,
                    n0_global=n, i0_global=i0)
    y0 = sysm.initial_condition(ic_seed)
    nc = n * n
    Y = y0.reshape(S + 1, nc)
    rng = np.random.RandomState(0)
    cells = [nc // 2 + n // 2, 0] + list(rng.randint(0, nc, n_sample))
    lam = 0.0
    for c in cells:
        one = O.System(1, 1, 1, S + 1, fast="chem", mech=mech, S=S, R=R, rho=rho)
        v0 = Y[:, c].copy()
        f0 = one.fast_rhs(v0)
        J = np.zeros((S, S))
        for k in range(S):
            e = 1e-7  # absolute: mass fractions are O(1e-3..1)
            vp = v0.copy(); vp[k] += e
            vm = v0.copy(); vm[k] -= e
            J[:, k] = (one.fast_rhs(vp)[:S] - one.fast_rhs(vm)[:S]) / (2 * e)
        lam = max(lam, float(np.abs(np.linalg.eigvals(J)).max()))
    return lam


def round_down(x, sig=2):
    e = math.floor(math.log10(x))
    return math.floor(x / 10 ** (e - sig + 1)) * 10 ** (e - sig + 1)


if __name__ == "__main__":
    sys.path.insert(0, ".")
    from paper_2211_03293_b200.configs import CONFIGS
    for name, cfg in CONFIGS.items():
        lam = lambda_max(cfg["S"], cfg["R"], cfg["mech_seed"], cfg["ic_seed"], cfg["n"], cfg["rho"])
        H = round_down(cfg["m"] * 1.0 / lam)
        print(f"{name}: lambda_max={lam:.4g}  H={H:.3g}")
