"""Design the composite odd minimax sign approximation S = p_r o ... o p_1 (Eq. 3-4).

The paper's own f, g (degree 9, alpha = 12, d_f = d_g = 2, "max error < 1e-4") are not given
and that claim is infeasible (reading R3).  We follow BASELINE.json configs[4]:
degrees (7, 15, 15), margin eps = 2^-7.  Each stage is an LP minimax fit (Chebyshev basis,
odd) of sign on [a, 1] with |p| <= 1 + delta on [0, a]; stages 1..r-1 are divided by
(1 + delta) so the next stage's domain is [(1 - delta)/(1 + delta), 1].

This is a parameter-design script: it writes coefficients (data) consumed by both the
oracle tests and the CUDA library through the secpe_sign_cfg argument.  It is neither
oracle nor product arithmetic.  Usage: python tools/design_sign.py
"""
import json
import os
import sys

import numpy as np
from numpy.polynomial import chebyshev as C
from scipy.optimize import linprog


def fit_stage(deg, a, final, n_pass=6000, n_trans=1500):
    ks = np.arange(1, deg + 1, 2)
    xp = 0.5 * (1 + a) + 0.5 * (1 - a) * np.cos(np.linspace(0, np.pi, n_pass))
    xt = np.linspace(0, a, n_trans)
    Tp = np.stack([C.chebval(xp, np.eye(deg + 1)[k]) for k in ks], axis=1)
    Tt = np.stack([C.chebval(xt, np.eye(deg + 1)[k]) for k in ks], axis=1)
    nv = len(ks) + 1  # coefficients + delta
    A, b = [], []
    # |p(x) - 1| <= delta on the pass band
    A.append(np.hstack([Tp, -np.ones((n_pass, 1))])); b.append(np.ones(n_pass))
    A.append(np.hstack([-Tp, -np.ones((n_pass, 1))])); b.append(-np.ones(n_pass))
    # 0 <= p(x) <= 1 + delta on the transition band
    A.append(np.hstack([Tt, -np.ones((n_trans, 1))])); b.append(np.ones(n_trans))
    A.append(np.hstack([-Tt, np.zeros((n_trans, 1))])); b.append(np.zeros(n_trans))
    cost = np.zeros(nv); cost[-1] = 1.0
    res = linprog(cost, A_ub=np.vstack(A), b_ub=np.concatenate(b),
                  bounds=[(None, None)] * (nv - 1) + [(0, None)], method="highs")
    assert res.success, res.message
    cheb = np.zeros(deg + 1); cheb[ks] = res.x[:-1]
    delta = res.x[-1]
    power = C.cheb2poly(cheb)
    if not final:
        power = power / (1.0 + delta)
    power[0::2] = 0.0
    return power, delta


def design(degrees, eps):
    a, stages = eps, []
    for i, d in enumerate(degrees):
        final = i == len(degrees) - 1
        p, delta = fit_stage(d, a, final)
        stages.append(p)
        if not final:
            x = np.linspace(a, 1, 200001)
            a = float(np.polynomial.polynomial.polyval(x, p).min())
        print("stage %d deg %d: delta %.3e next a %.6f" % (i, d, delta, a), file=sys.stderr)
    return stages


def composite(stages, x):
    for p in stages:
        x = np.polynomial.polynomial.polyval(x, p)
    return x


if __name__ == "__main__":
    eps_log2 = 7
    stages = design([7, 15, 15], 2.0 ** -eps_log2)
    x = np.linspace(2.0 ** -eps_log2, 1, 1000001)
    err = np.abs(composite(stages, x) - 1).max()
    print("max |1-S| on [2^-%d, 1]: %.3e" % (eps_log2, err), file=sys.stderr)
    out = {"name": "minimax_7_15_15", "eps_log2": eps_log2, "max_err_design": err,
           "degrees": [7, 15, 15], "coeffs": [[float(c) for c in p] for p in stages],
           "source": "tools/design_sign.py (LP minimax, BASELINE.json configs[4])"}
    here = os.path.dirname(os.path.abspath(__file__))
    with open(os.path.join(here, "..", "data", "sign_7_15_15.json"), "w") as f:
        json.dump(out, f, indent=1)
    toy = {"name": "f1_f1", "eps_log2": None, "degrees": [3, 3],
           "coeffs": [[0.0, 1.5, 0.0, -0.5], [0.0, 1.5, 0.0, -0.5]],
           "source": "BASELINE.json configs[0]: 2 iterations of f(x) = (3x - x^3)/2"}
    with open(os.path.join(here, "..", "data", "sign_f1_f1.json"), "w") as f:
        json.dump(toy, f, indent=1)
