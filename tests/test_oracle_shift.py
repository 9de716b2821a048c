"""Pin (cfg 5 row "Gradient"): every parameter of the ansatz enters through exactly
one e^{-i theta sigma/2} (reading 7), so each Hadamard-test value f(theta) = Re or Im of
<x(theta)|B|x(theta)> obeys the parameter-shift rule
    d f / d theta_p = [f(theta + pi/2 e_p) - f(theta - pi/2 e_p)] / 2          (exact)
and the cost's gradient follows from Re E, Re Psi by the quotient rule.  Checked against a central
finite difference of the oracle itself (O(h^2)): a wrong rotation angle convention (e^{-i theta
sigma}), a parameter index permutation that reuses a parameter, or a dropped gate breaks the exact
rule.  CPU only, small n."""

import numpy as np
import pytest

from dvqls_inputs import configs
from oracle import cost as ocost
from oracle import sim


def _terms(w, th):
    return sim.workload_terms(w, th)


@pytest.mark.parametrize("ent", [0, 1])
def test_parameter_shift_equals_central_difference(ent):
    w = configs.random_workload(3, 3, 2, seed=17, entangler=ent)
    th = w.theta0()
    h = 1e-4
    for p in range(w.n_params):
        e = np.zeros(w.n_params)
        e[p] = 1.0
        shift = (_terms(w, th + np.pi / 2 * e) - _terms(w, th - np.pi / 2 * e)) / 2
        fd = (_terms(w, th + h * e) - _terms(w, th - h * e)) / (2 * h)
        assert np.max(np.abs(shift - fd)) <= 5e-7, p


def test_cost_gradient_by_quotient_rule():
    """dC/dtheta_p from the shifted (E, Psi) pairs: C = 1/2 - Re E / (2 n Re Psi), so
    dC = -(dReE * RePsi - ReE * dRePsi) / (2 n RePsi^2), against a central difference of C."""
    w = configs.cfg1()
    th = w.theta0()
    co = ocost.coeffs_of(w)
    C0, E0, P0 = ocost.cost(_terms(w, th), co, w.n, w.L)
    h = 1e-5
    for p in (0, 7, 23, 47):
        e = np.zeros(w.n_params)
        e[p] = 1.0
        _, Ep, Pp = ocost.cost(_terms(w, th + np.pi / 2 * e), co, w.n, w.L)
        _, Em, Pm = ocost.cost(_terms(w, th - np.pi / 2 * e), co, w.n, w.L)
        dE, dP = (Ep.real - Em.real) / 2, (Pp.real - Pm.real) / 2
        g = -(dE * P0.real - E0.real * dP) / (2 * w.n * P0.real ** 2)
        Cp = ocost.cost(_terms(w, th + h * e), co, w.n, w.L)[0]
        Cm = ocost.cost(_terms(w, th - h * e), co, w.n, w.L)[0]
        assert abs(g - (Cp - Cm) / (2 * h)) <= 1e-8, p
