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
    """oracle.cost.workload_gradient (parameter shift + quotient rule, reading 23) against a
    central difference of the oracle's C: a dropped term of the quotient rule, a wrong sign, a
    missing 1/2 of the shift rule or a permuted parameter index fails at 1e-8."""
    w = configs.cfg1()
    th = w.theta0()
    co = ocost.coeffs_of(w)
    C0, g = ocost.workload_gradient(w, th, _terms)
    assert abs(C0 - ocost.cost(_terms(w, th), co, w.n, w.L)[0]) == 0.0
    h = 1e-5
    for p in range(w.n_params):
        e = np.zeros(w.n_params)
        e[p] = 1.0
        Cp = ocost.cost(_terms(w, th + h * e), co, w.n, w.L)[0]
        Cm = ocost.cost(_terms(w, th - h * e), co, w.n, w.L)[0]
        assert abs(g[p] - (Cp - Cm) / (2 * h)) <= 1e-8, p


def test_gradient_vanishes_at_the_solution():
    """At a minimiser of C the gradient is zero: A = I, b = |0>, theta = 0 gives x = b and C = 0
    (a global minimum of C >= 0), so every dC/dtheta_p = 0 by the shift rule."""
    n = 2
    w = configs.Workload("identity_n2", n, 1, [(1.0 + 0j, "II")], configs.B_AMPLITUDES,
                         np.array([1, 0, 0, 0], complex), 0)
    C0, g = ocost.workload_gradient(w, np.zeros(w.n_params), _terms)
    assert abs(C0) < 1e-15 and np.max(np.abs(g)) < 1e-14
