"""ORACLE - TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct CPU reference for the D-VQLS hot path
(arXiv 2604.14435).  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with the CUDA product path
(``paper_2604_14435_b200``); both consume inputs from ``dvqls_inputs``.

Modules
* ``sim``   - ctypes front-end of ``sim.cpp``: the gate-by-gate Hadamard-test
              state-vector simulator (SURVEY.md §8(c) "Plain definition").
* ``cost``  - Alg. 1 Steps 4b-4c: coefficient-weighted aggregation
              of the term expectations into (E, Psi) and C = 1/2 - Re E/(2 n Re Psi).
* ``dense`` - dense-matrix references used to PIN the simulator: Pauli matrices
              and products, brute-force trace decomposition, dense ansatz,
              dense local / global costs (Eq. 1, Eq. 2), closed-form Pauli
              expectations.

Parity status: every function is pinned by tests under ``tests/test_oracle_*.py``
(see DESIGN.md "Oracle pins").  Raw term values at random theta have no paper
value to compare against ("parity unpinned vs the paper");
they are pinned by closed forms, dense quadratic forms and invariants.
"""

from . import sim, cost, dense  # noqa: F401
