"""Seeded, synthetic input generators shared by the oracle (``oracle/``) and the
CUDA product path (``paper_2604_14435_b200``).

This package holds NO arithmetic of the hot path (Alg. 1 Step 4,
P:450-465).  It only manufactures the inputs the
hot path consumes:

* ``problems``  - the paper's linear systems A x = b (tridiagonal Toeplitz,
  P:476-490; 4x4 Hele-Shaw) as dense numpy matrices + rhs;
* ``lcu``       - the LCU input A = sum_l c_l A_l produced by the
  FWHT Pauli decomposition + 1 % l2 pruning of Alg. 1 Steps 1-2,
  which is pre-processing that happens once, before the optimiser loop;
* ``seeds``     - theta_0 draws and random robustness LCUs / b vectors;
* ``configs``   - the BASELINE.json configurations as concrete inputs.

Neither side imports the other; both import this.
"""

from . import problems, lcu, seeds, configs  # noqa: F401
