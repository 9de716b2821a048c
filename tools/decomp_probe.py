"""NEXT-4 probe: dvqls.decompose on the n = 12 (or argv[1]) tridiagonal matrix a few times, device ms.
Run under ncu --metrics gpu__time_duration.sum for the per-kernel breakdown."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from dvqls_inputs import problems  # noqa: E402
from paper_2604_14435_b200 import build, dvqls  # noqa: E402

build.build()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
A, _ = problems.tridiag_toeplitz(n, 2.0, -1.0, -1.0)
for _ in range(3):
    terms, nrm, ms = dvqls.decompose(A, 0.01, device=0, timing=True)
    print(n, len(terms), nrm, ms)
