"""B200-native hot path of D-VQLS (arXiv 2604.14435).

The product is ``libdvqls.so`` (C ABI in ``include/dvqls.h``, CUDA sources in
``csrc/``); ``dvqls`` is its thin ctypes binding.  Build with
``python -m paper_2604_14435_b200.build``.
"""

from .dvqls import (  # noqa: F401
    Context, DvqlsError, DegenerateError, dvqls_create, dvqls_terms, dvqls_cost, dvqls_cost_batch,
    dvqls_destroy, dvqls_nccl_unique_id, dvqls_build_info, from_workload, load,
)
