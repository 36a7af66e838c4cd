"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This module builds *problems* (a sparse matrix A in CSR and a block right-hand side B);
it contains none of the method's arithmetic (no inner products, no Arnoldi, no solves).
Both sides of every parity test consume exactly the arrays produced here.
"""
from .generators import (  # noqa: F401
    Problem,
    CONFIGS,
    TWINS,
    csr_sha256,
    make_config,
    make_twin,
    random_sparse,
    rhs,
    sample_rows,
    sketch_chunks,
    stencil,
    tridiag,
    tridiag_rhs,
    laplacian_1d,
    identity,
)
