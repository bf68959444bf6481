"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic (no Schur split, no secular
equation, no Cauchy matrix): it only draws seeded random numbers and builds the
initial factors A = U diag(sigma) V^T that the rank-1 update starts from.
Both sides (oracle/ and the CUDA path) receive the same bytes from here.

Recipes follow BASELINE.json `configs` and SURVEY.md §8(d) "Synthetic inputs":
seeds 170708369 + k for config Ck; haar(n) = Q of QR(N(0,1)) with columns
scaled by sign(diag R).  The paper itself uses random matrices with entries in
[1,9] (§7) and [0,1] (§7.1) for its experiments;
`paper_uniform` reproduces that recipe for the Table-2 analogue.
"""
from .gen import (SEED_BASE, haar, config_inputs, update_vectors, gaussian_factors,
                  graded_factors, paper_uniform, random_secular, interlaced_cauchy,
                  CONFIGS)
from .edge import EDGE_CASES, EDGE_RES_TOL, edge_case

__all__ = ["SEED_BASE", "haar", "config_inputs", "update_vectors", "gaussian_factors",
           "graded_factors", "paper_uniform", "random_secular", "interlaced_cauchy",
           "CONFIGS", "EDGE_CASES", "EDGE_RES_TOL", "edge_case"]
