"""CPU oracle for the rank-1 SVD update of Gandhi & Rajgor (arXiv 1707.08369).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg may import this package.  The product path
(paper_1707_08369_b200/) never imports, links or executes anything here, and
this package shares no code with it (no kernels, helpers, constants or
pre/post-processing).  See DESIGN.md §3 for the readings of the paper it takes
and the pins that check it against something other than itself.
"""
from .svd1_oracle import (  # noqa: F401
    EPS, schur_sym_2x2, schur_update_2x2, prepare_update, deflate, secular_w,
    secular_roots_bisect, loewner_zhat, cauchy_X, cauchy_apply_explicit,
    rank_one_update, svd_update, paper_error, orth_defect, column_residual,
    sym_rank_one_eig, DeflationResult, balance_factor,
)
