"""Host-side FMM plan logic (no GPU): the tree and interaction lists the apply builds
 stay O(n) in flops for the spectra of the BASELINE configs,
including isolated outlier eigenvalues and graded spectra."""
import numpy as np
import pytest

import oracle as O
from synth import interlaced_cauchy, random_secular
from paper_1707_08369_b200._lib import fmm_tree_stats


def _roots(d, z, rho):
    return O.secular_roots_bisect(d, z, rho)


@pytest.mark.parametrize("kind,rho", [("gaussian", 3.0), ("graded", 4096.0), ("uniform", -2.0),
                                      ("graded", -0.5)])
def test_flops_per_point_bounded(kind, rho):
    rng = np.random.default_rng(5)
    n = 2048
    d, z, _ = random_secular(n, rng, kind=kind)
    k, tau = _roots(d, z, rho)
    st = fmm_tree_stats(d, k, tau, 1e-10)
    assert st["max_leaf"] <= 33
    # the planner picks the depth by estimated cost (flops + launches), so one leaf
    # next to an isolated outlier root may keep a long near list
    assert st["max_near"] <= 40
    assert st["flops_per_row"] / n <= 700, st      # direct product: 2n = 4096 per point


def test_outliers_do_not_widen_leaves():
    """A handful of eigenvalues 1e7 x above a graded bulk (what rank-1 updates of C3
    create) must not make any leaf near-field to the whole spectrum."""
    rng = np.random.default_rng(0)
    n = 2048
    d = np.sort(np.concatenate([10.0 ** (-12 * np.arange(n - 16) / n), 1.7e7 * (1 + rng.random(16))]))
    z = rng.standard_normal(n)
    k, tau = _roots(d, z, 1.0)
    st = fmm_tree_stats(d, k, tau, 1e-10)
    assert st["max_near"] <= 8 and st["flops_per_row"] / n <= 700, st


@pytest.mark.parametrize("n", [40, 65, 777, 3000])
def test_small_and_ragged(n):
    d, k, tau, *_ = interlaced_cauchy(n, 1, n)
    st = fmm_tree_stats(d, k, tau, 1e-10)
    assert st["max_leaf"] <= 33 and st["tasks"] >= 1


@pytest.mark.parametrize("kind", ["gaussian", "graded", "uniform"])
def test_secular_fmm_plan_bounded(kind):
    """The secular FMM plan (K2'): every root's near field stays a small
    fraction of n (a few leaves; the sparse tails of a Gaussian spectrum give the widest
    lists, 24 leaves of 32 at n = 4096), and the directly-summed roots are the last one
    plus the outlier-gap ones."""
    from paper_1707_08369_b200._lib import secfmm_plan_stats
    rng = np.random.default_rng(3)
    n = 4096
    d, _, _ = random_secular(n, rng, kind=kind)
    st = secfmm_plan_stats(np.sort(d))
    assert st["max_near_terms"] <= n // 4, st
    assert 1 <= st["direct_roots"] <= 8, st
    assert st["leaves"] * 32 >= n


def test_secular_fmm_plan_outliers():
    """Outliers far above a graded bulk (C3 after updates): the outlier gap does not make
    any leaf near-field to the whole spectrum; the gap roots are summed directly."""
    from paper_1707_08369_b200._lib import secfmm_plan_stats
    rng = np.random.default_rng(0)
    n = 4096
    d = np.sort(np.concatenate([10.0 ** (-12 * np.arange(n - 16) / n), 1.7e7 * (1 + rng.random(16))]))
    st = secfmm_plan_stats(d)
    assert st["max_near_terms"] <= 6 * 32 and st["direct_roots"] >= 2, st


def test_one_sided_lists_shrink_the_near_field():
    """One-sided separation (P2L / M2P for leaf pairs the symmetric test
    rejects) on a graded spectrum: fewer near pairs and fewer flops than the symmetric
    lists (SVD1_ONE_SIDED=0, read once per process: compared in a subprocess)."""
    import json, os, subprocess, sys
    n = 2048
    d, z, _ = random_secular(n, np.random.default_rng(5), kind="graded")
    k, tau = _roots(d, z, 1.0)
    on = fmm_tree_stats(d, k, tau, 1e-10)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, json, numpy as np; sys.path.insert(0, %r); "
            "from paper_1707_08369_b200._lib import fmm_tree_stats; "
            "a = np.load(sys.argv[1]); print(json.dumps(fmm_tree_stats(a['d'], a['k'], a['tau'], 1e-10)))" % root)
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        f = os.path.join(td, "s.npz")
        np.savez(f, d=d, k=k, tau=tau)
        out = subprocess.run([sys.executable, "-c", code, f], capture_output=True, text=True, check=True,
                             env={**os.environ, "SVD1_ONE_SIDED": "0"}).stdout
    off = json.loads(out.strip().splitlines()[-1])
    assert on["near_pairs"] < off["near_pairs"], (on, off)
    assert on["flops_per_row"] < off["flops_per_row"], (on, off)
    assert on["max_near"] <= off["max_near"]
