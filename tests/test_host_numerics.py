"""Host-side numerics of the product library (FastMath tables, sigma search, relabel) against the committed
reference outputs -- CPU only, through the C-ABI (no compute kernels are launched)."""
import numpy as np

from conftest import load_golden


def test_fastmath_tables_match_reference_fit():
    from paper_2011_03479_b200 import engine as E
    g = load_golden("numerics.json")["tables"]
    for which, name in ((0, "erf"), (1, "exp_neg"), (2, "ratio")):
        flat, odd = E.fastmath_table(which)
        want = np.array([float(v) for v in g[name]["flat"]])
        assert odd == g[name]["odd_mirror"]
        assert np.array_equal(flat[:17], want[:17]) and np.array_equal(flat[65:], want[65:])  # knots, lo, hi
        # coefficients come from a differently-ordered linear solve: equal to rounding
        assert np.abs(flat[17:65] - want[17:65]).max() <= 5e-11


def test_table_values_agree_with_reference_tables_pointwise(oracle):
    """What matters downstream is the function the table represents: <= 1e-11 apart everywhere."""
    import ctypes as C
    import oracle as O
    from paper_2011_03479_b200 import engine as E
    g = load_golden("numerics.json")["tables"]
    mine = O.fastmath_from_flat(E.fastmath_table(0)[0], E.fastmath_table(2)[0])
    want = O.fastmath_from_flat([float(v) for v in g["erf"]["flat"]], [float(v) for v in g["ratio"]["flat"]])
    for x in np.linspace(-7.0, 9.0, 4001):
        a = oracle.lib.go_ratio_fast(C.byref(mine), float(x))
        b = oracle.lib.go_ratio_fast(C.byref(want), float(x))
        assert abs(a - b) <= 1e-11 * max(1.0, abs(b))


def test_sigma_search_matches_reference():
    from paper_2011_03479_b200 import engine as E
    for case in load_golden("numerics.json")["sigma"]:
        he, hn = np.array(case["edge"], np.uint64), np.array(case["nonedge"], np.uint64)
        s, steps = E.optimize_sigma(he, hn, case["nonedge_weight"], 1.5)
        assert s == float(case["sigma"]) and steps == case["steps"]
        obj = E.histogram_objective(he, hn, case["nonedge_weight"], 1.5, s)
        assert abs(obj - float(case["objective"])) <= 1e-12 * abs(float(case["objective"]))
        ds = E.histogram_objective_dsigma(he, hn, case["nonedge_weight"], 1.5, 1.0)
        assert abs(ds - float(case["dsigma_at_1"])) <= 1e-11 * abs(float(case["dsigma_at_1"]))


def test_relabel_and_seed_mixing_match_reference():
    from paper_2011_03479_b200 import engine as E
    for case in load_golden("prep.json")["relabel"]:
        assert E.random_relabel(case["n"], int(case["seed"])).tolist() == case["forward"]
    for s, c, out in load_golden("integer_layer.json")["mix_seed"]:
        assert E.mix_seed(int(s), int(c)) == int(out)


def test_empty_histogram_is_a_config_error():
    import pytest
    from paper_2011_03479_b200 import engine as E
    with pytest.raises(E.ConfigError):
        E.optimize_sigma(np.zeros(512, np.uint64), np.zeros(512, np.uint64), 1.0)
