"""Pins of the oracle's L0 arithmetic and rate table (CPU, -m "not gpu")."""
import math
import os

import numpy as np
import pytest

import oracle
from oracle.fskmc import rate_table, macro_steps, substeps, LIE, STRANG, RANDOM

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_philox_random123_kat():
    """Random123 known-answer vectors (tests/golden/philox_kat.txt)."""
    rows = [l.split() for l in open(os.path.join(GOLDEN, "philox_kat.txt")) if l.strip() and not l.startswith("#")]
    assert len(rows) == 3
    for r in rows:
        v = [int(x, 16) for x in r]
        assert oracle.philox4x32_10(v[0:4], v[4:6]) == tuple(v[6:10])


def _ulp_diff(a, b):
    ia = np.frombuffer(np.float64(a).tobytes(), dtype=np.int64)[0]
    ib = np.frombuffer(np.float64(b).tobytes(), dtype=np.int64)[0]
    return abs(int(ia) - int(ib))


def test_log_spec_within_one_ulp_of_libm():
    """The table-driven FMA log (R26) is within 1 ulp of a correctly rounded log on (0,1]."""
    rng = np.random.default_rng(1)
    xs = list(rng.random(20000)) + [1.0, 0.5, 0.25, 2.0 ** -53, 1 - 2.0 ** -53, 0.7071067811865476,
                                    0.7071067811865475, 1 - 1e-7, 1 - 1e-15, 0.999999]
    xs += list(np.exp(-rng.random(5000) * 36.0))
    worst = 0
    for x in xs:
        if x == 0.0:
            continue
        worst = max(worst, _ulp_diff(oracle.log_spec(x), math.log(x)))
    assert worst <= 1


def test_log_spec_exact_points():
    assert oracle.log_spec(1.0) == 0.0
    assert oracle.log_spec(0.5) == -math.log(2.0)
    assert oracle.log_spec(2.0 ** -53) == -53 * math.log(2.0)
    assert oracle.log_spec(0.0) == -math.inf


def test_rate_table_adsdes_values():
    """eq.(Arrhenius): vacant sites c_a; occupied c_d exp(-beta(K n + h)).
    SPEC S:132 example: c_d=1, beta=1, K=1, h=0, n=2 -> e^{-2} = 0.13534."""
    t = rate_table(0, 2, [0.3, 1.0, 1.0, 1.0, 0.0, 0.0, 0.4, 1.0], 64)
    assert t["n"] == 6
    assert list(t["type"]) == [0, 1, 1, 1, 1, 1]
    assert list(t["kappa"]) == [0, 0, 1, 2, 3, 4]
    assert t["rate"][0] == 0.3
    assert abs(t["rate"][3] - 0.13534) < 1e-5
    for n in range(5):
        assert math.isclose(t["rate"][1 + n], math.exp(-n), rel_tol=1e-15)


def test_rate_table_quantisation_R18():
    t = rate_table(1, 2, [1.0, 1.0, 1.5, 1.0, -2.0, 1.0, 0.4, 1.0], 64)
    F = t["F"]
    bound = max(t["rate"]) * 64 * (2 + 4)
    assert bound * 2.0 ** F <= 2.0 ** 62 < 2 * bound * 2.0 ** F
    for r, u in zip(t["rate"], t["rate_u64"]):
        assert abs(int(u) - r * 2.0 ** F) <= 0.5
    # hops: c_hop exp(-beta K n), n = 0..z-1, per direction (R12), n-major (R31)
    assert t["n"] == 6 + 16
    assert list(t["type"][6:]) == [2] * 16
    assert list(t["dir"][6:]) == [d for _ in range(4) for d in range(4)]
    assert list(t["kappa"][6:]) == [n for n in range(4) for _ in range(4)]
    for i in range(6, 22):
        assert math.isclose(t["rate"][i], math.exp(-1.5 * t["kappa"][i]), rel_tol=1e-15)


def test_rate_table_zgb_table_COrates():
    """Table COrates: CO adsorb k1; O2 adsorb (1-k1)/4 per vacant neighbour;
    CO+O react k2/4 per pair direction from either anchor (R13)."""
    k1, k2 = 0.4, 1.0
    t = rate_table(2, 2, [0, 0, 0, 0, 0, 0, k1, k2], 64)
    assert t["n"] == 13
    assert t["rate"][0] == k1
    assert np.allclose(t["rate"][1:5], (1 - k1) / 4)
    assert np.allclose(t["rate"][5:13], k2 / 4)


def test_macro_steps_R20():
    d, tr = macro_steps(10.0, 1.0)
    assert d == [1.0] * 10 and not tr
    d, tr = macro_steps(1.0, 0.1)
    assert len(d) == 10 and not tr
    d, tr = macro_steps(2.5, 1.0)
    assert d == [1.0, 1.0, 0.5] and tr


def test_substeps_schedules():
    """R1/R2: Lie colour 0 first; Strang half steps to colour 0 (S:295-296 analogues)."""
    assert substeps(LIE, 2, 1.0, 0, 0) == [(0, 1.0), (1, 1.0)]
    assert substeps(STRANG, 2, 1.0, 0, 0) == [(0, 0.5), (1, 1.0), (0, 0.5)]
    assert substeps(STRANG, 4, 1.0, 0, 0) == [(0, .5), (1, .5), (2, .5), (3, 1.0), (2, .5), (1, .5), (0, .5)]
    # random: colours uniform over C (eq.(SLPCS) P(xi=1)=P(xi=2)=1/2)
    cols = [c for w in range(0, 4000, 2) for c, _ in substeps(RANDOM, 2, 1.0, 7, w)]
    assert abs(np.mean(cols) - 0.5) < 4 * 0.5 / math.sqrt(len(cols))
    cols4 = [c for w in range(0, 8000, 4) for c, _ in substeps(RANDOM, 4, 1.0, 7, w)]
    counts = np.bincount(cols4, minlength=4)
    assert counts.min() > 0.25 * len(cols4) - 4 * math.sqrt(len(cols4) * 0.1875)
