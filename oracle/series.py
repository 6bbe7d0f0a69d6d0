"""f1 -- the coverage process and its statistics (reading R30).

TEST INFRASTRUCTURE (see oracle/__init__.py).

The coverage process of a replica, C_t = |Lambda|^-1 sum_x 1{S_t(x) = state}, sampled
at the start and after every macro-step, is what the paper plots as sample paths (Fig. path1D,
P:1057-1058), its autocorrelation function from M independent realisations (Fig. autocorr1D,
P:1059-1062; 2D: Fig. dynamics2d) and its equilibrium distribution (Fig. pdf2d,
P:1037-1040).  The paper prints no estimator; R30 takes the plain stationary one over samples
[first, n) and all M replicas, c = count / N, n' = n - first:

    c_bar    = sum_{i,r} c_{i,r} / (M n')
    gamma(l) = sum_r sum_{i=first}^{n-1-l} (c_{i,r} - c_bar)(c_{i+l,r} - c_bar) / (M (n' - l))
    acf(l)   = gamma(l) / gamma(0)           (0 when gamma(0) = 0)
    hist[b]  = #{(i, r) : floor(count_{i,r} bins / (N + 1)) = b}

written out below as plain loops.  Pins (tests/test_oracle_series.py): exact values on series whose
autocorrelation is known by hand (alternating, constant, two-level), and the non-interacting
closed forms (exact for the splitting, [L^E, L^O] = 0): acf(l) = e^{-(ka+kd) l dt} and
N C ~ Binomial(N, ka/(ka+kd)) at stationarity.
"""
import math

import numpy as np

from .fskmc import SCHEME, macro_steps


def counts(o, state=1):
    """Per-replica number of sites in `state` of an O2 lattice [R][H][W]."""
    return np.array([int((o.lat[r] == state).sum()) for r in range(o.R)], dtype=np.int64)


def record(o, T, dt, scheme="lie", state=1, step=None):
    """Sample 0 now, then one sample after every macro-step of run(T, dt, scheme) (the shortened
    last one included).  `step(d)` overrides the macro-step (multiscale / nested runs)."""
    sc = SCHEME[scheme] if isinstance(scheme, str) else int(scheme)
    out = [counts(o, state)]
    durs, _ = macro_steps(T, dt)
    for d in durs:
        if step is None:
            o.macro_step(sc, d)
        else:
            step(d)
        out.append(counts(o, state))
    return np.array(out, dtype=np.int64)


def stats(series, nsite, max_lag, first=0, bins=0):
    """R30 estimator over samples [first, n) of `series` ([n][M] counts)."""
    ser = np.asarray(series, dtype=np.int64)
    n, M = ser.shape
    np_ = n - first
    if not (0 <= first < n) or not (0 <= max_lag < np_):
        raise ValueError("need 0 <= first < n and 0 <= max_lag < n - first")
    tot = 0
    for i in range(first, n):
        for r in range(M):
            tot += int(ser[i, r])
    mean = tot / (float(nsite) * np_ * M)
    gamma = []
    for l in range(max_lag + 1):
        s = 0.0
        for i in range(first, n - l):
            for r in range(M):
                a = float(ser[i, r]) / nsite - mean
                b = float(ser[i + l, r]) / nsite - mean
                s += a * b
        gamma.append(s / ((np_ - l) * M))
    g0 = gamma[0]
    acf = np.array([g / g0 if g0 > 0 else 0.0 for g in gamma])
    hist = None
    if bins:
        hist = np.zeros(bins, dtype=np.int64)
        for i in range(first, n):
            for r in range(M):
                hist[min(int(ser[i, r]) * bins // (nsite + 1), bins - 1)] += 1
    return {"mean": mean, "var": g0, "acf": acf, "hist": hist}


def noninteracting_acf(lag_time, ca, cd, beta=1.0, h=0.0):
    """Stationary autocorrelation of the coverage of independent two-state sites (K = 0):
    every site relaxes at rate ka + kd, so Cov(C_t, C_{t+s}) = theta (1 - theta) / N e^{-(ka+kd) s}
    and acf(s) = e^{-(ka+kd) s}, ka = ca, kd = cd e^{-beta h} (eq.(Arrhenius) with K = 0)."""
    return math.exp(-(ca + cd * math.exp(-beta * h)) * lag_time)


def binomial_pmf(N, theta):
    """Stationary law of N C for independent sites: Binomial(N, theta)."""
    k = np.arange(N + 1)
    logp = (np.array([math.lgamma(N + 1) - math.lgamma(j + 1) - math.lgamma(N - j + 1) for j in k])
            + k * math.log(theta) + (N - k) * math.log1p(-theta))
    return np.exp(logp)
