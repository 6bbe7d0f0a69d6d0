"""Closed forms the paper fixes (pins for the oracles).

TEST INFRASTRUCTURE (see oracle/__init__.py).

* noninteracting_theta   K=0 two-state law (north_star; [L^E,L^O]=0)
* paper_cov1d            eq.(exactcov1d) P:1022-1034 (paper's own variables)
* paper_cov2d, beta_c    eq.(exactcov2d), sinh(beta_c K/2)=1 P:1080-1081
* tm_coverage_1d         finite-N transfer matrix of the literal rates' stationary
                         law (R9): pi ~ exp(beta K sum_<xy> s s' + mu sum s),
                         mu = beta h + ln(ca/cd)
* h_dyn_from_paper       R9: h_dyn = h_paper - z K
"""
import math

import numpy as np


def noninteracting_theta(t, ca, cd, beta=1.0, h=0.0):
    """P(sigma=1) at time t from the empty site: ka/(ka+kd) (1 - e^{-(ka+kd) t}),
    ka = ca, kd = cd e^{-beta h} (eq.(Arrhenius) with K = 0)."""
    ka = ca
    kd = cd * math.exp(-beta * h)
    return ka / (ka + kd) * (1.0 - math.exp(-(ka + kd) * t))


def paper_cov1d(beta, K, h_paper):
    """eq.(exactcov1d): c = 1/2 (1 + sinh h' / sqrt(sinh^2 h' + e^{-4K'})), K' = beta K/4,
    h' = beta (h - K)/2."""
    Kp = beta * K / 4.0
    hp = beta * (h_paper - K) / 2.0
    return 0.5 * (1.0 + math.sinh(hp) / math.sqrt(math.sinh(hp) ** 2 + math.exp(-4.0 * Kp)))


def beta_c(K=1.0):
    """sinh(beta_c K / 2) = 1."""
    return 2.0 * math.asinh(1.0) / K


def paper_cov2d(beta, K=1.0):
    """eq.(exactcov2d): 1/2 (1 + [1 - sinh(beta K/2)^-4]^{1/8}) for beta > beta_c, else 1/2."""
    if beta <= beta_c(K):
        return 0.5
    return 0.5 * (1.0 + (1.0 - math.sinh(0.5 * beta * K) ** -4) ** 0.125)


def h_dyn_from_paper(h_paper, K, ndim):
    """R9: the paper's field maps onto the literal rates' h by h_dyn = h_paper - z K."""
    return h_paper - 2 * ndim * K


def tm_coverage_1d(N, beta, K, h_dyn, ca=1.0, cd=1.0):
    """Exact equilibrium coverage of the literal Arrhenius rates on a periodic ring of N
    sites (N = None: thermodynamic limit), by the 2x2 transfer matrix."""
    mu = beta * h_dyn + math.log(ca / cd)
    T = np.array([[math.exp(beta * K * a * b + mu * (a + b) / 2.0) for b in (0, 1)] for a in (0, 1)])
    if N is None:
        w, v = np.linalg.eigh(T)
        lead = v[:, np.argmax(w)]
        return float(lead[1] ** 2 / (lead @ lead))
    TN = np.linalg.matrix_power(T, N)
    return float(TN[1, 1] / np.trace(TN))


def tm_correlation_1d(N, beta, K, h_dyn, r, ca=1.0, cd=1.0):
    """Exact equilibrium E[sigma_0 sigma_r] of the literal rates on a periodic ring of N sites
    (N = None: thermodynamic limit), by the transfer matrix: Tr(D T^r D T^{N-r}) / Tr(T^N)."""
    mu = beta * h_dyn + math.log(ca / cd)
    T = np.array([[math.exp(beta * K * a * b + mu * (a + b) / 2.0) for b in (0, 1)] for a in (0, 1)])
    D = np.diag([0.0, 1.0])
    if N is None:
        w, v = np.linalg.eigh(T)
        order = np.argsort(w)[::-1]
        w, v = w[order], v[:, order]
        # sum_k (w_k/w_0)^r <v0|D|vk><vk|D|v0>
        return float(sum((w[k] / w[0]) ** r * (v[:, 0] @ D @ v[:, k]) ** 2 for k in range(2)))
    TN = np.linalg.matrix_power(T, N)
    return float(np.trace(D @ np.linalg.matrix_power(T, r) @ D @ np.linalg.matrix_power(T, N - r)) / np.trace(TN))


def paper_corr1d_corrected(beta, K, h_paper, r):
    """eq.(exactcorr1d) read as R15: E[s_0 s_r] = c^2 + 1/4 (1 + e^{4K'} sinh^2 h')^{-1}
    (lambda_-/lambda_+)^r, with the printed bracket for lambda_-/lambda_+ and c from eq.(exactcov1d)
    (the printed prefactor is inverted and c^2 is missing)."""
    Kp = beta * K / 4.0
    hp = beta * (h_paper - K) / 2.0
    c = paper_cov1d(beta, K, h_paper)
    root = math.sqrt(1.0 + math.exp(4 * Kp) * math.sinh(hp) ** 2)
    ratio = (math.exp(Kp) * math.cosh(hp) - math.exp(-Kp) * root) / (math.exp(Kp) * math.cosh(hp) + math.exp(-Kp) * root)
    return c * c + 0.25 / (1.0 + math.exp(4 * Kp) * math.sinh(hp) ** 2) * ratio ** r


def stationary_event_rate(ca, theta):
    """P7: in any stationary spin-flip state adsorption flux = desorption flux, so the
    event rate per site is 2 ca (1 - theta)."""
    return 2.0 * ca * (1.0 - theta)
