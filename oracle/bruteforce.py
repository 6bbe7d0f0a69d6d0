"""Brute-force master equation on tiny lattices (<= 12 sites).

TEST INFRASTRUCTURE (see oracle/__init__.py).  Written independently of the
C oracle: the generator matrix Q of eq.(generator) is assembled
over the full configuration space from the paper's rates (eq.(Arrhenius)
P:963-968, eq.(adsdesrate), Table COrates, R12-R13),
and split by cell colour as in eq.(gendecomp)/eq.(opdecomp) (P:323-329,
P:356-359).  The exact law of every scheme is then the product of matrix
exponentials p0 * prod_k exp(d_k Q^{c_k}) (eq.(lie), eq.(strang), eq.(SL)).

Conventions: row-vector laws, Q[from, to]; configuration index
sum_i sigma_i S^i with sites i = y*W + x.  FP64 rates, no quantisation.
"""
import itertools
import math

import numpy as np
import scipy.sparse as sp
from scipy.sparse.linalg import expm_multiply


class Lattice:
    """A periodic 1D ring (H=1) or 2D torus with a cell partition and colouring."""

    def __init__(self, ndim, H, W, qy, qx, C):
        self.ndim, self.H, self.W, self.qy, self.qx, self.C = ndim, H, W, qy, qx, C
        self.N = H * W

    def site(self, y, x):
        return (y % self.H) * self.W + (x % self.W)

    def nbrs(self, i):
        y, x = divmod(i, self.W)
        out = [self.site(y, x - 1), self.site(y, x + 1)]
        if self.ndim == 2:
            out += [self.site(y - 1, x), self.site(y + 1, x)]
        return out   # order: -x, +x, -y, +y

    def colour(self, i):
        y, x = divmod(i, self.W)
        cy, cx = y // self.qy, x // self.qx
        if self.C == 2:
            return cx % 2 if self.ndim == 1 else (cx + cy) % 2
        return cx % 2 + 2 * (cy % 2)


def _events(model, lat, conf, i):
    """All (rate, {site: new_state}) events anchored at site i in configuration conf."""
    kind = model["kind"]
    s = conf[i]
    nb = lat.nbrs(i)
    ev = []
    if kind in ("adsdes", "adsdes_diff"):
        n = sum(conf[j] == 1 for j in nb)
        if s == 0:
            ev.append((model["ca"], {i: 1}))
        else:
            U = model["K"] * n + model["h"]
            ev.append((model["cd"] * math.exp(-model["beta"] * U), {i: 0}))
        if kind == "adsdes_diff" and s == 1:
            for j in nb:
                if conf[j] == 0:
                    ev.append((model["c_hop"] * math.exp(-model["beta"] * model["K"] * n), {i: 0, j: 1}))
    else:  # ZGB: 0 vacant, 1 CO, 2 O
        z = len(nb)
        k1, k2 = model["k1"], model["k2"]
        if s == 0:
            ev.append((k1, {i: 1}))
            for j in nb:
                if conf[j] == 0:
                    ev.append(((1 - k1) / z, {i: 2, j: 2}))
        if s == 1:
            for j in nb:
                if conf[j] == 2:
                    ev.append((k2 / z, {i: 0, j: 0}))
                if kind == "zgb_diff" and conf[j] == 0:
                    ev.append((model["c_hop"], {i: 0, j: 1}))
        if s == 2:
            for j in nb:
                if conf[j] == 1:
                    ev.append((k2 / z, {i: 0, j: 0}))
                if kind == "zgb_odiff" and conf[j] == 0:     # fast O diffusion
                    ev.append((model["c_hop"], {i: 0, j: 2}))
    return ev


def _is_hop(i, upd, conf):
    """Diffusion events move a particle: the anchor empties and one neighbour takes its species."""
    return (len(upd) == 2 and upd[i] == 0 and conf[i] != 0
            and any(j != i and v == conf[i] for j, v in upd.items()))


def generators(model, lat, mech=None):
    """Return (Q, [Q^0..Q^{C-1}], S) as sparse CSR matrices; Q = sum_c Q^c.
    mech = "fast" keeps only diffusion (hop) events, "slow" only the others (eq.(fastslow))."""
    S = 2 if model["kind"] in ("adsdes", "adsdes_diff") else 3
    N = lat.N
    nconf = S ** N
    powers = [S ** i for i in range(N)]
    rows = [[] for _ in range(lat.C)]
    cols = [[] for _ in range(lat.C)]
    vals = [[] for _ in range(lat.C)]
    for idx, conf in enumerate(itertools.product(range(S), repeat=N)):
        conf = conf[::-1]  # conf[i] = digit i (least significant first)
        for i in range(N):
            c = lat.colour(i)
            for rate, upd in _events(model, lat, conf, i):
                if rate == 0.0:
                    continue
                if mech is not None and (mech == "fast") != _is_hop(i, upd, conf):
                    continue
                to = idx + sum((v - conf[j]) * powers[j] for j, v in upd.items())
                rows[c].append(idx); cols[c].append(to); vals[c].append(rate)
    Qc = []
    for c in range(lat.C):
        A = sp.csr_matrix((vals[c], (rows[c], cols[c])), shape=(nconf, nconf))
        A = A - sp.diags(np.asarray(A.sum(axis=1)).ravel())
        Qc.append(A.tocsr())
    Q = Qc[0]
    for A in Qc[1:]:
        Q = Q + A
    return Q.tocsr(), Qc, S


def evolve(p, Q, t):
    """p e^{tQ} for a row vector p."""
    if t == 0.0:
        return p.copy()
    return expm_multiply(Q.T * t, p)


def law(p0, Q, Qc, scheme, dt, T, C):
    """Exact law at time T of: 'exact' (e^{TQ}), 'lie', 'strang', 'random' (xi-averaged)."""
    if scheme == "exact":
        return evolve(p0, Q, T)
    n = int(round(T / dt))
    p = p0.copy()
    for _ in range(n):
        if scheme == "lie":
            for c in range(C):
                p = evolve(p, Qc[c], dt)
        elif scheme == "strang":
            if C == 2:
                seq = [(0, dt / 2), (1, dt), (0, dt / 2)]
            else:
                h = dt / 2
                seq = [(0, h), (1, h), (2, h), (3, dt), (2, h), (1, h), (0, h)]
            for c, d in seq:
                p = evolve(p, Qc[c], d)
        elif scheme == "random":
            for _w in range(C):
                p = sum(evolve(p, Qc[c], dt) for c in range(C)) / C
        else:
            raise ValueError(scheme)
    return p


def _inner(inner, C, d):
    if inner == "lie":
        return [(c, d) for c in range(C)]
    h = d / 2
    if C == 2:
        return [(0, h), (1, d), (0, h)]
    return [(0, h), (1, h), (2, h), (3, d), (2, h), (1, h), (0, h)]


def law_multiscale(p0, Qslow_c, Qfast_c, dt, T, n_fast, inner, C):
    """Exact law of the spatio-temporal scheme of eq.(strang3): per macro-step
    e^{dt/2 L_slow} [e^{(dt/n) L_fast}]^n e^{dt/2 L_slow}, each factor split over the colours by the
    deterministic `inner` scheme ('lie' or 'strang')."""
    p = p0.copy()
    for _ in range(int(round(T / dt))):
        for dur, Qs in [(dt / 2, Qslow_c)] + [(dt / n_fast, Qfast_c)] * n_fast + [(dt / 2, Qslow_c)]:
            for c, d in _inner(inner, C, dur):
                p = evolve(p, Qs[c], d)
    return p


def law_sequence(p0, Qc, seq):
    """Exact law after the given window sequence [(colour, duration), ...]: p0 prod e^{d Q^c}
    (e.g. one realisation xi_1, xi_2, ... of the random schedule, eq.(SL))."""
    p = p0.copy()
    for c, d in seq:
        p = evolve(p, Qc[c], d)
    return p


class NestedLattice(Lattice):
    """f3 (eq.(sublatt2), R28): the cell partition of Lattice, grouped into outer
    blocks of `block` cells along the last cell axis of the lattice (cell rows in 2D, cells in
    1D) coloured by block parity.  colour(i) = outer * C + cell colour, so generators() returns
    the 2C generators L^{o,c} of eq.(opdecomp2), indexed o*C + c."""

    def __init__(self, ndim, H, W, qy, qx, C, block):
        super().__init__(ndim, H, W, qy, qx, C)
        self.C_cell, self.block = C, block
        self.C = 2 * C

    def colour(self, i):
        y, x = divmod(i, self.W)
        cy, cx = y // self.qy, x // self.qx
        if self.C_cell == 2:
            c = cx % 2 if self.ndim == 1 else (cx + cy) % 2
        else:
            c = cx % 2 + 2 * (cy % 2)
        o = ((cy if self.ndim == 2 else cx) // self.block) % 2
        return o * self.C_cell + c


def law_nested(p0, Qc2, C, dt, T, n_inner, outer, inner):
    """Exact law of the nested scheme (R28) with a deterministic inner scheme: per macro-step the
    outer Lie [(0,dt),(1,dt)] or Strang [(0,dt/2),(1,dt),(0,dt/2)] factors, each split into
    n_inner cycles of `inner` ('lie' / 'strang') over the C cell colours; Qc2[o*C + c]."""
    outer_list = [(0, dt), (1, dt)] if outer == "lie" else [(0, dt / 2), (1, dt), (0, dt / 2)]
    p = p0.copy()
    for _ in range(int(round(T / dt))):
        for o, Do in outer_list:
            for _k in range(n_inner):
                for c, d in _inner(inner, C, Do / n_inner):
                    p = evolve(p, Qc2[o * C + c], d)
    return p


def coverage_values(lat, S, state=1, sites=None):
    """Per-configuration coverage of `state` (fraction of `sites`, default all)."""
    N = lat.N
    sites = list(range(N)) if sites is None else list(sites)
    confs = np.array(list(itertools.product(range(S), repeat=N)))[:, ::-1]
    return (confs[:, sites] == state).sum(axis=1) / len(sites)


def point_mass(S, N, conf):
    idx = sum(int(v) * S ** i for i, v in enumerate(conf))
    p = np.zeros(S ** N)
    p[idx] = 1.0
    return p
