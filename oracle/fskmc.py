"""O2 -- the serial fractional-step KMC oracle (bit-exact reference).

TEST INFRASTRUCTURE (see oracle/__init__.py).  Plain Python for the
schedule and observables; the per-window cell loop is plain C
(``orc_window`` in fskmc_oracle.c), a literal linear scan over the canonical
slot list.

Paper map (P:n = PAPER.md line n):
  cells and colours      eq.(decomposition), eq.(sublatt) P:346-350,
                         other groupings P:342-345 (R6: 2 or 4 colours)
  one window             eq.(exact) P:402-417 -- cells of one colour evolve
                         independently for the window
  Lie                    eq.(lie), Steps 1-3 P:422-433 (R1, R3)
  Strang                 eq.(strang) P:452-455 (R2, R3)
  random (SL) schedule   eq.(SLPCS), eq.(SL) P:523-526 (R4)
  observables            mean coverage P:991-995; Hamiltonian P:959-961 (R24)
"""
import ctypes
import math

import numpy as np

from . import lib, philox4x32_10

KIND = {"adsdes": 0, "adsdes_diff": 1, "zgb": 2, "zgb_diff": 3, "zgb_odiff": 4}
NSTATES = {0: 2, 1: 2, 2: 3, 3: 3, 4: 3}
LIE, STRANG, RANDOM = 0, 1, 2
SCHEME = {"lie": LIE, "strang": STRANG, "random": RANDOM}
TAG_SCHED = 1


def model_params(ca=1.0, cd=1.0, beta=1.0, K=0.0, h=0.0, c_hop=0.0, k1=0.4, k2=1.0):
    return [float(ca), float(cd), float(beta), float(K), float(h), float(c_hop), float(k1), float(k2)]


def rate_table(kind: int, ndim: int, params, sites_per_cell: int):
    """a1: the class list with FP64 rates and the R18 u64 quantisation."""
    L = lib()
    n = 64
    ct = (ctypes.c_int * n)(); cd = (ctypes.c_int * n)(); ck = (ctypes.c_int * n)()
    cr = (ctypes.c_double * n)()
    p = (ctypes.c_double * 8)(*params)
    nc = L.orc_classes(kind, ndim, p, ct, cd, ck, cr)
    if nc < 0:
        raise ValueError("unknown model kind")
    u = (ctypes.c_uint64 * nc)()
    F = L.orc_quantise(cr, nc, sites_per_cell, L.orc_types_per_site(kind, ndim), u)
    if F < 0:
        raise ValueError("rates cannot be quantised (negative/inf or too large)")
    return {
        "n": nc,
        "type": np.array(ct[:nc], dtype=np.int32),
        "dir": np.array(cd[:nc], dtype=np.int32),
        "kappa": np.array(ck[:nc], dtype=np.int32),
        "rate": np.array(cr[:nc], dtype=np.float64),
        "rate_u64": np.array(u[:nc], dtype=np.uint64),
        "F": F,
    }


def macro_steps(T: float, dt: float):
    """R20: number of macro-steps and their durations (last one shortened)."""
    if not (dt > 0.0) or T < 0.0:
        raise ValueError("need dt > 0 and T >= 0")
    if T == 0.0:
        return [], False
    n = int(math.ceil(T / dt - 1e-9))
    if n < 1:
        n = 1
    last = T - (n - 1) * dt
    truncated = True
    if abs(last - dt) <= 1e-9 * dt:
        last = dt
        truncated = False
    return [dt] * (n - 1) + [last], truncated


def random_colour(seed: int, window: int, C: int) -> int:
    """R4: xi_w = (C * x0) >> 32 with x0 = Philox(key=seed, ctr=(0, 0, w_lo, w_hi | SCHED<<28))."""
    ctr = (0, 0, window & 0xFFFFFFFF, ((window >> 32) & 0x0FFFFFFF) | (TAG_SCHED << 28))
    x0 = philox4x32_10(ctr, (seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF))[0]
    return (C * x0) >> 32


def substeps(scheme: int, C: int, d: float, seed: int, w0: int):
    """The sub-step list (colour, duration) of ONE macro-step of duration d (R1-R4).

    Lie     eq.(lie):    colours 0..C-1, each for d; colour 0 acts first (R1).
    Strang  eq.(strang): C=2: (0,d/2),(1,d),(0,d/2); C=4: the 7-factor palindrome (R2).
    random  eq.(SLPCS):  C windows of duration d, colour xi_w per global window id (R4).
    """
    h = d * 0.5
    if scheme == LIE:
        return [(c, d) for c in range(C)]
    if scheme == STRANG:
        if C == 2:
            return [(0, h), (1, d), (0, h)]
        return [(0, h), (1, h), (2, h), (3, d), (2, h), (1, h), (0, h)]
    if scheme == RANDOM:
        return [(random_colour(seed, w0 + i, C), d) for i in range(C)]
    raise ValueError("unknown scheme")


def nested_substeps(outer: int, inner: int, C: int, d: float, n_inner: int, seed: int, w0: int):
    """f3, R28: the windows (outer colour o, cell colour c, duration) of ONE nested macro-step.

    Outer factor list over the two outer colours (eq.(opdecomp) on the outer blocks):
      Lie [(0, d), (1, d)];  Strang [(0, d/2), (1, d), (0, d/2)].
    Each outer factor e^{D L^o} is itself split by eq.(opdecomp2): n_inner cycles of
    the inner scheme over the C cell colours of duration D/n_inner each.  Window ids are consumed
    in list order from w0 (the random inner scheme draws xi_w by those ids, R4)."""
    if outer == LIE:
        outer_list = [(0, d), (1, d)]
    elif outer == STRANG:
        outer_list = [(0, d * 0.5), (1, d), (0, d * 0.5)]
    else:
        raise ValueError("nested outer scheme must be lie or strang")
    out = []
    w = w0
    for o, Do in outer_list:
        di = Do / n_inner
        for _ in range(n_inner):
            for c, D in substeps(inner, C, di, seed, w):
                out.append((o, c, D))
                w += 1
    return out


class FSKMC:
    """O2: fractional-step KMC on a uint8 site-major lattice [R][H][W], periodic."""

    def __init__(self, ndim, dims, cell, kind="adsdes", params=None, colours=0, replicas=1, seed=0):
        self.kind = KIND[kind] if isinstance(kind, str) else int(kind)
        self.ndim = int(ndim)
        H, W = (1, int(dims[0])) if self.ndim == 1 else (int(dims[0]), int(dims[1]))
        qy, qx = (1, int(cell[0])) if self.ndim == 1 else (int(cell[0]), int(cell[1]))
        self.H, self.W, self.qy, self.qx = H, W, qy, qx
        self.R = int(replicas)
        cross = self.kind != 0  # hops / pair events write outside the anchor cell
        C = int(colours) or (2 if (self.ndim == 1 or not cross) else 4)
        if C not in (2, 4) or (self.ndim == 1 and C != 2):
            raise ValueError("colours must be 2 (1D) or 2/4 (2D)")
        if cross and self.ndim == 2 and C == 2:
            raise ValueError("cross-cell-writing model needs 4 colours in 2D (R6)")
        if W % qx or H % qy or qx * qy > 64:
            raise ValueError("dims must be divisible by the cell; cell <= 64 sites")
        self.Mx, self.My = W // qx, H // qy
        if self.Mx % 2 or (self.ndim == 2 and self.My % 2):
            raise ValueError("need an even number of cells per axis")
        if cross and (qx < 2 or (self.ndim == 2 and qy < 2)):
            raise ValueError("cross-cell-writing model needs cell extent >= 2 (R7)")
        self.C = C
        self.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
        self.params = params if params is not None else model_params()
        self.table = rate_table(self.kind, self.ndim, self.params, qx * qy)
        self.nstates = NSTATES[self.kind]
        self.lat = np.zeros((self.R, H, W), dtype=np.uint8)
        self.window = 0
        self.time = 0.0
        self.events = 0
        self.W_events = np.zeros(self.R * self.Mx * self.My, dtype=np.uint32)

    # -- state -----------------------------------------------------------
    def set_config(self, lat):
        lat = np.ascontiguousarray(lat, dtype=np.uint8).reshape(self.R, self.H, self.W)
        if lat.size and lat.max() >= self.nstates:
            raise ValueError("spin value out of range")
        self.lat = lat.copy()

    def get_config(self):
        return self.lat.copy()

    # -- one window: eq.(exact) --------------------------------------------
    def substep(self, colour: int, D: float, classes=None) -> int:
        """One window; `classes` (optional set of class indices) restricts the window to those
        mechanisms -- the other classes' rates are 0 (multiscale sub-steps, eq.(strang3))."""
        t = self.table
        ip = ctypes.POINTER(ctypes.c_int)
        rates = t["rate_u64"].copy()
        if classes is not None:
            for i in range(t["n"]):
                if i not in classes:
                    rates[i] = 0
        ev = lib().orc_window(
            self.lat.ctypes.data, self.R, self.H, self.W, self.ndim, self.qx, self.qy,
            self.C, int(colour), float(D), self.window, self.seed,
            t["n"], t["type"].ctypes.data_as(ip), t["dir"].ctypes.data_as(ip),
            t["kappa"].ctypes.data_as(ip), rates.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
            t["F"], self.W_events.ctypes.data)
        self.window += 1
        self.events += int(ev)
        return int(ev)

    def window_cells(self, cells, D: float, window: int):
        """Run window `window` (duration D) on the listed cells only ([n][3] = replica, cy, cx,
        all of one colour), in place; returns the per-cell event counts.  Used to check sampled
        cells of a full-size GPU window from the pre-window lattice (cells are independent)."""
        t = self.table
        ip = ctypes.POINTER(ctypes.c_int)
        cells = np.ascontiguousarray(cells, dtype=np.int64).reshape(-1, 3)
        ev = np.zeros(len(cells), dtype=np.uint32)
        lib().orc_window_cells(
            self.lat.ctypes.data, self.R, self.H, self.W, self.ndim, self.qx, self.qy,
            cells.ctypes.data, len(cells), float(D), int(window), self.seed,
            t["n"], t["type"].ctypes.data_as(ip), t["dir"].ctypes.data_as(ip),
            t["kappa"].ctypes.data_as(ip), t["rate_u64"].ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
            t["F"], ev.ctypes.data)
        return ev

    def macro_step(self, scheme: int, d: float) -> int:
        ev = 0
        for colour, D in substeps(scheme, self.C, d, self.seed, self.window):
            ev += self.substep(colour, D)
        self.time += d
        return ev

    def run(self, T: float, dt: float, scheme="lie") -> bool:
        """kmc_run: returns True when the last macro-step was shortened (R20)."""
        sc = SCHEME[scheme] if isinstance(scheme, str) else int(scheme)
        durs, truncated = macro_steps(T, dt)
        for d in durs:
            self.macro_step(sc, d)
        return truncated

    def run_multiscale(self, T: float, dt: float, n_fast: int, inner="lie", fast_classes=None) -> bool:
        """f2, eq.(strang3): per macro-step d, e^{d/2 L_slow} [e^{(d/n) L_fast}]^n
        e^{d/2 L_slow}, each factor split over the colours with the `inner` scheme.
        Fast classes default to the hop slot types (R12 diffusion / ZGB CO or O diffusion)."""
        sc = SCHEME[inner] if isinstance(inner, str) else int(inner)
        n = self.table["n"]
        if fast_classes is None:
            fast = {i for i in range(n) if int(self.table["type"][i]) in (2, 7, 8)}   # T_HOP, T_COHOP, T_OHOP
        else:
            fast = set(fast_classes)
        slow = set(range(n)) - fast
        if not fast or not slow:
            raise ValueError("multiscale needs a non-empty proper subset of fast classes")
        durs, truncated = macro_steps(T, dt)
        for d in durs:
            h, df = d * 0.5, d / n_fast
            for dur, cls in [(h, slow)] + [(df, fast)] * n_fast + [(h, slow)]:
                for colour, D in substeps(sc, self.C, dur, self.seed, self.window):
                    self.substep(colour, D, cls)
            self.time += d
        return truncated

    def nested_cells(self, outer_colour: int, colour: int, block: int):
        """Cells (replica, cy, cx) of cell colour `colour` inside the outer blocks of colour
        `outer_colour` (R28): outer block = cell row // block (2D) or cell // block (1D), outer
        colour = block index mod 2."""
        r, cy, cx = np.meshgrid(np.arange(self.R), np.arange(self.My), np.arange(self.Mx), indexing="ij")
        ob = (cy if self.ndim == 2 else cx) // block
        if self.C == 2:
            col = cx % 2 if self.ndim == 1 else (cx + cy) % 2
        else:
            col = cx % 2 + 2 * (cy % 2)
        sel = (ob % 2 == outer_colour) & (col == colour)
        return np.stack([r[sel], cy[sel], cx[sel]], axis=1).astype(np.int64)

    def run_nested(self, T: float, dt: float, n_inner: int, outer="lie", inner="lie", block=2) -> bool:
        """f3, eq.(sublatt2)/eq.(opdecomp2), R28: per macro-step d the outer scheme
        over the two outer block colours, each outer factor split into n_inner cycles of the inner
        scheme over the cell colours (nested_substeps); one window per (outer, cell colour)."""
        so = SCHEME[outer] if isinstance(outer, str) else int(outer)
        si = SCHEME[inner] if isinstance(inner, str) else int(inner)
        n_inner = int(n_inner)
        block = int(block)
        nb = self.My if self.ndim == 2 else self.Mx
        if n_inner < 1 or block < 2 or block % 2 or nb % (2 * block):
            raise ValueError("nested: need n_inner >= 1, even block >= 2, cells per axis % (2 block) == 0")
        durs, truncated = macro_steps(T, dt)
        cache = {}
        M = self.Mx * self.My
        for d in durs:
            for o, c, D in nested_substeps(so, si, self.C, d, n_inner, self.seed, self.window):
                if (o, c) not in cache:
                    cache[(o, c)] = self.nested_cells(o, c, block)
                cells = cache[(o, c)]
                ev = self.window_cells(cells, D, self.window)
                gid = cells[:, 0] * M + cells[:, 1] * self.Mx + cells[:, 2]
                self.W_events[gid] += ev
                self.events += int(ev.sum())
                self.window += 1
            self.time += d
        return truncated

    # -- a8 observables ----------------------------------------------------
    def colour_map(self):
        cy = np.arange(self.H) // self.qy
        cx = np.arange(self.W) // self.qx
        if self.C == 2:
            if self.ndim == 1:
                return np.broadcast_to((cx & 1)[None, :], (self.H, self.W))
            return (cx[None, :] + cy[:, None]) & 1
        return (cx[None, :] & 1) + 2 * (cy[:, None] & 1)

    def correlation(self, rmax: int, state: int = 1):
        """f1: pair counts of the 2-point correlation: x[r] = #{sites x : sigma(x) =
        sigma(x + r e_x) = state}, y[r] along y (zeros in 1D), summed over replicas; periodic."""
        occ = self.lat == state
        x = np.array([int((occ & np.roll(occ, -r, axis=2)).sum()) for r in range(rmax + 1)], dtype=np.int64)
        if self.ndim == 2:
            y = np.array([int((occ & np.roll(occ, -r, axis=1)).sum()) for r in range(rmax + 1)], dtype=np.int64)
        else:
            y = np.zeros(rmax + 1, dtype=np.int64)
        return {"x": x, "y": y}

    def observables(self):
        lat = self.lat
        S = self.nstates
        n_state = np.array([int((lat == s).sum()) for s in range(S)] + [0] * (4 - S), dtype=np.int64)
        nn = np.zeros((4, 4), dtype=np.int64)
        axes = [2] if self.ndim == 1 else [2, 1]
        for ax in axes:
            nb = np.roll(lat, -1, axis=ax)           # bond (x, x+e)
            for a in range(S):
                for b in range(S):
                    c = int(((lat == a) & (nb == b)).sum())
                    lo, hi = min(a, b), max(a, b)
                    nn[lo, hi] += c
        for a in range(4):
            for b in range(a):
                nn[a, b] = nn[b, a]
        cmap = self.colour_map()
        by_col = np.zeros((4, 4), dtype=np.int64)
        for c in range(self.C):
            m = cmap == c
            for s in range(S):
                by_col[c, s] = int(((lat == s) & m[None, :, :]).sum())
        N = lat.size
        K, h = self.params[3], self.params[4]
        return {
            "time": self.time, "windows": self.window, "events": self.events,
            "n_state": n_state, "nn_pairs": nn, "n_state_by_colour": by_col,
            "coverage": n_state.astype(np.float64) / N,
            # R24: paper Hamiltonian H = -K sum_<xy> s s' + h sum s
            "energy": -K * float(nn[1, 1]) + h * float(n_state[1]),
        }
