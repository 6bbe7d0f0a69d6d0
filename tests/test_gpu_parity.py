"""GPU parity: the CUDA path (through the C ABI) against the O2 oracle, bit-exact after
EVERY window (lattice, per-cell event counts, totals) and on the observables.

Bar: integer / bit work is bit-exact.  The clock is FP64 but both sides
execute the same IEEE operation sequence, so the lattice is bit-exact too.
"""
import numpy as np
import pytest

import synth_inputs as si
from oracle.fskmc import FSKMC, model_params

pytestmark = pytest.mark.gpu


def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def make_pair(ndim, dims, cell, kind, params, colours=0, replicas=1, seed=1234):
    import paper_1105_4673_b200 as kmc
    _cuda()
    gpu = kmc.KMC(ndim, dims, cell, kind=kind, colours=colours, replicas=replicas, seed=seed, **params)
    orc = FSKMC(ndim, dims, cell, kind, model_params(**params), colours=colours, replicas=replicas, seed=seed)
    return gpu, orc


def assert_same_state(gpu, orc, tag=""):
    a = gpu.get_config()
    b = orc.get_config()
    if not np.array_equal(a, b):
        diff = np.argwhere(a != b)
        raise AssertionError(f"{tag}: {len(diff)} sites differ, first {diff[:4].tolist()}")
    obs = gpu.observables(per_cell=True)
    assert obs["events"] == orc.events, (tag, obs["events"], orc.events)
    R, My, Mx = obs["per_cell_events"].shape
    assert np.array_equal(obs["per_cell_events"].reshape(-1), orc.W_events), tag
    assert obs["windows"] == orc.window


def run_windows(gpu, orc, scheme, dt, nmacro):
    """Drive both through the same schedule one window at a time (oracle schedule), and
    separately check the library's own kmc_run schedule reproduces it."""
    from oracle.fskmc import substeps, SCHEME
    sc = SCHEME[scheme]
    for i in range(nmacro):
        for colour, D in substeps(sc, orc.C, dt, orc.seed, orc.window):
            gpu.substep(colour, D)
            orc.substep(colour, D)
            assert_same_state(gpu, orc, f"macro {i} colour {colour}")
        orc.time += dt


CASES = {
    # name: (ndim, dims, cell, kind, params, colours, replicas, init, scheme, dt, nmacro)
    "1d_noninteracting_cfg1": (1, (1024,), (32,), "adsdes", dict(ca=1.0, cd=0.5, beta=1.0, K=0.0, h=0.0), 0, 16, 0.0, "lie", 0.5, 3),
    "1d_ising_strang": (1, (4096,), (32,), "adsdes", dict(ca=1, cd=1, beta=2.0, K=1.0, h=-0.5), 0, 3, 0.5, "strang", 0.5, 3),
    "1d_ising_q4_random": (1, (512,), (4,), "adsdes", dict(ca=1, cd=1, beta=1.0, K=1.0, h=-1.0), 0, 4, 0.5, "random", 1.0, 3),
    "1d_ising_q64": (1, (1024,), (64,), "adsdes", dict(ca=1, cd=1, beta=1.0, K=1.0, h=-1.0), 0, 2, 0.3, "lie", 1.0, 2),
    "2d_ising_8x8": (2, (128, 128), (8, 8), "adsdes", dict(ca=1, cd=1, beta=1.5, K=1.0, h=-2.0), 0, 1, 0.5, "lie", 1.0, 2),
    "2d_ising_random": (2, (64, 64), (8, 8), "adsdes", dict(ca=1, cd=1, beta=2.2, K=1.0, h=-2.0), 0, 2, 0.9, "random", 1.0, 2),
    "2d_ising_rect_cell": (2, (64, 128), (2, 16), "adsdes", dict(ca=1, cd=1, beta=1.0, K=1.0, h=-2.0), 0, 1, 0.5, "strang", 0.5, 2),
    "2d_ising_1x1_cell": (2, (16, 16), (1, 1), "adsdes", dict(ca=1, cd=1, beta=1.0, K=1.0, h=-2.0), 0, 3, 0.5, "lie", 0.7, 3),
    # quiescent cells: no adsorption (c_a = 0), so every cell whose sites are all vacant has lambda = 0
    "2d_ising_quiescent": (2, (64, 64), (8, 8), "adsdes", dict(ca=0.0, cd=1.0, beta=1.0, K=1.0, h=-2.0), 0, 2, 0.02, "strang", 1.0, 3),
    "2d_ising_ragged": (2, (24, 40), (4, 4), "adsdes", dict(ca=0.7, cd=1.3, beta=1.2, K=0.8, h=-1.0), 0, 5, 0.4, "strang", 1.0, 2),
    "2d_diffusion_4col": (2, (64, 64), (8, 8), "adsdes_diff", dict(ca=1, cd=1, beta=1.5, K=1.0, h=-2.0, c_hop=1.0), 0, 1, 0.5, "strang", 0.5, 2),
    "2d_diffusion_q2": (2, (32, 32), (2, 2), "adsdes_diff", dict(ca=0.3, cd=0.3, beta=1.0, K=1.0, h=-2.0, c_hop=2.0), 0, 2, 0.5, "lie", 0.5, 2),
    "1d_diffusion": (1, (512,), (8,), "adsdes_diff", dict(ca=0.5, cd=0.5, beta=1.0, K=1.0, h=-1.0, c_hop=1.5), 0, 3, 0.5, "lie", 0.5, 3),
    "2d_zgb": (2, (64, 64), (4, 4), "zgb", dict(k1=0.4, k2=1.0), 0, 1, None, "lie", 0.5, 3),
    "2d_zgb_diff": (2, (32, 64), (4, 8), "zgb_diff", dict(k1=0.45, k2=1.0, c_hop=1.0), 0, 2, None, "strang", 0.5, 2),
    "1d_zgb": (1, (256,), (4,), "zgb", dict(k1=0.4, k2=1.0), 0, 4, None, "random", 0.5, 3),
    # ZGB with fast O diffusion (R33)
    "2d_zgb_odiff": (2, (64, 32), (4, 4), "zgb_odiff", dict(k1=0.45, k2=1.0, c_hop=2.0), 0, 2, None, "lie", 0.5, 3),
    "2d_zgb_odiff_rect": (2, (32, 64), (2, 8), "zgb_odiff", dict(k1=0.4, k2=1.0, c_hop=1.0), 0, 1, None, "strang", 0.5, 2),
    "1d_zgb_odiff": (1, (256,), (4,), "zgb_odiff", dict(k1=0.4, k2=1.0, c_hop=3.0), 0, 4, None, "random", 0.5, 3),
    # 8 x 8 cells: the window kernels built with the cell shape as a compile-time constant
    "2d_zgb_8x8": (2, (64, 128), (8, 8), "zgb", dict(k1=0.42, k2=1.0), 0, 1, None, "lie", 0.5, 3),
    "2d_zgb_diff_8x8": (2, (64, 64), (8, 8), "zgb_diff", dict(k1=0.4, k2=1.0, c_hop=1.0), 0, 2, None, "strang", 0.5, 2),
    "2d_zgb_odiff_8x8": (2, (64, 64), (8, 8), "zgb_odiff", dict(k1=0.4, k2=1.0, c_hop=2.0), 0, 1, None, "random", 0.5, 3),
}


@pytest.mark.parametrize("name", list(CASES))
def test_bit_exact_every_window(name):
    ndim, dims, cell, kind, params, C, R, init, scheme, dt, nmacro = CASES[name]
    gpu, orc = make_pair(ndim, dims, cell, kind, params, C, R)
    shape = gpu.local_shape
    if init is None:
        lat = si.categorical_lattice(shape, [0.6, 0.2, 0.2], seed=si.SEED_BASE + 5)
    else:
        lat = si.bernoulli_lattice(shape, init, seed=si.SEED_BASE + 3)
    gpu.set_config(lat)
    orc.set_config(lat)
    assert_same_state(gpu, orc, "init")
    run_windows(gpu, orc, scheme, dt, nmacro)
    assert orc.events > 0


SPIN_FLIP_2D = [n for n, c in CASES.items() if c[0] == 2 and c[3] == "adsdes"]
SPIN_FLIP_2D_EXTRA = {
    # 4 colours for a spin-flip model; partial tiles (dims not multiples of the 32x64-cell tile)
    "2d_ising_4col": (2, (48, 80), (2, 2), "adsdes", dict(ca=1, cd=1, beta=1.3, K=1.0, h=-2.0), 4, 2, 0.5, "strang", 0.5, 2),
    "2d_ising_big_partial": (2, (328, 544), (4, 4), "adsdes", dict(ca=1, cd=1, beta=1.5, K=1.0, h=-2.0), 0, 1, 0.5, "lie", 0.05, 3),
}


SPIN_FLIP = [n for n, c in CASES.items() if c[3] == "adsdes"]


@pytest.mark.parametrize("kernel", ["queue", "tile", "group2", "group8", "group32"])
@pytest.mark.parametrize("name", SPIN_FLIP + list(SPIN_FLIP_2D_EXTRA))
def test_bit_exact_kernel_modes(name, kernel):
    """Every window kernel (lane-queue, shared-memory tile, g lanes per cell) is bit-exact vs O2
    every window."""
    ndim, dims, cell, kind, params, C, R, init, scheme, dt, nmacro = {**CASES, **SPIN_FLIP_2D_EXTRA}[name]
    if kernel == "tile" and ndim == 1:
        pytest.skip("the tile kernel is 2D only")
    gpu, orc = make_pair(ndim, dims, cell, kind, params, C, R)
    gpu.set_kernel(kernel)
    lat = si.bernoulli_lattice(gpu.local_shape, init, seed=si.SEED_BASE + 4)
    gpu.set_config(lat)
    orc.set_config(lat)
    run_windows(gpu, orc, scheme, dt, nmacro)
    assert orc.events > 0


@pytest.mark.parametrize("scheme", ["lie", "strang", "random"])
def test_library_schedule_matches_oracle_run(scheme):
    """kmc_run's own schedule (R1-R4, R20 truncation) equals the oracle's run()."""
    p = dict(ca=1, cd=1, beta=1.5, K=1.0, h=-2.0)
    gpu, orc = make_pair(2, (64, 64), (8, 8), "adsdes", p, 0, 2)
    lat = si.bernoulli_lattice(gpu.local_shape, 0.5, seed=7)
    gpu.set_config(lat); orc.set_config(lat)
    tr_g = gpu.run(2.5, 1.0, scheme)
    tr_o = orc.run(2.5, 1.0, scheme)
    assert tr_g and tr_o
    assert_same_state(gpu, orc, scheme)
    assert abs(gpu.get_state()[1] - 2.5) < 1e-12


@pytest.mark.parametrize("kernel", ["auto", "group2", "group4"])
@pytest.mark.parametrize("ndim,dims,cell,colours,scheme,dt", [
    (2, (64, 64), (8, 8), 0, "lie", 1.0),
    (2, (64, 64), (8, 8), 0, "strang", 0.7),
    (2, (48, 80), (2, 2), 4, "strang", 0.5),         # 7 windows per macro-step
    (2, (32, 64), (4, 4), 4, "random", 0.5),
    (1, (1024,), (32,), 0, "random", 1.0),
    (1, (512,), (8,), 0, "strang", 0.5),
])
def test_group_kernel_run_matches_oracle_run(kernel, ndim, dims, cell, colours, scheme, dt):
    """kmc_run's own schedule on small spin-flip lattices (the lane-group kernel, auto or forced g)
    with 2 and 4 colours: the lattice, the per-cell event counts and the totals equal the oracle's
    run() after every call, including a truncated last step (R20)."""
    p = dict(ca=1, cd=1, beta=1.3, K=1.0, h=-2.0 if ndim == 2 else -1.0)
    gpu, orc = make_pair(ndim, dims, cell, "adsdes", p, colours, 3)
    gpu.set_kernel(kernel)
    lat = si.bernoulli_lattice(gpu.local_shape, 0.5, seed=11)
    gpu.set_config(lat)
    orc.set_config(lat)
    for T in (2 * dt, 2.5 * dt):
        assert gpu.run(T, dt, scheme) == orc.run(T, dt, scheme)
        assert_same_state(gpu, orc, f"{scheme} T={T}")
    assert orc.events > 0


@pytest.mark.parametrize("kind,ndim,dims,cell,colours,replicas", [
    ("adsdes", 2, (64, 96), (4, 8), 0, 2),
    ("zgb", 2, (64, 96), (4, 8), 0, 2),             # 3 states, 4 colours
    ("adsdes", 2, (48, 80), (2, 2), 4, 3),          # spin flip with 4 colours
    ("adsdes", 1, (512,), (8,), 0, 5),              # 1D rings (one +e bond per site)
    ("zgb_odiff", 1, (256,), (4,), 0, 3),
    ("adsdes", 2, (16, 16), (1, 1), 0, 1),          # 1-site cells
    ("adsdes_diff", 2, (24, 40), (4, 4), 0, 7),     # ragged: rows of 10 cells, 7 replicas
    # rows of 128 cells: the kernel's row-aligned fast path (one locate per 128 cells, +x words by shuffle)
    ("adsdes", 1, (1024,), (8,), 0, 3),
    ("zgb", 2, (16, 1024), (4, 8), 0, 2),
    ("adsdes", 2, (32, 2048), (8, 8), 0, 1),        # 256 cells per row, 4 cell rows
])
def test_observables_match_oracle(kind, ndim, dims, cell, colours, replicas):
    """a8 counters (sites per state, by colour, unordered bonds), coverage and energy = the oracle's
    (itself pinned by hand-counted lattices, tests/test_oracle_observables.py).  The kernel counts
    only the occupied states and completes the vacant entries from the lattice identities."""
    params = {"adsdes": dict(ca=1, cd=1, beta=1.5, K=1.0, h=-2.0), "zgb": dict(k1=0.4, k2=1.0),
              "zgb_odiff": dict(k1=0.4, k2=1.0, c_hop=1.0),
              "adsdes_diff": dict(ca=1, cd=1, beta=1.5, K=1.0, h=-2.0, c_hop=1.0)}[kind]
    init = None if kind.startswith("zgb") else 0.5
    gpu, orc = make_pair(ndim, dims, cell, kind, params, colours, replicas)
    lat = (si.bernoulli_lattice(gpu.local_shape, 0.4, seed=3) if init is not None
           else si.categorical_lattice(gpu.local_shape, [0.5, 0.3, 0.2], seed=3))
    gpu.set_config(lat); orc.set_config(lat)
    gpu.run(1.0, 0.5, "lie"); orc.run(1.0, 0.5, "lie")
    a, b = gpu.observables(), orc.observables()
    for key in ("n_state", "nn_pairs", "n_state_by_colour"):
        assert np.array_equal(a[key], b[key]), (kind, key, a[key], b[key])
    assert a["events"] == b["events"] and a["windows"] == b["windows"]
    assert np.allclose(a["coverage"], b["coverage"], rtol=0, atol=1e-15)
    assert abs(a["energy"] - b["energy"]) <= 1e-9 * max(1.0, abs(b["energy"]))


@pytest.mark.parametrize("kind,ndim,dims,cell", [("adsdes", 2, (64, 64), (8, 8)), ("zgb", 2, (32, 32), (4, 4)),
                                                  ("adsdes_diff", 1, (256,), (8,))])
def test_observables_device_matches_sync(kind, ndim, dims, cell):
    """kmc_observables_device (enqueued, no host sync) + kmc_obs_decode == kmc_observables for the
    same states, including the events, windows and time words; several snapshots in one buffer."""
    torch = _cuda()
    import paper_1105_4673_b200 as kmc
    g = kmc.KMC(ndim, dims, cell, kind=kind, replicas=2, seed=4)
    lat = (si.bernoulli_lattice(g.local_shape, 0.5, seed=3) if g.nstates == 2
           else si.categorical_lattice(g.local_shape, [0.5, 0.25, 0.25], seed=3))
    g.set_config(lat)
    buf = torch.zeros((4, kmc.OBS_WORDS), dtype=torch.int64, device="cuda")
    ref = []
    for i in range(4):
        g.run(0.5, 0.25, "strang")
        g.observables_device(buf[i].data_ptr())
        ref.append(g.observables())
    host = buf.cpu().numpy()
    for i in range(4):
        got = g.obs_decode(host[i])
        for key in ("time", "windows", "events", "energy"):
            assert got[key] == ref[i][key], (i, key)
        for key in ("n_state", "nn_pairs", "n_state_by_colour", "coverage"):
            assert np.array_equal(got[key], ref[i][key]), (i, key)
    assert host[3, 37] == ref[3]["windows"] and host[3, 39] == 0


def test_resume_run_split_equals_whole():
    p = dict(ca=1, cd=1, beta=1.5, K=1.0, h=-2.0, c_hop=1.0)
    import paper_1105_4673_b200 as kmc
    _cuda()
    lat = si.bernoulli_lattice((1, 64, 64), 0.5, seed=9)
    a = kmc.KMC(2, (64, 64), (8, 8), kind="adsdes_diff", seed=5, **p)
    b = kmc.KMC(2, (64, 64), (8, 8), kind="adsdes_diff", seed=5, **p)
    a.set_config(lat); b.set_config(lat)
    a.run(3.0, 1.0, "strang")
    b.run(1.0, 1.0, "strang"); b.run(2.0, 1.0, "strang")
    assert np.array_equal(a.get_config(), b.get_config())
    # checkpoint / restore into a fresh context
    w, t = a.get_state()
    c = kmc.KMC(2, (64, 64), (8, 8), kind="adsdes_diff", seed=5, **p)
    c.set_config(a.get_config()); c.set_state(w, t)
    a.run(1.0, 1.0, "strang"); c.run(1.0, 1.0, "strang")
    assert np.array_equal(a.get_config(), c.get_config())


def test_set_state_same_parity_after_claimed_chunks():
    """Restoring a window counter of the same parity as the last window (kmc_set_state) after a
    window whose warps claimed chunks from the dynamic pool (8192^2: more active cells than one
    chunk per resident warp): the next window still covers every cell -- identical to a fresh
    context restored to the same state."""
    import paper_1105_4673_b200 as kmc
    _cuda()
    p = dict(ca=1, cd=1, beta=1.5, K=1.0, h=-2.0)
    a = kmc.KMC(2, (8192, 8192), (8, 8), kind="adsdes", seed=3, **p)
    a.init_random((0.5, 0.5), seed=1)
    a.substep(0, 1.0)                                  # window 0 (parity 0) claims pool chunks
    lat = a.get_config()
    a.set_state(2, 0.0)                                # window 2: parity 0 again
    a.substep(1, 1.0)
    b = kmc.KMC(2, (8192, 8192), (8, 8), kind="adsdes", seed=3, **p)
    b.set_config(lat)
    b.set_state(2, 0.0)
    b.substep(1, 1.0)
    assert np.array_equal(a.get_config(), b.get_config())


def test_degenerate_cases():
    import paper_1105_4673_b200 as kmc
    _cuda()
    # all rates zero: quiescent cells, no events
    g = kmc.KMC(2, (32, 32), (8, 8), kind="adsdes", ca=0.0, cd=0.0)
    g.set_config(si.bernoulli_lattice(g.local_shape, 0.5, seed=1))
    before = g.get_config()
    g.run(5.0, 1.0, "lie")
    assert np.array_equal(before, g.get_config()) and g.observables()["events"] == 0
    # zero-duration window
    g = kmc.KMC(2, (32, 32), (8, 8), kind="adsdes", ca=1.0, cd=1.0)
    g.substep(0, 0.0)
    assert g.observables()["events"] == 0
    # invalid spin value: rejected, lattice unchanged
    lat = si.bernoulli_lattice(g.local_shape, 0.5, seed=2)
    g.set_config(lat)
    bad = lat.copy(); bad[0, 3, 3] = 2
    with pytest.raises(kmc.KmcError) as e:
        g.set_config(bad)
    assert e.value.status == kmc.KMC_EINVAL
    assert np.array_equal(g.get_config(), lat)
    with pytest.raises(kmc.KmcError):
        g.substep(2, 1.0)          # colour out of range


def test_device_buffers_roundtrip():
    torch = _cuda()
    import paper_1105_4673_b200 as kmc
    g = kmc.KMC(2, (64, 64), (8, 8), kind="zgb", stream=torch.cuda.current_stream().cuda_stream)
    lat = si.categorical_lattice(g.local_shape, [0.4, 0.3, 0.3], seed=4)
    t = torch.from_numpy(lat).cuda()
    g.set_config_device(t.data_ptr(), t.numel())
    out = torch.empty_like(t)
    g.get_config_device(out.data_ptr(), out.numel())
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), lat)
    assert np.array_equal(g.get_config(), lat)


FULL_SIZE = {"adsdes": "ising2d_32768", "zgb": "zgb2d_32768", "adsdes_diff": "diff2d_8192"}


@pytest.mark.parametrize("kind", list(FULL_SIZE))
def test_full_size_sampled_cells(kind):
    """The bench workloads at full size (BASELINE target 32768^2, ZGB 32768^2, diffusion 8192^2) in
    the launch configuration bench.py times: one window on the GPU; 512 sampled active cells
    recomputed by the oracle from the pre-window lattice (cells of one colour are independent
    within a window, eq.(exact))."""
    torch = _cuda()
    import paper_1105_4673_b200 as kmc
    wl = dict(si.WORKLOADS[FULL_SIZE[kind]])
    H, W = wl["dims"]
    qy, qx = wl["cell"]
    g = kmc.KMC(2, (H, W), (qy, qx), kind=kind, seed=99, **wl["params"])
    if kind.startswith("adsdes"):
        lat = si.bernoulli_lattice((1, H, W), 0.5, seed=si.SEED_BASE)
    else:
        lat = si.categorical_lattice((1, H, W), [0.5, 0.25, 0.25], seed=si.SEED_BASE)
    g.set_config(lat)
    g.run(2.0 * wl["dt"], wl["dt"], wl["scheme"])   # advance a little so the state is not the input
    pre = g.get_config()
    w0, _ = g.get_state()
    ev_pre = g.observables(per_cell=True)["per_cell_events"][0]
    colour = 1
    D = wl["dt"]
    g.substep(colour, D)
    post = g.get_config()
    ev_post = g.observables(per_cell=True)["per_cell_events"][0]
    orc = FSKMC(2, (H, W), (qy, qx), kind, model_params(**wl["params"]), seed=99)
    orc.set_config(pre)
    rng = np.random.default_rng(17)
    Mx, My = W // qx, H // qy
    C = orc.C
    cells = []
    while len(cells) < 512:
        cy, cx = int(rng.integers(My)), int(rng.integers(Mx))
        col = ((cx + cy) & 1) if C == 2 else ((cx & 1) + 2 * (cy & 1))
        if col == colour:
            cells.append((0, cy, cx))
    cells = np.array(sorted(set(cells)))
    ev = orc.window_cells(cells, D, w0)
    got = orc.get_config()
    for (r, cy, cx), k in zip(cells, ev):
        ys, xs = slice(cy * qy, (cy + 1) * qy), slice(cx * qx, (cx + 1) * qx)
        assert np.array_equal(post[0, ys, xs], got[0, ys, xs]), (cy, cx)
        assert int(ev_post[cy, cx]) - int(ev_pre[cy, cx]) == int(k), (cy, cx)
    assert ev.sum() > 0


@pytest.mark.parametrize("kind,params,scheme,dt,cell", [
    ("adsdes", dict(ca=1, cd=1, beta=1.5, K=1.0, h=-2.0), "lie", 1.0, (8, 8)),
    ("adsdes_diff", dict(ca=0.5, cd=0.5, beta=1.0, K=1.0, h=-2.0, c_hop=2.0), "strang", 0.5, (4, 4)),
    ("zgb", dict(k1=0.45, k2=1.0), "random", 0.5, (2, 4)),
])
@pytest.mark.parametrize("world", [2, 4])
def test_virtual_ranks_bit_identical(kind, params, scheme, dt, cell, world):
    """slabs + halo exchange (+ reverse XOR deltas) on G virtual ranks of one GPU give
    the bit-identical lattice, event counts and observables of G = 1 (global ids)."""
    import paper_1105_4673_b200 as kmc
    _cuda()
    dims = (64, 32)
    one = kmc.KMC(2, dims, cell, kind=kind, seed=33, replicas=2, **params)
    grp = kmc.VGroup(world, dims, cell, kind=kind, seed=33, replicas=2, **params)
    if kind == "adsdes":          # ghost-row slabs through the tile kernel, G = 1 through the queue kernel
        one.set_kernel("queue")
        for rk in grp.ranks:
            rk.set_kernel("tile")
    lat = (si.bernoulli_lattice(one.local_shape, 0.5, seed=2) if kind != "zgb"
           else si.categorical_lattice(one.local_shape, [0.5, 0.25, 0.25], seed=2))
    one.set_config(lat)
    grp.set_config(lat)
    for _ in range(3):
        one.run(2 * dt, dt, scheme)
        grp.run(2 * dt, dt, scheme)
        assert np.array_equal(one.get_config(), grp.get_config())
    a, b = one.observables(), grp.observables()
    assert a["events"] == b["events"] > 0
    for key in ("n_state", "nn_pairs", "n_state_by_colour"):
        assert np.array_equal(a[key], b[key]), key


@pytest.mark.parametrize("ndim,dims,cell,kind,R,rmax", [
    (2, (64, 96), (8, 8), "adsdes", 2, 40),
    (2, (48, 40), (4, 2), "zgb", 3, 39),
    (1, (512,), (32,), "adsdes", 4, 100),
    (1, (256,), (4,), "zgb", 2, 70),
])
def test_correlation_counts_match_oracle(ndim, dims, cell, kind, R, rmax):
    """f1: kmc_correlation pair counts equal the oracle's numpy definition (every state, x and y)."""
    gpu, orc = make_pair(ndim, dims, cell, kind, {}, 0, R)
    lat = (si.bernoulli_lattice(gpu.local_shape, 0.45, seed=8) if kind == "adsdes"
           else si.categorical_lattice(gpu.local_shape, [0.4, 0.35, 0.25], seed=8))
    gpu.set_config(lat)
    orc.set_config(lat)
    for state in range(gpu.nstates):
        a, b = gpu.correlation(rmax, state), orc.correlation(rmax, state)
        assert np.array_equal(a["x"], b["x"]), (state, "x")
        assert np.array_equal(a["y"], b["y"]), (state, "y")


@pytest.mark.parametrize("ndim,dims,cell,kind,params,inner,nf", [
    (2, (64, 64), (4, 4), "adsdes_diff", dict(ca=0.5, cd=0.5, beta=1.0, K=1.0, h=-2.0, c_hop=8.0), "lie", 4),
    (2, (32, 64), (4, 8), "zgb_diff", dict(k1=0.45, k2=1.0, c_hop=10.0), "strang", 5),
    (1, (256,), (4,), "adsdes_diff", dict(ca=0.5, cd=0.5, beta=1.0, K=1.0, h=-1.0, c_hop=5.0), "random", 3),
    # the paper's named case: ZGB with fast O diffusion sub-cycled
    (2, (64, 64), (4, 4), "zgb_odiff", dict(k1=0.45, k2=1.0, c_hop=10.0), "strang", 5),
    (2, (32, 64), (4, 8), "zgb_odiff", dict(k1=0.4, k2=1.0, c_hop=20.0), "lie", 8),
])
def test_multiscale_bit_exact(ndim, dims, cell, kind, params, inner, nf):
    """f2: kmc_run_multiscale (eq.(strang3), fast hops sub-cycled) is bit-exact vs O2."""
    gpu, orc = make_pair(ndim, dims, cell, kind, params, 0, 2)
    lat = (si.bernoulli_lattice(gpu.local_shape, 0.4, seed=12) if kind == "adsdes_diff"
           else si.categorical_lattice(gpu.local_shape, [0.5, 0.3, 0.2], seed=12))
    gpu.set_config(lat)
    orc.set_config(lat)
    for _ in range(2):
        gpu.run_multiscale(1.0, 0.5, nf, inner)
        orc.run_multiscale(1.0, 0.5, nf, inner)
        assert_same_state(gpu, orc, f"multiscale {kind} {inner}")
    assert orc.events > 0


@pytest.mark.parametrize("ndim,dims,cell", [(2, (64, 64), (4, 4)), (1, (256,), (8,))])
def test_multiscale_split_hop_blocks_bit_exact(ndim, dims, cell):
    """f2 with a fast set that splits the R31 hop blocks (x-direction hops fast, y-direction hops and
    the spin flips slow): hop rates differ within a block, so the windows run the generic 22-mask
    diffusion step instead of the block-walk step -- bit-exact vs O2 either way."""
    z = 2 * ndim
    fast = [2 + z + n * z + d for n in range(z) for d in (0, 1) if d < z and (ndim == 2 or d == 0)]
    params = dict(ca=0.5, cd=0.5, beta=1.0, K=1.0, h=-2.0, c_hop=6.0)
    gpu, orc = make_pair(ndim, dims, cell, "adsdes_diff", params, 0, 2)
    lat = si.bernoulli_lattice(gpu.local_shape, 0.4, seed=13)
    gpu.set_config(lat)
    orc.set_config(lat)
    mask = sum(1 << c for c in fast)
    for _ in range(2):
        gpu.run_multiscale(1.0, 0.5, 3, "strang", fast_classes=mask)
        orc.run_multiscale(1.0, 0.5, 3, "strang", fast_classes=fast)
        assert_same_state(gpu, orc, "multiscale split hop blocks")
    assert orc.events > 0


def test_multiscale_split_zgb_odiff_groups_bit_exact():
    """ZGB_ODIFF with the O hops along x fast and along y slow (splits the hop group): the generic
    ZGB step with the O-hop classes -- bit-exact vs O2."""
    params = dict(k1=0.45, k2=1.0, c_hop=4.0)
    gpu, orc = make_pair(2, (32, 32), (4, 4), "zgb_odiff", params, 0, 2)
    lat = si.categorical_lattice(gpu.local_shape, [0.5, 0.2, 0.3], seed=15)
    gpu.set_config(lat)
    orc.set_config(lat)
    fast = [13, 14]                                  # O hops -x, +x (classes 1 + 3 z + d)
    for _ in range(2):
        gpu.run_multiscale(1.0, 0.5, 3, "strang", fast_classes=sum(1 << c for c in fast))
        orc.run_multiscale(1.0, 0.5, 3, "strang", fast_classes=fast)
        assert_same_state(gpu, orc, "multiscale split zgb_odiff groups")
    assert orc.events > 0


def test_multiscale_split_zgb_groups_bit_exact():
    """f2 with a fast set that splits a ZGB direction group (O2 adsorption along x fast, the rest
    slow): group rates differ within a window, so the windows run the generic ZGB step instead of
    the grouped one -- bit-exact vs O2 either way."""
    params = dict(k1=0.45, k2=1.0, c_hop=2.0)
    gpu, orc = make_pair(2, (32, 64), (4, 8), "zgb_diff", params, 0, 2)
    lat = si.categorical_lattice(gpu.local_shape, [0.5, 0.3, 0.2], seed=14)
    gpu.set_config(lat)
    orc.set_config(lat)
    fast = [1, 2]                                    # O2 adsorption, directions -x and +x
    for _ in range(2):
        gpu.run_multiscale(1.0, 0.5, 2, "lie", fast_classes=sum(1 << c for c in fast))
        orc.run_multiscale(1.0, 0.5, 2, "lie", fast_classes=fast)
        assert_same_state(gpu, orc, "multiscale split zgb groups")
    assert orc.events > 0


NESTED = [
    # ndim, dims, cell, kind, params, block, outer, inner, n_inner
    (2, (64, 128), (8, 8), "adsdes", dict(ca=1, cd=1, beta=1.5, K=1.0, h=-2.0), 2, "lie", "lie", 2),
    (2, (64, 64), (4, 4), "zgb", dict(k1=0.45, k2=1.0), 4, "strang", "strang", 2),
    (2, (32, 64), (4, 4), "adsdes_diff", dict(ca=0.5, cd=0.5, beta=1.0, K=1.0, h=-2.0, c_hop=2.0), 2, "lie", "random", 3),
    (1, (1024,), (32,), "adsdes", dict(ca=1, cd=1, beta=2.0, K=1.0, h=-0.5), 4, "strang", "lie", 1),
    (1, (256,), (4,), "zgb_diff", dict(k1=0.4, k2=1.0, c_hop=0.8), 8, "lie", "strang", 2),
    (2, (64, 64), (4, 4), "zgb_odiff", dict(k1=0.45, k2=1.0, c_hop=1.5), 4, "lie", "strang", 2),
]


@pytest.mark.parametrize("ndim,dims,cell,kind,params,block,outer,inner,n_inner", NESTED)
def test_nested_bit_exact(ndim, dims, cell, kind, params, block, outer, inner, n_inner):
    """f3: kmc_run_nested (eq.(opdecomp2), R28) is bit-exact vs O2's run_nested after every call."""
    gpu, orc = make_pair(ndim, dims, cell, kind, params, 0, 2)
    lat = (si.bernoulli_lattice(gpu.local_shape, 0.4, seed=14) if kind.startswith("adsdes")
           else si.categorical_lattice(gpu.local_shape, [0.5, 0.3, 0.2], seed=14))
    gpu.set_config(lat)
    orc.set_config(lat)
    for i in range(2):
        t1 = gpu.run_nested(1.0, 0.5, n_inner, outer, inner, block)
        t2 = orc.run_nested(1.0, 0.5, n_inner, outer, inner, block)
        assert t1 == t2 is False
        assert_same_state(gpu, orc, f"nested {kind} {outer}/{inner} call {i}")
    assert orc.events > 0


@pytest.mark.parametrize("kind,params,cell,block", [
    ("adsdes", dict(ca=1, cd=1, beta=1.5, K=1.0, h=-2.0), (8, 8), 2),
    ("adsdes_diff", dict(ca=0.5, cd=0.5, beta=1.0, K=1.0, h=-2.0, c_hop=2.0), (4, 4), 2),
    ("zgb", dict(k1=0.45, k2=1.0), (4, 4), 4),
])
@pytest.mark.parametrize("world", [2, 4])
def test_nested_virtual_ranks_bit_identical(kind, params, cell, block, world):
    """f3 on G virtual ranks: ONE halo exchange (+ reverse XOR deltas) per outer factor instead of
    per window gives the bit-identical result of G = 1 -- the ghost rows belong to the inactive
    outer colour for the whole factor (R28)."""
    import paper_1105_4673_b200 as kmc
    _cuda()
    dims = (64, 32) if cell == (8, 8) else (64, 16)
    one = kmc.KMC(2, dims, cell, kind=kind, seed=35, replicas=2, **params)
    grp = kmc.VGroup(world, dims, cell, kind=kind, seed=35, replicas=2, **params)
    if (dims[0] // cell[0]) // world % block:
        pytest.skip("blocks would straddle ranks")
    lat = (si.bernoulli_lattice(one.local_shape, 0.5, seed=3) if kind != "zgb"
           else si.categorical_lattice(one.local_shape, [0.5, 0.25, 0.25], seed=3))
    one.set_config(lat)
    grp.set_config(lat)
    for outer, inner, n in (("lie", "lie", 3), ("strang", "strang", 2)):
        one.run_nested(1.0, 0.5, n, outer, inner, block)
        grp.run_nested(1.0, 0.5, n, outer, inner, block)
        assert np.array_equal(one.get_config(), grp.get_config()), (outer, inner)
    a, b = one.observables(), grp.observables()
    assert a["events"] == b["events"] > 0


def test_nested_uneven_slabs_validated_globally():
    """f3 on uneven slabs (advisor finding): the nested geometry is checked against the GLOBAL
    cell-row count and every slab bound, identically on every rank.  48 x 32 with 4 x 4 cells has
    12 cell rows = 3 outer blocks of 4 (odd: blocks 0 and 2 would share an outer colour across the
    periodic seam) -- rejected even though rank 0's slab (4 rows) x world looks fine; a bound that
    splits an outer block is rejected too."""
    import paper_1105_4673_b200 as kmc
    _cuda()
    grp = kmc.VGroup(2, (48, 32), (4, 4), kind="adsdes", row_bounds=[0, 4, 12], ca=1, cd=1, beta=1.0, K=1.0, h=-2.0)
    with pytest.raises(kmc.KmcError) as e:
        grp.run_nested(1.0, 0.5, 1, "lie", "lie", 4)
    assert e.value.status == 2
    grp = kmc.VGroup(2, (64, 32), (4, 4), kind="adsdes", row_bounds=[0, 6, 16], ca=1, cd=1, beta=1.0, K=1.0, h=-2.0)
    with pytest.raises(kmc.KmcError) as e:
        grp.run_nested(1.0, 0.5, 1, "lie", "lie", 4)
    assert e.value.status == 2
    grp.run_nested(1.0, 0.5, 1, "lie", "lie", 2)    # block 2 divides every bound: accepted


def test_nested_errors():
    """kmc_run_nested argument checks (include/kmc.h): KMC_EINVAL / KMC_EPARTITION."""
    import paper_1105_4673_b200 as kmc
    _cuda()
    g = kmc.KMC(2, (48, 64), (8, 8), kind="adsdes", seed=1)     # 6 cell rows
    for args, code in [((1, "lie", "lie", 3), 1), ((0, "lie", "lie", 2), 1), ((1, "random", "lie", 2), 1),
                       ((1, "lie", "lie", 2), 2), ((1, "lie", "lie", 6), 2)]:
        with pytest.raises(kmc.KmcError) as e:
            g.run_nested(1.0, 0.5, *args)
        assert e.value.status == code, (args, e.value)
    assert g.observables()["windows"] == 0          # nothing ran


def _pack_words(lat, qy, qx, nplanes):
    """The documented kmc_set_config_packed layout, written out with numpy (test helper):
    words[p][cy][r][cx] bit (ly*qx + lx) = (site value == p + 1)."""
    R, H, W = lat.shape
    My, Mx = H // qy, W // qx
    out = np.zeros((nplanes, My, R, Mx), dtype=np.uint64)
    weights = (np.uint64(1) << np.arange(qy * qx, dtype=np.uint64))
    for p in range(nplanes):
        b = (lat == p + 1).reshape(R, My, qy, Mx, qx).transpose(1, 0, 3, 2, 4).reshape(My, R, Mx, qy * qx)
        out[p] = (b.astype(np.uint64) * weights).sum(axis=-1, dtype=np.uint64)
    return out


@pytest.mark.parametrize("ndim,dims,cell,kind,R", [
    (2, (64, 96), (8, 8), "adsdes", 2),
    (2, (32, 48), (4, 2), "zgb", 3),
    (1, (512,), (32,), "adsdes", 4),
    (1, (96,), (6,), "zgb_diff", 2),
])
def test_packed_config_roundtrip_and_run(ndim, dims, cell, kind, R):
    """kmc_set/get_config_packed: the documented bit layout (numpy packing) round-trips against the
    uint8 path, and a run from a packed upload is bit-identical to a run from the uint8 upload."""
    gpu, orc = make_pair(ndim, dims, cell, kind, {}, 0, R)
    lat = (si.bernoulli_lattice(gpu.local_shape, 0.45, seed=21) if kind == "adsdes"
           else si.categorical_lattice(gpu.local_shape, [0.4, 0.35, 0.25], seed=21))
    qy, qx = (1, cell[0]) if ndim == 1 else cell
    words = _pack_words(lat, qy, qx, gpu.packed_shape[0])
    assert words.shape == gpu.packed_shape
    gpu.set_config(lat)
    assert np.array_equal(gpu.get_config_packed(), words)
    import paper_1105_4673_b200 as kmc
    g2 = kmc.KMC(ndim, dims, cell, kind=kind, replicas=R, seed=1234)
    g2.set_config_packed(words)
    assert np.array_equal(g2.get_config(), lat)
    gpu.run(1.0, 0.5, "strang")
    g2.run(1.0, 0.5, "strang")
    assert np.array_equal(gpu.get_config(), g2.get_config())
    orc.set_config(lat)
    orc.run(1.0, 0.5, "strang")
    assert np.array_equal(g2.get_config(), orc.get_config())


def test_packed_config_validation():
    """Bits outside a cell's sites (cell of 8 sites) and CO+O on one site are KMC_EINVAL; the
    lattice is left unchanged."""
    import paper_1105_4673_b200 as kmc
    _cuda()
    g = kmc.KMC(2, (16, 16), (4, 2), kind="zgb", seed=3)
    lat = si.categorical_lattice(g.local_shape, [0.5, 0.25, 0.25], seed=4)
    g.set_config(lat)
    w = g.get_config_packed()
    bad = w.copy()
    bad[0, 0, 0, 0] |= np.uint64(1) << np.uint64(8)              # site 8 of a 4x2 cell does not exist
    with pytest.raises(kmc.KmcError) as e:
        g.set_config_packed(bad)
    assert e.value.status == 1
    bad = w.copy()
    bad[1, 1, 0, 1] |= bad[0, 1, 0, 1] | np.uint64(1)             # a site both CO and O
    bad[0, 1, 0, 1] |= np.uint64(1)
    with pytest.raises(kmc.KmcError):
        g.set_config_packed(bad)
    assert np.array_equal(g.get_config(), lat)
    with pytest.raises(ValueError):
        g.set_config_packed(w[:, :1])


@pytest.mark.parametrize("kind,dims,cell,params", [
    ("adsdes", (64, 64), (8, 8), dict(ca=1, cd=1, beta=1.5, K=1.0, h=-2.0)),
    ("zgb", (32, 32), (4, 4), dict(k1=0.4, k2=1.0)),
])
def test_staged_config_pipelined_upload(kind, dims, cell, params):
    """kmc_stage_config_packed / kmc_commit_config: the staged copy overlaps the run in flight
    without touching it; after the commit the next run starts from the staged lattice, bit-identical
    to the synchronous set_config_packed path; protocol errors are KMC_ESTATE and an invalid staged
    configuration is discarded at the commit (KMC_EINVAL, lattice unchanged)."""
    import paper_1105_4673_b200 as kmc
    _cuda()
    a = kmc.KMC(2, dims, cell, kind=kind, replicas=2, seed=9, **params)
    b = kmc.KMC(2, dims, cell, kind=kind, replicas=2, seed=9, **params)
    np_ = a.packed_shape[0]
    mk = ((lambda s: si.bernoulli_lattice(a.local_shape, 0.5, seed=s)) if kind == "adsdes"
          else (lambda s: si.categorical_lattice(a.local_shape, [0.5, 0.25, 0.25], seed=s)))
    lat1, lat2 = mk(1), mk(2)
    w1, w2 = _pack_words(lat1, *cell, np_), _pack_words(lat2, *cell, np_)
    a.set_config_packed(w1)
    b.set_config_packed(w1)
    for step in range(3):
        a.run(2.0, 0.5, "strang")                      # enqueued, may still be running ...
        a.stage_config_packed(w2 if step % 2 == 0 else w1)   # ... while the next input is copied
        b.run(2.0, 0.5, "strang")
        assert np.array_equal(a.get_config(), b.get_config()), "staging touched the running state"
        a.commit_config()
        b.set_config_packed(w2 if step % 2 == 0 else w1)
        assert np.array_equal(a.get_config(), b.get_config())
    a.run(1.0, 0.5, "lie")
    b.run(1.0, 0.5, "lie")
    assert np.array_equal(a.get_config(), b.get_config())
    assert a.observables()["events"] == b.observables()["events"]
    with pytest.raises(kmc.KmcError) as e:
        a.commit_config()                              # nothing staged
    assert e.value.status == 6
    a.stage_config_packed(w2)
    with pytest.raises(kmc.KmcError):
        a.stage_config_packed(w2)                      # one pending stage at a time
    with pytest.raises(kmc.KmcError):
        a.set_config(lat1)                             # synchronous setters wait for the commit
    a.commit_config()
    assert np.array_equal(a.get_config(), lat2)
    if kind == "zgb":
        bad = w1.copy()
        bad[1, 1, 0, 1] |= bad[0, 1, 0, 1] | np.uint64(1)    # a site both CO and O
        bad[0, 1, 0, 1] |= np.uint64(1)
        a.stage_config_packed(bad)
        with pytest.raises(kmc.KmcError) as e:
            a.commit_config()
        assert e.value.status == 1
        assert np.array_equal(a.get_config(), lat2)
        a.stage_config_packed(w1)                      # usable again after the rejected commit
        a.commit_config()
        assert np.array_equal(a.get_config(), lat1)


@pytest.mark.parametrize("kind,dims,cell,params", [
    ("adsdes", (64, 64), (8, 8), dict(ca=1, cd=1, beta=1.5, K=1.0, h=-2.0)),
    ("zgb", (32, 32), (4, 4), dict(k1=0.4, k2=1.0)),
])
def test_async_download_consistent(kind, dims, cell, params):
    """kmc_download_config_packed: the asynchronous D2H returns the lattice as of the call even when
    windows are enqueued right after it -- in place (they wait for the copy) or on a configuration
    committed after it (they overlap the copy) -- and the state after those windows is the same as
    without any download."""
    import paper_1105_4673_b200 as kmc
    torch = _cuda()
    a = kmc.KMC(2, dims, cell, kind=kind, replicas=2, seed=19, **params)
    b = kmc.KMC(2, dims, cell, kind=kind, replicas=2, seed=19, **params)
    mk = ((lambda s: si.bernoulli_lattice(a.local_shape, 0.5, seed=s)) if kind == "adsdes"
          else (lambda s: si.categorical_lattice(a.local_shape, [0.5, 0.25, 0.25], seed=s)))
    lat = mk(1)
    a.set_config(lat)
    b.set_config(lat)
    pinned = torch.empty(int(np.prod(a.packed_shape)), dtype=torch.int64).pin_memory()
    buf = pinned.numpy().view(np.uint64).reshape(a.packed_shape)
    # (1) windows in place right after the download
    a.run(1.0, 0.5, "lie")
    a.download_config_packed(buf)
    a.run(1.0, 0.5, "lie")
    a.download_wait()
    b.run(1.0, 0.5, "lie")
    assert np.array_equal(buf, b.get_config_packed())
    b.run(1.0, 0.5, "lie")
    assert np.array_equal(a.get_config_packed(), b.get_config_packed())
    # (2) stage -> run -> download -> commit -> run (the e2e pipeline of bench.py)
    nxt = _pack_words(mk(2), cell[0], cell[1], a.packed_shape[0])
    a.stage_config_packed(nxt)
    a.run(1.0, 0.5, "strang")
    a.download_config_packed(buf)
    a.commit_config()
    a.run(1.0, 0.5, "strang")
    a.download_wait()
    b.run(1.0, 0.5, "strang")
    assert np.array_equal(buf, b.get_config_packed())
    b.set_config_packed(nxt)
    b.run(1.0, 0.5, "strang")
    assert np.array_equal(a.get_config_packed(), b.get_config_packed())


def test_e2e_pipeline_every_download():
    """bench.py's end-to-end loop for several steps on an 8192^2 lattice with short windows (so that
    each step's download is still in flight when the next step's upload is staged): every step's
    downloaded lattice equals a synchronous reference -- the staged upload goes to a third plane
    buffer, never into the planes being downloaded."""
    import paper_1105_4673_b200 as kmc
    torch = _cuda()
    p = dict(ca=1, cd=1, beta=1.5, K=1.0, h=-2.0)
    a = kmc.KMC(2, (8192, 8192), (8, 8), kind="adsdes", seed=23, **p)
    b = kmc.KMC(2, (8192, 8192), (8, 8), kind="adsdes", seed=23, **p)
    ins = [_pack_words(si.bernoulli_lattice(a.local_shape, 0.2 + 0.1 * i, seed=40 + i), 8, 8, 1) for i in range(4)]
    outs = [torch.empty(int(np.prod(a.packed_shape)), dtype=torch.int64).pin_memory() for _ in range(6)]
    bufs = [o.numpy().view(np.uint64).reshape(a.packed_shape) for o in outs]
    a.stage_config_packed(ins[0])
    a.commit_config()
    for s in range(6):
        if s + 1 < 6:
            a.stage_config_packed(ins[(s + 1) % 4])
        a.run(0.02, 0.01, "lie")
        a.download_config_packed(bufs[s])
        if s + 1 < 6:
            a.commit_config()
    a.download_wait()
    for s in range(6):
        b.set_config_packed(ins[s % 4])
        b.run(0.02, 0.01, "lie")
        assert np.array_equal(bufs[s], b.get_config_packed()), s


@pytest.mark.parametrize("fused", [False, True])
def test_staged_config_on_virtual_ranks(fused):
    """The pipelined upload on the slabs of a virtual-rank group (ghost rows kept defined at the
    commit, refreshed by the next exchange; with the fused exchange the commit copies into the
    IPC-stable planes): identical to G = 1 with a synchronous upload."""
    import paper_1105_4673_b200 as kmc
    _cuda()
    p = dict(ca=1, cd=1, beta=1.5, K=1.0, h=-2.0)
    one = kmc.KMC(2, (64, 32), (8, 8), kind="adsdes", replicas=2, seed=6, **p)
    grp = kmc.VGroup(4, (64, 32), (8, 8), kind="adsdes", replicas=2, seed=6, **p)
    if fused:
        grp.set_fused(True)
    lat1 = si.bernoulli_lattice(one.local_shape, 0.5, seed=1)
    lat2 = si.bernoulli_lattice(one.local_shape, 0.3, seed=2)
    one.set_config(lat1)
    grp.set_config(lat1)
    one.run(2.0, 1.0)
    grp.run(2.0, 1.0)
    for rk in grp.ranks:
        h = rk.local_shape[1]
        rk.stage_config_packed(_pack_words(lat2[:, rk.row_offset:rk.row_offset + h], 8, 8, 1))
    for rk in grp.ranks:
        rk.commit_config()
    one.set_config(lat2)
    assert np.array_equal(grp.get_config(), lat2)
    one.run(3.0, 1.0)
    grp.run(3.0, 1.0)
    assert np.array_equal(one.get_config(), grp.get_config())
    assert one.observables()["events"] == grp.observables()["events"]


@pytest.mark.parametrize("ndim,dims,cell,kind,R,probs", [
    (1, (256,), (16,), "adsdes", 3, (0.6, 0.4)),
    (2, (32, 48), (4, 8), "zgb", 2, (0.5, 0.3, 0.2)),
    (2, (24, 40), (2, 4), "adsdes_diff", 1, (0.0, 1.0)),
])
def test_init_random_matches_oracle(ndim, dims, cell, kind, R, probs):
    """kmc_init_random (device, R32) == oracle/init.py site by site; a run from it == a run of O2
    from the same lattice."""
    from oracle.init import init_random
    gpu, orc = make_pair(ndim, dims, cell, kind, {}, 0, R)
    gpu.init_random(probs, seed=0xC0FFEE)
    H, W = (1, dims[0]) if ndim == 1 else dims
    ref = init_random(R, H, W, probs, 0xC0FFEE)
    assert np.array_equal(gpu.get_config(), ref)
    orc.set_config(ref)
    gpu.run(1.0, 0.5, "lie")
    orc.run(1.0, 0.5, "lie")
    assert_same_state(gpu, orc, "after init_random")


def test_init_random_virtual_ranks_and_errors():
    """Each virtual rank fills its own slab; together they equal G = 1 (global site ids)."""
    import paper_1105_4673_b200 as kmc
    _cuda()
    one = kmc.KMC(2, (64, 32), (8, 8), kind="adsdes", replicas=2, seed=1)
    grp = kmc.VGroup(4, (64, 32), (8, 8), kind="adsdes", replicas=2, seed=1)
    one.init_random((0.35, 0.65), seed=7)
    for rk in grp.ranks:
        rk.init_random((0.35, 0.65), seed=7)
    assert np.array_equal(one.get_config(), grp.get_config())
    with pytest.raises(kmc.KmcError):
        one.init_random((0.5, 0.3, 0.2), seed=1)           # adsdes has 2 states
    with pytest.raises(kmc.KmcError):
        one.init_random((-0.1, 1.1), seed=1)


def _half_full(shape):
    lat = np.zeros(shape, dtype=np.uint8)
    lat[:, : shape[1] // 2] = 1                 # top half full: few events; bottom half empty: many
    return lat


@pytest.mark.parametrize("ndim,dims,cell,kind,R,parts,granule", [
    (2, (128, 64), (8, 8), "adsdes", 2, 4, 2),
    (2, (64, 32), (4, 4), "zgb", 1, 3, 2),
    (1, (1024,), (16,), "adsdes", 3, 5, 1),
])
def test_workload_partition_matches_oracle(ndim, dims, cell, kind, R, parts, granule):
    """f4: strip loads since kmc_workload_mark, the cdf bounds and both imbalance figures equal
    oracle/workload.py applied to the per-cell event counts (eq.(wload), R29)."""
    from oracle import workload as wk
    gpu, _ = make_pair(ndim, dims, cell, kind, dict(ca=1, cd=1, beta=1.5, K=1.0, h=-2.0) if kind == "adsdes" else {}, 0, R)
    lat = _half_full(gpu.local_shape) if ndim == 2 else si.bernoulli_lattice(gpu.local_shape, 0.3, seed=2)
    gpu.set_config(lat)
    gpu.run(1.0, 0.5, "lie")
    gpu.workload_mark()
    c0 = gpu.observables(per_cell=True)["per_cell_events"].astype(np.int64)
    gpu.run(2.0, 0.5, "lie")
    c1 = gpu.observables(per_cell=True)["per_cell_events"].astype(np.int64)
    W = (c1 - c0).astype(np.uint64)
    loads = wk.strip_loads(W, ndim)
    res = gpu.workload_partition(parts, granule)
    assert np.array_equal(res["strip_load"], loads)
    b = wk.cdf_bounds(loads, parts, granule)
    assert np.array_equal(res["bounds"], b), (res["bounds"], b)
    assert res["imbalance"] == wk.imbalance(loads, b)
    assert res["imbalance_even"] == wk.imbalance(loads, wk.even_bounds(len(loads), parts, granule))
    if ndim == 2 and kind == "adsdes":
        assert res["imbalance"] < res["imbalance_even"]           # the half-full start is imbalanced


@pytest.mark.parametrize("world", [2, 4])
def test_rebalanced_slabs_bit_identical(world):
    """f4 -> a7: the cdf bounds used as kmc_dist.row_bounds (uneven slabs) give the bit-identical
    lattice and counters of G = 1 and of the even split (global ids); the group's strip loads and
    bounds equal the single context's."""
    import paper_1105_4673_b200 as kmc
    _cuda()
    dims, cell = (128, 32), (8, 8)
    p = dict(ca=1, cd=1, beta=1.5, K=1.0, h=-2.0)
    one = kmc.KMC(2, dims, cell, kind="adsdes", seed=41, replicas=2, **p)
    even = kmc.VGroup(world, dims, cell, kind="adsdes", seed=41, replicas=2, **p)
    lat = _half_full(one.local_shape)
    one.set_config(lat)
    even.set_config(lat)
    one.run(1.0, 0.5, "lie")
    even.run(1.0, 0.5, "lie")
    r1 = one.workload_partition(world, 2)
    rg = even.workload_partition(world, 2)
    assert np.array_equal(r1["bounds"], rg["bounds"]) and np.array_equal(r1["strip_load"], rg["strip_load"])
    b = r1["bounds"]
    assert len(set(np.diff(b))) > 1                                # really uneven
    reb = kmc.VGroup(world, dims, cell, kind="adsdes", seed=41, replicas=2, row_bounds=b, **p)
    assert [rk.local_shape[1] // cell[0] for rk in reb.ranks] == list(np.diff(b))
    reb.set_config(one.get_config())
    for r in reb.ranks:
        r.set_state(*one.get_state())
    for _ in range(2):
        one.run(1.0, 0.5, "lie")
        reb.run(1.0, 0.5, "lie")
        even.run(1.0, 0.5, "lie")
        assert np.array_equal(one.get_config(), reb.get_config())
        assert np.array_equal(one.get_config(), even.get_config())


def test_workload_partition_errors():
    import paper_1105_4673_b200 as kmc
    _cuda()
    g = kmc.KMC(2, (48, 64), (8, 8), kind="adsdes", seed=1)     # 6 strips
    for parts, gr in [(0, 1), (4, 2), (2, 4), (7, 1)]:
        with pytest.raises(kmc.KmcError) as e:
            g.workload_partition(parts, gr)
        assert e.value.status == 1
    r = g.workload_partition(3, 2)                                  # no events yet: the even split
    assert list(r["bounds"]) == [0, 2, 4, 6] and r["imbalance"] == 1.0
    with pytest.raises(kmc.KmcError) as e:
        kmc.VGroup(2, (48, 64), (8, 8), kind="adsdes", row_bounds=[0, 3, 6])
    assert e.value.status == 2


@pytest.mark.parametrize("kind,params,cell,scheme,dt", [
    ("adsdes", dict(ca=1, cd=1, beta=1.5, K=1.0, h=-2.0), (8, 8), "lie", 1.0),
    ("adsdes_diff", dict(ca=0.5, cd=0.5, beta=1.0, K=1.0, h=-2.0, c_hop=2.0), (4, 4), "strang", 0.5),
    ("zgb", dict(k1=0.45, k2=1.0), (2, 4), "random", 0.5),
    ("zgb_diff", dict(k1=0.4, k2=1.0, c_hop=0.8), (4, 2), "lie", 0.25),
    ("zgb_odiff", dict(k1=0.4, k2=1.0, c_hop=1.5), (4, 4), "strang", 0.25),
])
@pytest.mark.parametrize("world", [2, 4])
def test_fused_exchange_bit_identical(kind, params, cell, scheme, dt, world):
    """SURVEY §8(e) fused exchange: window kernels that mirror their boundary-row writes and ghost-row
    XOR deltas straight into the neighbour slabs (no exchange between windows) give the lattice,
    event counts and observables of G = 1, also across a configuration upload mid-run and with
    uneven slabs."""
    import paper_1105_4673_b200 as kmc
    _cuda()
    dims = (64, 32)
    qy = cell[0]
    rows = dims[0] // qy
    bounds = None
    if world == 2:                                   # uneven slabs as well
        bounds = [0, 2 * (rows // 8), rows]
    one = kmc.KMC(2, dims, cell, kind=kind, seed=37, replicas=2, **params)
    grp = kmc.VGroup(world, dims, cell, kind=kind, seed=37, replicas=2, row_bounds=bounds, **params)
    grp.set_fused(True)
    lat = (si.bernoulli_lattice(one.local_shape, 0.5, seed=5) if not kind.startswith("zgb")
           else si.categorical_lattice(one.local_shape, [0.5, 0.25, 0.25], seed=5))
    one.set_config(lat)
    grp.set_config(lat)
    for i in range(3):
        one.run(2 * dt, dt, scheme)
        grp.run(2 * dt, dt, scheme)
        assert np.array_equal(one.get_config(), grp.get_config()), i
        if i == 1:                                   # upload mid-run: planes must stay in place
            lat2 = one.get_config()
            one.set_config(lat2)
            grp.set_config(lat2)
    if (dims[0] // qy) % 4 == 0 and all(rk.local_shape[1] // qy % 2 == 0 for rk in grp.ranks):
        one.run_nested(1.0, 0.5, 2, "lie", "lie", 2)   # nested runs keep the exchange path
        grp.run_nested(1.0, 0.5, 2, "lie", "lie", 2)
        assert np.array_equal(one.get_config(), grp.get_config())
        one.run(2 * dt, dt, scheme)                  # and fused windows resume after them
        grp.run(2 * dt, dt, scheme)
        assert np.array_equal(one.get_config(), grp.get_config())
    a, b = one.observables(), grp.observables()
    assert a["events"] == b["events"] > 0
    for key in ("n_state", "nn_pairs", "n_state_by_colour"):
        assert np.array_equal(a[key], b[key]), key


def test_maximum_size_lattice():
    """A 65536^2 lattice (4.3e9 sites, 2^26 cells: 32-bit word and cell ids near their range) runs a
    Lie macro-step: the observables count every site, events happen, two contexts with the same seed
    and configuration give identical lattices (no index overflow, no races), and a replica offset
    beyond 2^31 cells is refused (kmc_create keeps every id below 2^32)."""
    torch = _cuda()
    import paper_1105_4673_b200 as kmc
    n = 65536
    p = dict(ca=1, cd=1, beta=1.5, K=1.0, h=-2.0)
    outs = []
    for _ in range(2):
        g = kmc.KMC(2, (n, n), (8, 8), kind="adsdes", seed=5, **p)
        g.init_random((0.5, 0.5), seed=9)
        g.run(1.0, 1.0, "lie")
        o = g.observables()
        assert int(o["n_state"][0] + o["n_state"][1]) == n * n
        assert o["events"] > 1.0 * n * n
        w = torch.from_numpy(g.get_config_packed().view(np.int64)).cuda()
        outs.append((int(w.sum().item()), int((w * 3 + 1).sum().item()), int(w[::7].sum().item())))
        del g, w
        torch.cuda.empty_cache()
    assert outs[0] == outs[1]
    with pytest.raises(kmc.KmcError):
        kmc.KMC(2, (n, n), (8, 8), kind="adsdes", replicas=65, seed=5, **p)   # 65 x 2^26 cells > 2^32


@pytest.mark.parametrize("kind,ndim,dims,cell,loopback", [
    ("adsdes", 2, (64, 64), (8, 8), False),
    ("zgb", 2, (32, 64), (4, 8), False),
    ("adsdes_diff", 2, (64, 32), (4, 4), True),       # ghost rows: the NCCL loopback ring
    ("adsdes", 1, (1024,), (32,), False),
])
def test_borrowed_planes(kind, ndim, dims, cell, loopback):
    """kmc_attach_planes (§8(b) borrowed device buffer): the windows run on a caller-owned torch
    tensor that always holds the current packed lattice (owned rows = get_config_packed, ghost rows
    around them); configuration uploads copy into it; results are bit-identical to a context on its
    own planes; the tensor outlives the context."""
    torch = _cuda()
    import paper_1105_4673_b200 as kmc
    params = {"adsdes": dict(ca=1, cd=1, beta=1.5, K=1.0, h=-2.0), "zgb": dict(k1=0.4, k2=1.0),
              "adsdes_diff": dict(ca=1, cd=1, beta=1.0, K=1.0, h=-2.0, c_hop=1.0)}[kind]
    extra = dict(nccl_id=kmc.nccl_unique_id()) if loopback else {}
    a = kmc.KMC(ndim, dims, cell, kind=kind, replicas=2, seed=21, **params)
    b = kmc.KMC(ndim, dims, cell, kind=kind, replicas=2, seed=21, **params, **extra)
    init = (lambda s: si.categorical_lattice(a.local_shape, [0.5, 0.25, 0.25], seed=s)) if kind == "zgb" else \
           (lambda s: si.bernoulli_lattice(a.local_shape, 0.5, seed=s))
    lat = init(3)
    a.set_config(lat)
    b.set_config(lat)
    lay = b.planes_layout()
    assert lay["ghost"] == (1 if loopback else 0)
    buf = torch.full((lay["planes"] * lay["words_per_plane"],), -1, dtype=torch.int64, device="cuda")
    with pytest.raises(kmc.KmcError):
        b.attach_planes(buf.data_ptr(), buf.numel() - 1)
    b.attach_planes(buf.data_ptr(), buf.numel())

    def owned_rows():
        torch.cuda.synchronize()
        v = buf.cpu().numpy().view(np.uint64).reshape(lay["planes"], lay["storage_rows"], -1)
        gh = lay["ghost"]
        return v[:, gh:lay["storage_rows"] - gh].reshape(b.packed_shape)

    assert np.array_equal(owned_rows(), b.get_config_packed())
    for i in range(3):
        a.run(1.0, 0.5, "strang")
        b.run(1.0, 0.5, "strang")
        assert np.array_equal(a.get_config(), b.get_config()), i
        assert np.array_equal(owned_rows(), b.get_config_packed()), i
        assert a.observables()["events"] == b.observables()["events"]
    lat2 = init(4)                                      # an upload lands in the borrowed buffer
    a.set_config(lat2)
    b.set_config(lat2)
    assert np.array_equal(owned_rows(), a.get_config_packed())
    a.run(1.0, 0.5, "lie")
    b.run(1.0, 0.5, "lie")
    assert np.array_equal(a.get_config(), b.get_config())
    last = b.get_config_packed()
    b.close()
    assert np.array_equal(owned_rows(), last)           # the caller's tensor outlives the context
