"""Pins of the oracle's a8 observables (FSKMC.observables, oracle/fskmc.py) on hand-built lattices
(CPU, -m "not gpu").

The paper's observables: mean coverage c_t = |Lambda|^-1 sum_x sigma_t(x) and the Ising
Hamiltonian H = -(K/2) sum_x sum_{|y-x|=1} sigma(x) sigma(y) + h sum_x sigma(x), whose
double sum runs over ORDERED neighbour pairs (every bond twice).  Every expected number below was
counted by hand from the printed lattice (the working is in the comments) -- nothing is recomputed
with the oracle's own numpy expressions.  The energy is also evaluated by a literal double loop over
x and its 2d neighbours, so a dropped factor 1/2, a missed periodic wrap or a sign error in R24's
E = -K nn[1][1] + h n[1] fails here.
"""
import numpy as np
import pytest

from oracle.fskmc import FSKMC, model_params

# 2-state 4x4 torus, rows y = 0..3 (x to the right)
LAT2 = np.array([[1, 1, 0, 0],
                 [1, 0, 0, 1],
                 [0, 0, 0, 0],
                 [1, 0, 0, 1]], dtype=np.uint8)
# 3-state (ZGB storage: 0 vacant, 1 CO, 2 O) 4x4 torus
LAT3 = np.array([[1, 2, 0, 0],
                 [0, 2, 2, 1],
                 [1, 0, 0, 0],
                 [0, 0, 1, 2]], dtype=np.uint8)


def _oracle(ndim, dims, cell, kind, lat, colours=0, replicas=1, K=0.0, h=0.0):
    o = FSKMC(ndim, dims, cell, kind, model_params(K=K, h=h), colours=colours, replicas=replicas)
    o.set_config(lat)
    return o.observables()


def _energy_double_loop(lat2d, K, h):
    """P:959-961 written out: -(K/2) sum_x sum_{|y-x|=1} sigma(x) sigma(y) + h sum_x sigma(x), periodic."""
    H, W = lat2d.shape
    pair = 0
    for y in range(H):
        for x in range(W):
            for dy, dx in ((0, -1), (0, 1), (-1, 0), (1, 0)):
                pair += int(lat2d[y, x] == 1) * int(lat2d[(y + dy) % H, (x + dx) % W] == 1)
    return -(K / 2.0) * pair + h * int((lat2d == 1).sum())


def test_observables_2state_torus_hand_counted():
    # occupied: row 0 two, row 1 two, row 2 none, row 3 two -> 6 of 16
    # horizontal bonds (with the x = 3 -> 0 wrap): row0 11,01,00,01  row1 01,00,01,11  row2 00 x4
    #   row3 01,00,01,11  -> 11: 3, 01: 6, 00: 7
    # vertical bonds (with the y = 3 -> 0 wrap): col0 (1,1,0,1) 11,01,01,11  col1 (1,0,0,0) 01,00,00,01
    #   col2 00 x4  col3 (0,1,0,1) 01 x4  -> 11: 2, 01: 8, 00: 6
    K, h = 1.3, -0.7
    obs = _oracle(2, (4, 4), (2, 2), "adsdes", LAT2[None], K=K, h=h)
    assert list(obs["n_state"][:2]) == [10, 6]
    nn = obs["nn_pairs"]
    assert nn[1, 1] == 5 and nn[0, 1] == 14 and nn[1, 0] == 14 and nn[0, 0] == 13
    assert nn[:2, :2].sum() - nn[0, 1] == 32                 # 32 bonds on a 4x4 torus (2 per site)
    assert np.allclose(obs["coverage"][:2], [10 / 16, 6 / 16])
    # H = -(K/2) * (2 * 5 ordered 1-1 pairs) + h * 6 = -5K + 6h
    assert obs["energy"] == pytest.approx(-5 * K + 6 * h, rel=0, abs=1e-12)
    assert obs["energy"] == pytest.approx(_energy_double_loop(LAT2, K, h), rel=0, abs=1e-12)


def test_observables_2state_colours_hand_counted():
    # 2x2 cells: cell (cy0,cx0) sites 1,1,1,0 -> 3 occupied; (cy0,cx1) 0,0,0,1 -> 1;
    # (cy1,cx0) 0,0,1,0 -> 1; (cy1,cx1) 0,0,0,1 -> 1
    two = _oracle(2, (4, 4), (2, 2), "adsdes", LAT2[None], colours=2)
    # checkerboard colour (cx+cy)&1: colour 0 = cells (0,0),(1,1): 4 occupied of 8; colour 1: 2 of 8
    assert two["n_state_by_colour"][0, :2].tolist() == [4, 4]
    assert two["n_state_by_colour"][1, :2].tolist() == [6, 2]
    four = _oracle(2, (4, 4), (2, 2), "adsdes", LAT2[None], colours=4)
    # colour (cx&1) + 2(cy&1): one cell each
    assert four["n_state_by_colour"][:4, :2].tolist() == [[1, 3], [3, 1], [3, 1], [3, 1]]


def test_observables_3state_torus_hand_counted():
    # CO: one per row -> 4; O: row0 1, row1 2, row3 1 -> 4; vacant 8
    # horizontal: row0 (1,2,0,0) 12,02,00,01  row1 (0,2,2,1) 02,22,12,01  row2 (1,0,0,0) 01,00,00,01
    #   row3 (0,0,1,2) 00,01,12,02  -> 00:4 01:5 02:3 11:0 12:3 22:1
    # vertical: col0 (1,0,1,0) 01 x4  col1 (2,2,0,0) 22,02,00,02  col2 (0,2,0,1) 02,02,01,01
    #   col3 (0,1,0,2) 01,01,02,02  -> 00:1 01:8 02:6 11:0 12:0 22:1
    obs = _oracle(2, (4, 4), (2, 2), "zgb", LAT3[None])
    assert list(obs["n_state"][:3]) == [8, 4, 4]
    nn = obs["nn_pairs"]
    want = {(0, 0): 5, (0, 1): 13, (0, 2): 9, (1, 1): 0, (1, 2): 3, (2, 2): 2}
    for (a, b), v in want.items():
        assert nn[a, b] == v and nn[b, a] == v, (a, b)
    # per-species degree sums: 4 bonds per site
    assert 2 * nn[1, 1] + nn[0, 1] + nn[1, 2] == 4 * 4
    assert 2 * nn[2, 2] + nn[0, 2] + nn[1, 2] == 4 * 4
    # 4 colours, one 2x2 cell each: (0,0) 1,2,0,2; (0,1) 0,0,2,1; (1,0) 1,0,0,0; (1,1) 0,0,1,2
    assert obs["n_state_by_colour"][:4, :3].tolist() == [[1, 1, 2], [2, 1, 1], [3, 1, 0], [2, 1, 1]]


def test_observables_1d_ring_and_replicas_hand_counted():
    # replica 0: 1 1 0 1 0 0 -> bonds 11, 10, 01, 10, 00, 01 (wrap x = 5 -> 0): 11:1 01:4 00:1
    # replica 1: all occupied -> 6 bonds 11; no bond joins the two replicas
    lat = np.array([[[1, 1, 0, 1, 0, 0]], [[1, 1, 1, 1, 1, 1]]], dtype=np.uint8)
    K, h = 0.8, 0.25
    obs = _oracle(1, (6,), (3,), "adsdes", lat, replicas=2, K=K, h=h)
    assert list(obs["n_state"][:2]) == [3, 9]
    nn = obs["nn_pairs"]
    assert nn[1, 1] == 7 and nn[0, 1] == 4 and nn[0, 0] == 1
    # cells of 3 sites: colour = cx & 1; replica 0 cells (1,1,0) (1,0,0), replica 1 (1,1,1) (1,1,1)
    assert obs["n_state_by_colour"][:2, :2].tolist() == [[1, 5], [2, 4]]
    # H per replica: -(K/2)(2 n11) + h n1 summed: replica 0 -K + 3h, replica 1 -6K + 6h
    assert obs["energy"] == pytest.approx(-7 * K + 9 * h, rel=0, abs=1e-12)


def test_energy_double_loop_matches_on_random_lattices():
    rng = np.random.default_rng(5)
    for _ in range(5):
        lat = (rng.random((8, 8)) < 0.45).astype(np.uint8)
        obs = _oracle(2, (8, 8), (2, 2), "adsdes", lat[None], K=0.9, h=0.4)
        assert obs["energy"] == pytest.approx(_energy_double_loop(lat, 0.9, 0.4), rel=0, abs=1e-9)
