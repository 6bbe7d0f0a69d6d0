"""The multi-GPU data plane executed on hardware.

* NCCL loopback (one GPU): a world = 1 context given an NCCL unique id runs its 2D lattice as a
  one-rank periodic ring through the real transport of the NCCL path -- ghost rows, ncclCommInitRank,
  the grouped ncclSend/ncclRecv forward exchange with itself (rank_up == rank_down, the world = 2
  ordering), the ghost snapshot and the reverse XOR-delta exchange for pair models -- and, with
  fused_exchange = 1, the peer-write (PEER) window kernel plus the device-flag wait/signal kernels
  on its own planes.  Every macro-step must be bit-identical to a plain world = 1 context, which is
  itself bit-exact to the O2 oracle (tests/test_gpu_parity.py); the oracle is checked here too.
* Two processes, two GPUs (skipped when fewer than 2 devices): kmc_run at world = 2 over NCCL and
  over the CUDA-IPC fused exchange, gathered lattice and per-cell counters vs O2 after every
  macro-step.
"""
import os
import tempfile

import numpy as np
import pytest

import synth_inputs as si
from oracle.fskmc import FSKMC, model_params

pytestmark = pytest.mark.gpu

MODELS = {
    "adsdes": (dict(ca=1, cd=1, beta=1.5, K=1.0, h=-2.0), (8, 8), "lie", 1.0),
    "adsdes_diff": (dict(ca=0.5, cd=0.5, beta=1.0, K=1.0, h=-2.0, c_hop=2.0), (4, 4), "strang", 0.5),
    "zgb": (dict(k1=0.45, k2=1.0), (2, 4), "random", 0.5),
    "zgb_diff": (dict(k1=0.4, k2=1.0, c_hop=0.8), (4, 2), "lie", 0.25),
    "zgb_odiff": (dict(k1=0.4, k2=1.0, c_hop=1.5), (4, 4), "strang", 0.25),
}


def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _init(kind, shape, seed):
    return (si.bernoulli_lattice(shape, 0.5, seed=seed) if not kind.startswith("zgb")
            else si.categorical_lattice(shape, [0.5, 0.25, 0.25], seed=seed))


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("kind", list(MODELS))
def test_nccl_loopback_bit_identical(kind, fused):
    import paper_1105_4673_b200 as kmc
    _cuda()
    params, cell, scheme, dt = MODELS[kind]
    dims = (64, 32)
    one = kmc.KMC(2, dims, cell, kind=kind, seed=41, replicas=2, **params)
    ring = kmc.KMC(2, dims, cell, kind=kind, seed=41, replicas=2, nccl_id=kmc.nccl_unique_id(),
                   fused_exchange=fused, **params)
    orc = FSKMC(2, dims, cell, kind, model_params(**params), replicas=2, seed=41)
    lat = _init(kind, one.local_shape, 6)
    for x in (one, ring, orc):
        x.set_config(lat)
    for i in range(3):
        one.run(dt, dt, scheme)
        ring.run(dt, dt, scheme)
        orc.run(dt, dt, scheme)
        a, b = one.get_config(), ring.get_config()
        assert np.array_equal(a, b), i
        assert np.array_equal(a, orc.get_config()), i
        oa, ob = one.observables(per_cell=True), ring.observables(per_cell=True)
        assert np.array_equal(oa["per_cell_events"], ob["per_cell_events"]), i
        assert oa["events"] == ob["events"] == orc.events > 0
        for key in ("n_state", "nn_pairs", "n_state_by_colour"):
            assert np.array_equal(oa[key], ob[key]), key
        if i == 1:                                   # upload mid-run (fused: planes stay mapped)
            lat2 = one.get_config()
            one.set_config(lat2)
            ring.set_config(lat2)
    # nested runs exchange once per outer factor (f3) through the same transport
    one.run_nested(1.0, 0.5, 2, "lie", "lie", 2)
    ring.run_nested(1.0, 0.5, 2, "lie", "lie", 2)
    assert np.array_equal(one.get_config(), ring.get_config())
    # correlation counts across the ghost rows (rmax <= q_y on a ring)
    ca, cb = one.correlation(cell[0]), ring.correlation(cell[0])
    assert np.array_equal(ca["x"], cb["x"]) and np.array_equal(ca["y"], cb["y"])
    assert ring.device_errors() == {"bad_spins": False, "wait_timeouts": False}


def test_nccl_loopback_coverage_series_and_timing():
    """The coverage process and kernel timing on the loopback ring match world = 1."""
    import paper_1105_4673_b200 as kmc
    _cuda()
    params, cell, scheme, dt = MODELS["adsdes"]
    one = kmc.KMC(2, (64, 64), cell, kind="adsdes", seed=3, **params)
    ring = kmc.KMC(2, (64, 64), cell, kind="adsdes", seed=3, nccl_id=kmc.nccl_unique_id(), **params)
    lat = _init("adsdes", one.local_shape, 9)
    for x in (one, ring):
        x.set_config(lat)
        x.record_coverage(8)
        x.run(4.0, 1.0, "strang")
    assert np.array_equal(one.coverage_series(), ring.coverage_series())
    a, b = one.coverage_stats(2), ring.coverage_stats(2)
    assert a["mean"] == b["mean"] and np.allclose(a["acf"], b["acf"], rtol=0, atol=1e-12)


def _worker(rank, world, uid, kind, fused, lat, nmacro, outdir):
    import torch
    import paper_1105_4673_b200 as kmc
    torch.cuda.set_device(rank)
    params, cell, scheme, dt = MODELS[kind]
    k = kmc.KMC(2, (64, 32), cell, kind=kind, seed=41, replicas=2, rank=rank, world=world, device=rank,
                nccl_id=uid, fused_exchange=fused, **params)
    h = k.local_shape[1]
    k.set_config(lat[:, k.row_offset:k.row_offset + h])
    for i in range(nmacro):
        k.run(dt, dt, scheme)
        obs = k.observables(per_cell=True)
        np.save(os.path.join(outdir, f"r{rank}_m{i}_lat.npy"), k.get_config())
        np.save(os.path.join(outdir, f"r{rank}_m{i}_cells.npy"), obs["per_cell_events"])
        np.save(os.path.join(outdir, f"r{rank}_m{i}_events.npy"), np.array([obs["events"]]))
    k.close()


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("kind", ["adsdes", "adsdes_diff", "zgb"])
def test_two_process_nccl_world2(kind, fused):
    torch = _cuda()
    if torch.cuda.device_count() < 2:
        pytest.skip(f"needs 2 GPUs (this box has {torch.cuda.device_count()}); the one-GPU loopback "
                    "test covers the same transport")
    import torch.multiprocessing as mp
    import paper_1105_4673_b200 as kmc
    params, cell, scheme, dt = MODELS[kind]
    orc = FSKMC(2, (64, 32), cell, kind, model_params(**params), replicas=2, seed=41)
    lat = _init(kind, (2, 64, 32), 6)
    orc.set_config(lat)
    nmacro = 3
    with tempfile.TemporaryDirectory() as d:
        uid = kmc.nccl_unique_id()
        mp.start_processes(_worker, args=(2, uid, kind, fused, lat, nmacro, d), nprocs=2, join=True,
                           start_method="spawn")
        for i in range(nmacro):
            orc.run(dt, dt, scheme)
            got = np.concatenate([np.load(os.path.join(d, f"r{r}_m{i}_lat.npy")) for r in range(2)], axis=1)
            assert np.array_equal(got, orc.get_config()), i
            cells = np.concatenate([np.load(os.path.join(d, f"r{r}_m{i}_cells.npy")) for r in range(2)], axis=1)
            assert np.array_equal(cells.reshape(-1), orc.W_events), i
            for r in range(2):       # observables are all-reduced: every rank sees the global total
                assert int(np.load(os.path.join(d, f"r{r}_m{i}_events.npy"))[0]) == orc.events
