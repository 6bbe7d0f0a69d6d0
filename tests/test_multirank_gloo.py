"""Multi-rank host logic on CPU (gloo, world size 2 and 4): the slab partition plan of the C
library (kmc_partition_plan) and the halo-exchange protocol of kmc_capi.cu (forward ghost-row
exchange before each window in the library's message order; reverse XOR-delta exchange after
windows of cross-cell-writing models), driven with the O2 oracle as the per-cell compute.  The
gathered result must be bit-identical to the single-process O2 run (global ids).

The CUDA kernels need a GPU; this test checks the decomposition and the exchange order/merge
rules that the NCCL path in the library implements (same order, same XOR merge)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth_inputs as si

CASES = {
    "ising_lie": (2, (32, 16), (4, 4), "adsdes", dict(ca=1, cd=1, beta=1.5, K=1.0, h=-2.0), "lie", 1.0, 2),
    "diff_strang": (2, (32, 16), (4, 4), "adsdes_diff", dict(ca=0.5, cd=0.5, beta=1.0, K=1.0, h=-2.0, c_hop=2.0), "strang", 0.5, 2),
    "zgb_random": (2, (32, 16), (2, 4), "zgb", dict(k1=0.45, k2=1.0), "random", 0.5, 2),
}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _xchg(ops):
    reqs = [op() for op in ops]
    for r in reqs:
        r.wait()


def _worker(rank, world, port, case, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1105_4673_b200 as kmc
        from oracle.fskmc import FSKMC, model_params, substeps, SCHEME
        ndim, dims, cell, kind, params, scheme, dt, nmacro = CASES[case]
        H, W = dims
        qy, qx = cell
        plan = kmc.partition_plan(ndim, dims, cell, 1, kind, world, rank)
        r0, nr = plan["row_offset"], plan["rows_local"]           # in cell rows
        up, down = plan["rank_up"], plan["rank_down"]
        My = H // qy
        full = (si.bernoulli_lattice((1, H, W), 0.5, seed=21) if kind != "zgb"
                else si.categorical_lattice((1, H, W), [0.5, 0.25, 0.25], seed=21))
        orc = FSKMC(ndim, dims, cell, kind, model_params(**params), seed=77)
        lat = np.zeros_like(full)
        own = slice(r0 * qy, (r0 + nr) * qy)
        lat[:, own] = full[:, own]
        orc.lat = lat
        cross = kind != "adsdes"

        def rows(cr):                                            # site rows of cell row cr (periodic)
            cr %= My
            return slice(cr * qy, (cr + 1) * qy)

        first, last = rows(r0), rows(r0 + nr - 1)
        gtop, gbot = rows(r0 - 1), rows(r0 + nr)
        C = orc.C
        window = 0
        for _ in range(nmacro):
            for colour, D in substeps(SCHEME[scheme], C, dt, orc.seed, window):
                # forward: same message order as exchange_forward() in kmc_capi.cu
                s_last = torch.from_numpy(np.ascontiguousarray(orc.lat[0, last]))
                s_first = torch.from_numpy(np.ascontiguousarray(orc.lat[0, first]))
                r_top = torch.empty_like(s_first)
                r_bot = torch.empty_like(s_first)
                _xchg([lambda: dist.isend(s_last, down), lambda: dist.isend(s_first, up),
                       lambda: dist.irecv(r_top, up), lambda: dist.irecv(r_bot, down)])
                orc.lat[0, gtop] = r_top.numpy()
                orc.lat[0, gbot] = r_bot.numpy()
                snap_top, snap_bot = orc.lat[0, gtop].copy(), orc.lat[0, gbot].copy()
                # the window on my owned cells of this colour (global coordinates -> global ids)
                cells = []
                for cy in range(r0, r0 + nr):
                    for cx in range(W // qx):
                        col = ((cx + cy) & 1) if C == 2 else ((cx & 1) + 2 * (cy & 1))
                        if col == colour:
                            cells.append((0, cy, cx))
                orc.window_cells(np.array(cells), D, window)
                window += 1
                if cross:   # reverse: ghost deltas back to their owners, XOR merge (exchange_reverse)
                    d_top = torch.from_numpy(np.ascontiguousarray(orc.lat[0, gtop] ^ snap_top))
                    d_bot = torch.from_numpy(np.ascontiguousarray(orc.lat[0, gbot] ^ snap_bot))
                    r_last = torch.empty_like(d_top)
                    r_first = torch.empty_like(d_top)
                    _xchg([lambda: dist.isend(d_top, up), lambda: dist.isend(d_bot, down),
                           lambda: dist.irecv(r_last, down), lambda: dist.irecv(r_first, up)])
                    orc.lat[0, last] ^= r_last.numpy()
                    orc.lat[0, first] ^= r_first.numpy()
        mine = torch.from_numpy(np.ascontiguousarray(orc.lat[0, own]))
        gathered = [torch.empty_like(mine) for _ in range(world)] if rank == 0 else None
        dist.gather(mine, gathered, dst=0)
        if rank == 0:
            out_q.put(np.concatenate([g.numpy() for g in gathered], axis=0))
    finally:
        dist.destroy_process_group()


def _single(case):
    from oracle.fskmc import FSKMC, model_params
    ndim, dims, cell, kind, params, scheme, dt, nmacro = CASES[case]
    H, W = dims
    full = (si.bernoulli_lattice((1, H, W), 0.5, seed=21) if kind != "zgb"
            else si.categorical_lattice((1, H, W), [0.5, 0.25, 0.25], seed=21))
    o = FSKMC(ndim, dims, cell, kind, model_params(**params), seed=77)
    o.set_config(full)
    o.run(nmacro * dt, dt, scheme)
    return o.get_config()[0], o.events


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("case", list(CASES))
def test_slab_decomposition_bit_identical(case, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref, events = _single(case)
    assert events > 0
    assert np.array_equal(got, ref), (case, world, int((got != ref).sum()))


# ---- f3 + f4 host logic: nested schedule (one exchange per outer factor) on UNEVEN slabs (row
# bounds as kmc_dist.row_bounds), and the all-reduced strip loads -> identical cdf bounds ----
NESTED = {
    # kind, params, outer, inner, n_inner, block, bounds per world
    "ising_nested": ("adsdes", dict(ca=1, cd=1, beta=1.5, K=1.0, h=-2.0), "lie", "strang", 2, 2,
                     {2: [0, 6, 16], 4: [0, 2, 6, 12, 16]}),
    "zgb_nested": ("zgb", dict(k1=0.45, k2=1.0), "strang", "lie", 2, 2, {2: [0, 10, 16], 4: [0, 4, 6, 10, 16]}),
}
NDIMS, NCELL = (64, 16), (4, 4)


def _nested_worker(rank, world, port, case, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.fskmc import FSKMC, model_params, nested_substeps, SCHEME
        from oracle import workload as wk
        kind, params, outer, inner, n_inner, block, bnd = NESTED[case]
        (H, W), (qy, qx) = NDIMS, NCELL
        b = bnd[world]
        r0, nr = b[rank], b[rank + 1] - b[rank]
        up, down = (rank + world - 1) % world, (rank + 1) % world
        My, Mx = H // qy, W // qx
        full = (si.bernoulli_lattice((1, H, W), 0.5, seed=23) if kind != "zgb"
                else si.categorical_lattice((1, H, W), [0.5, 0.25, 0.25], seed=23))
        orc = FSKMC(2, NDIMS, NCELL, kind, model_params(**params), seed=79)
        lat = np.zeros_like(full)
        own = slice(r0 * qy, (r0 + nr) * qy)
        lat[:, own] = full[:, own]
        orc.lat = lat
        cross = kind != "adsdes"

        def rows(cr):
            cr %= My
            return slice(cr * qy, (cr + 1) * qy)

        first, last, gtop, gbot = rows(r0), rows(r0 + nr - 1), rows(r0 - 1), rows(r0 + nr)
        C = orc.C
        window, nexch = 0, 0
        loads = np.zeros(My, dtype=np.int64)
        for _ in range(2):                                           # 2 macro-steps of dt = 0.5
            sched = nested_substeps(SCHEME[outer], SCHEME[inner], C, 0.5, n_inner, orc.seed, window)
            k = 0
            while k < len(sched):
                o = sched[k][0]
                # forward exchange once per outer factor (kmc_run_nested)
                s_last = torch.from_numpy(np.ascontiguousarray(orc.lat[0, last]))
                s_first = torch.from_numpy(np.ascontiguousarray(orc.lat[0, first]))
                r_top, r_bot = torch.empty_like(s_first), torch.empty_like(s_first)
                _xchg([lambda: dist.isend(s_last, down), lambda: dist.isend(s_first, up),
                       lambda: dist.irecv(r_top, up), lambda: dist.irecv(r_bot, down)])
                nexch += 1
                orc.lat[0, gtop] = r_top.numpy()
                orc.lat[0, gbot] = r_bot.numpy()
                snap_top, snap_bot = orc.lat[0, gtop].copy(), orc.lat[0, gbot].copy()
                while k < len(sched) and sched[k][0] == o:
                    _, colour, D = sched[k]
                    cells = [(0, cy, cx) for cy in range(r0, r0 + nr) for cx in range(Mx)
                             if (cy // block) % 2 == o
                             and (((cx + cy) & 1) if C == 2 else ((cx & 1) + 2 * (cy & 1))) == colour]
                    if cells:
                        ev = orc.window_cells(np.array(cells), D, window)
                        for (_, cy, _), e in zip(cells, ev):
                            loads[cy] += int(e)
                    window += 1
                    k += 1
                if cross:
                    d_top = torch.from_numpy(np.ascontiguousarray(orc.lat[0, gtop] ^ snap_top))
                    d_bot = torch.from_numpy(np.ascontiguousarray(orc.lat[0, gbot] ^ snap_bot))
                    r_last, r_first = torch.empty_like(d_top), torch.empty_like(d_top)
                    _xchg([lambda: dist.isend(d_top, up), lambda: dist.isend(d_bot, down),
                           lambda: dist.irecv(r_last, down), lambda: dist.irecv(r_first, up)])
                    orc.lat[0, last] ^= r_last.numpy()
                    orc.lat[0, first] ^= r_first.numpy()
        tl = torch.from_numpy(loads)
        dist.all_reduce(tl)                                          # f4: global strip loads
        bounds = wk.cdf_bounds(tl.numpy().astype(np.uint64), world, 2)
        slabs = [None] * world                                       # uneven slabs: gather as objects
        dist.all_gather_object(slabs, np.ascontiguousarray(orc.lat[0, own]))
        allb = [None] * world
        dist.all_gather_object(allb, [int(x) for x in bounds])
        if rank == 0:
            out_q.put((np.concatenate(slabs, axis=0), allb, nexch, tl.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("case", list(NESTED))
def test_nested_uneven_slabs_and_workload_bounds(case, world):
    """f3 on uneven slabs: one forward (+ reverse) exchange per outer factor reproduces the
    single-process nested O2 run bit for bit; f4: the all-reduced strip loads give every rank the
    bounds the single-process counters give."""
    from oracle.fskmc import FSKMC, model_params
    from oracle import workload as wk
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_nested_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, allb, nexch, loads = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    kind, params, outer, inner, n_inner, block, _ = NESTED[case]
    (H, W), (qy, qx) = NDIMS, NCELL
    full = (si.bernoulli_lattice((1, H, W), 0.5, seed=23) if kind != "zgb"
            else si.categorical_lattice((1, H, W), [0.5, 0.25, 0.25], seed=23))
    o = FSKMC(2, NDIMS, NCELL, kind, model_params(**params), seed=79)
    o.set_config(full)
    o.run_nested(1.0, 0.5, n_inner, outer, inner, block)
    assert np.array_equal(got, o.get_config()[0])
    assert nexch == 2 * (2 if outer == "lie" else 3)                 # one per outer factor
    ref_loads = wk.strip_loads(o.W_events.reshape(1, H // qy, W // qx), 2)
    assert np.array_equal(loads.astype(np.uint64), ref_loads)
    ref_b = list(wk.cdf_bounds(ref_loads, world, 2))
    assert all(list(b) == ref_b for b in allb)
