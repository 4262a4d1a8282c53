"""Multi-rank host logic on CPU (gloo, world_size 2 and 3).

The CUDA/NCCL slab path cannot run here (no GPU) and must not be emulated with ranks
sharing one GPU (B200_PROFILING.md).  These tests drive the SAME host-side plans the
library uses -- sf_slab_plan (partition), sf_slab_halo_plan (which planes go where
every step), sf_sparse_owner (who writes a record row) -- through a rank-local fp64
slab emulation with real gloo send/recv, and require the assembled result to equal
the single-domain oracle: any error in the partition, the halo plan, the injection
ownership (corners by owning plane) or the record ownership (base plane) fails them.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    p = synth.random_problem(3, (23, 13, 11), 4, 40, seed=3, nbl=3, nsrc=2, nrec=9, random_wavelet=True)
    h = p.h
    # sources / receivers on and across slab boundaries (x = 7.5 h, 11.5 h, 15.5 h ...)
    p.src_coords = np.array([[11.5 * h, 6.3 * h, 5.2 * h], [7.25 * h, 4.0 * h, 5.0 * h]], dtype=np.float32)
    xs = [7.0, 7.5, 7.9, 11.0, 11.5, 12.0, 15.5, 3.2, 19.7]
    p.rec_coords = np.array([[x * h, 6.5 * h, 5.5 * h] for x in xs], dtype=np.float32)
    return p


def _slab_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1707_03776_b200 as sf
        p = _problem()
        so, r = p.space_order, p.space_order // 2
        n0 = p.shape[0]
        x0, nl = sf.slab_plan(n0, so, rank, world)
        plan = sf.slab_halo_plan(n0, so, rank, world)
        nb = nl + 2 * r
        gidx = np.arange(x0 - r, x0 + nl + r)
        valid = (gidx >= 0) & (gidx < n0)
        m = np.ones((nb,) + p.shape[1:])
        eta = np.zeros((nb,) + p.shape[1:])
        m[valid] = p.m.astype(np.float64)[gidx[valid]]
        eta[valid] = p.damp.astype(np.float64)[gidx[valid]]
        w = oracle.fd_weights(so)
        dt, h = p.dt, p.h
        prv = np.zeros((nb,) + p.shape[1:])
        cur = np.zeros_like(prv)
        rec = np.zeros((p.nt, len(p.rec_coords)))
        own_rec = [sf.sparse_owner(n0, so, world, h, float(c[0])) == rank for c in p.rec_coords]
        st_src = [oracle.point_stencil(p.shape, h, c) for c in p.src_coords.astype(np.float64)]
        st_rec = [oracle.point_stencil(p.shape, h, c) for c in p.rec_coords.astype(np.float64)]
        plane = int(np.prod(p.shape[1:]))

        def loc(gflat):
            gx, rest = divmod(int(gflat), plane)
            return gx, gx - x0 + r, rest

        def exchange(a):
            flat = a.reshape(nb, -1)
            P = plan["planes"]
            reqs = []
            bufs = []
            if plan["has_left"]:
                reqs.append(dist.isend(torch.from_numpy(flat[plan["send_left"]:plan["send_left"] + P].copy()), rank - 1))
                b = torch.empty((P, plane), dtype=torch.float64)
                reqs.append(dist.irecv(b, rank - 1))
                bufs.append((plan["recv_left"], b))
            if plan["has_right"]:
                reqs.append(dist.isend(torch.from_numpy(flat[plan["send_right"]:plan["send_right"] + P].copy()), rank + 1))
                b = torch.empty((P, plane), dtype=torch.float64)
                reqs.append(dist.irecv(b, rank + 1))
                bufs.append((plan["recv_right"], b))
            for rq in reqs:
                rq.wait()
            for start, b in bufs:
                flat[start:start + P] = b.numpy()

        def record(a, n):
            for i, (idx, W) in enumerate(st_rec):
                if not own_rec[i]:
                    continue
                acc = 0.0
                for c in range(len(W)):
                    if W[c] != 0.0:
                        gx, lx, rest = loc(idx[c])
                        assert 0 <= lx < nb, "record corner outside the local buffer (halo too thin?)"
                        acc += W[c] * a.reshape(nb, -1)[lx, rest]
                rec[n, i] = acc

        record(cur, 0)
        for n in range(p.nt - 1):
            lap = oracle.laplacian(cur, h, so)
            nxt = np.zeros_like(cur)
            sl = slice(r, r + nl)
            nxt[sl] = (2 * m[sl] * cur[sl] - (m[sl] - 0.5 * eta[sl] * dt) * prv[sl] + dt * dt * lap[sl]) \
                / (m[sl] + 0.5 * eta[sl] * dt)
            for s, (idx, W) in enumerate(st_src):
                for c in range(len(W)):
                    gx, lx, rest = loc(idx[c])
                    if W[c] != 0.0 and x0 <= gx < x0 + nl:        # corner owned by its plane's rank
                        nf = nxt.reshape(nb, -1)
                        nf[lx, rest] += W[c] * float(p.wavelet[n, s]) * dt * dt / m.reshape(nb, -1)[lx, rest]
            exchange(nxt)
            record(nxt, n + 1)
            prv, cur = cur, nxt
        t = torch.from_numpy(rec)
        dist.all_reduce(t)
        parts = [None] * world
        dist.all_gather_object(parts, (x0, nl, cur[r:r + nl].copy()))
        if rank == 0:
            q.put((t.numpy(), parts))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_decomposition_matches_single_domain(world):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    mp.spawn(_slab_worker, args=(world, port, q), nprocs=world, join=True)
    rec, parts = q.get()
    p = _problem()
    ref = oracle.forward(p)
    np.testing.assert_allclose(rec, ref["rec"], rtol=0, atol=1e-12 * np.abs(ref["rec"]).max())
    u = np.concatenate([c for (_, _, c) in sorted(parts, key=lambda t: t[0])])
    assert u.shape == ref["u_state"][1].shape
    np.testing.assert_allclose(u, ref["u_state"][1], rtol=0, atol=1e-12 * np.abs(u).max())


def _shot_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = synth.random_problem(2, (30, 26), 4, 80, seed=7, nbl=4, nsrc=world, nrec=10)
        m_true = (p.m * 0.95).astype(np.float32)
        # one shot per rank (configs[4]: one shot per GPU)
        p.src_coords = p.src_coords[rank:rank + 1]
        p.wavelet = p.wavelet[:, rank:rank + 1]
        d_obs = oracle.forward(p, m=m_true)["rec"]
        g = oracle.gradient(p, d_obs, save_every=2)
        t = torch.from_numpy(g["grad"].copy())
        J = torch.tensor([g["J"]], dtype=torch.float64)
        dist.all_reduce(t)
        dist.all_reduce(J)
        if rank == 0:
            q.put((t.numpy(), float(J.item())))
    finally:
        dist.destroy_process_group()


def test_multishot_gradient_allreduce():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    mp.spawn(_shot_worker, args=(world, _free_port(), q), nprocs=world, join=True)
    g, J = q.get()
    p = synth.random_problem(2, (30, 26), 4, 80, seed=7, nbl=4, nsrc=world, nrec=10)
    m_true = (p.m * 0.95).astype(np.float32)
    gs, Js = np.zeros(p.shape), 0.0
    for s in range(world):
        ps = synth.random_problem(2, (30, 26), 4, 80, seed=7, nbl=4, nsrc=world, nrec=10)
        ps.src_coords = ps.src_coords[s:s + 1]
        ps.wavelet = ps.wavelet[:, s:s + 1]
        d_obs = oracle.forward(ps, m=m_true)["rec"]
        r = oracle.gradient(ps, d_obs, save_every=2)
        gs += r["grad"]
        Js += r["J"]
    np.testing.assert_allclose(g, gs, rtol=0, atol=1e-12 * np.abs(gs).max())
    assert abs(J - Js) <= 1e-12 * Js


def test_bench_weak_scaling_slabs_tile_the_global_model():
    """bench.py --gpus N builds rank-local slabs (with r halo planes) of the x-tiled
    configs[1] model; stacked, the owned planes must form the global model and the
    absorbing layer must sit only at the global x edges."""
    import sys
    sys.path.insert(0, ROOT)
    import bench
    world = 2
    slabs = []
    for rank in range(world):
        p, m_loc, eta_loc, gshape = bench.build_problem(nt_override=8, rank=rank, nranks=world)
        r = p.space_order // 2
        slabs.append((m_loc[r:-r], eta_loc[r:-r]))
    m = np.concatenate([s[0] for s in slabs])
    eta = np.concatenate([s[1] for s in slabs])
    assert m.shape == gshape and gshape[0] == 336 * world
    assert np.all(m == m[0:1])                          # x-invariant model
    sig = synth.damping_profile(gshape, p.nbl, p.h, 2500.0)
    np.testing.assert_allclose(eta, (m.astype(np.float64) * sig).astype(np.float32))
    assert np.all(eta[p.nbl:-p.nbl, p.nbl:-p.nbl, p.nbl:-p.nbl] == 0)


def test_bench_multishot_ranks_get_distinct_shots():
    """bench.py --gpus N --config 4: every rank runs its own shot (BASELINE configs[4], one
    shot per GPU) on the same full 400^3 model -- distinct source positions, identical
    model and receiver grid, no slab decomposition."""
    import sys
    sys.path.insert(0, ROOT)
    import bench
    shots = [bench.build_problem(nt_override=4, rank=q, nranks=3, cfg=4) for q in range(3)]
    p0, m0, d0, g0 = shots[0]
    assert g0 == p0.shape == (400, 400, 400) and d0 is None
    xs = [s[0].src_coords[0, 0] for s in shots]
    assert len(set(xs)) == 3
    for p, m, d, g in shots[1:]:
        assert g == g0 and d is None
        assert np.array_equal(m, m0)
        assert np.array_equal(p.rec_coords, p0.rec_coords)


def _c3_worker(rank, world, port, strong, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, ROOT)
        import bench
        p, m_loc, eta_loc, gshape = bench.build_problem(nt_override=4, rank=rank, nranks=world, cfg=3,
                                                        strong=strong)
        import paper_1707_03776_b200 as sf
        r = p.space_order // 2
        x0, nl = sf.slab_plan(gshape[0], p.space_order, rank, world)
        assert m_loc.shape == (nl + 2 * r,) + tuple(gshape[1:]) and eta_loc is None
        # fingerprint of the owned planes: the z profile of every owned plane (the model is
        # x-invariant) and the planes' global indices
        prof = torch.from_numpy(m_loc[r:r + nl, 7, :].astype(np.float64).copy())
        idx = torch.arange(x0, x0 + nl, dtype=torch.int64)
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([nl]))
        mx = int(max(s.item() for s in sizes))
        pad = lambda t, fill: torch.cat([t, torch.full((mx - t.shape[0],) + t.shape[1:], fill, dtype=t.dtype)])
        profs = [torch.zeros((mx, gshape[2]), dtype=torch.float64) for _ in range(world)]
        idxs = [torch.zeros(mx, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(profs, pad(prof, -1.0))
        dist.all_gather(idxs, pad(idx, -1))
        if rank == 0:
            q.put((gshape, [int(s.item()) for s in sizes], [t.numpy() for t in profs], [t.numpy() for t in idxs],
                   p.src_coords.copy(), p.rec_coords.copy(), p.h))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("strong", [False, True])
def test_bench_config3_slabs_gloo(strong):
    """bench.py --gpus 2 --config 3 [--strong] (BASELINE configs[3], run at 1/2/4/8 GPUs):
    two gloo ranks build their slabs with bench.build_problem; gathered, the owned planes
    cover the global grid exactly once in order (weak: 1024 N planes, strong: the literal
    1024), every plane carries the configs[3] layered profile, the source sits at the global
    centre and the receivers are one per global plane along x."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_c3_worker, args=(r, world, port, strong, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = q.get(timeout=600)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    gshape, sizes, profs, idxs, src, rec, h = out
    ref = synth.make_config(3, nt=4)
    assert gshape == ((1024,) if strong else (1024 * world,)) + (512, 512)
    assert sum(sizes) == gshape[0]
    allidx = np.concatenate([i[:n] for i, n in zip(idxs, sizes)])
    assert np.array_equal(allidx, np.arange(gshape[0]))
    zprof = ref.m[0, 7, :].astype(np.float64)
    for pr_, n in zip(profs, sizes):
        assert np.array_equal(pr_[:n], np.broadcast_to(zprof, (n, gshape[2])))
    assert np.isclose(src[0, 0], (gshape[0] - 1) * h / 2.0)
    assert rec.shape[0] == gshape[0] and np.array_equal(rec[:, 0], np.arange(gshape[0]) * np.float32(h))
