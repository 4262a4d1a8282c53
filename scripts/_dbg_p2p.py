import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import synth, oracle
import paper_1707_03776_b200 as S
from test_gpu_parity import _slab_inputs, _run_ranks, dev
for nt in (3, 4):
    p = synth.random_problem(3, (41, 30, 64), 8, nt, seed=91, nbl=5, nsrc=3, nrec=40)
    h = p.h
    p.src_coords[0, 0] = 13.5 * h; p.src_coords[1, 0] = 20.2 * h
    p.rec_coords[:20, 0] = np.linspace(8 * h, 33 * h, 20)
    prop = S.Propagator(dev(p.m), dev(p.damp), shape=p.shape, h=p.h, space_order=8, nt=p.nt, dt=p.dt,
                        src_coords=p.src_coords.astype(np.float64), rec_coords=p.rec_coords.astype(np.float64))
    rec1, u1, _ = prop.forward(dev(p.wavelet)); torch.cuda.synchronize(); u1 = u1.cpu().numpy(); rec1 = rec1.cpu().numpy()
    group = S.local_group_create(2); r = 4
    def fn(rank):
        x0, nl, m, eta = _slab_inputs(p, rank, 2)
        pr = S.Propagator(dev(m), dev(eta), shape=p.shape, h=p.h, space_order=8, nt=p.nt, dt=p.dt,
                          src_coords=p.src_coords.astype(np.float64), rec_coords=p.rec_coords.astype(np.float64),
                          comm=group, rank=rank, nranks=2)
        pr.set_option(8, 1)
        rec, u, _ = pr.forward(dev(p.wavelet)); torch.cuda.current_stream().synchronize()
        n = pr.debug_probe(None)
        return x0, nl, u.cpu().numpy(), rec.cpu().numpy(), n
    outs = _run_ranks(2, fn)
    S.local_group_destroy(group)
    for x0, nl, u, rec, n in outs:
        for lv in (0, 1):
            own = u[lv, r:r + nl]; ref = u1[lv, x0:x0 + nl]
            bad = np.argwhere(own != ref)
            print("nt", nt, "rank x0", x0, "lv", lv, "onelaunch", n, "bad", len(bad), "planes", sorted(set((bad[:, 0] + x0).tolist()))[:12])
            # halos
            for side, (lo, hi) in (("L", (0, r)), ("R", (r + nl, 2 * r + nl))):
                g0 = x0 - r if side == "L" else x0 + nl
                if g0 < 0 or g0 + r > p.shape[0]: continue
                hb = np.argwhere(u[lv, lo:hi] != u1[lv, g0:g0 + r])
                print("   halo", side, "bad", len(hb), sorted(set((hb[:, 0] + g0).tolist()))[:8], "rows", sorted(set(hb[:, 1].tolist()))[:20])
                for b in hb[:4]:
                    pl, yy, zz = b
                    print("      ", (pl + g0, yy, zz), "halo", u[lv, lo + pl, yy, zz], "ref", u1[lv, g0 + pl, yy, zz])
