#!/usr/bin/env python
"""Slab path at full configs[1] size on ONE B200: 2 or 3 rank threads over the in-process
transport (NCCL exchange planes) or with peer stores (SF_OPT_P2P), every rank's local grid
large enough for the side-stream records (the concurrency the small unit tests do not
reach).  Records, owned planes of the final state and the gradient must equal the single-
domain run bit for bit.  python scripts/slab_check.py [--nranks 2] [--p2p] [--nt 30]"""
import argparse
import os
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1707_03776_b200 as sf  # noqa: E402
import synth  # noqa: E402


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nranks", type=int, default=2)
    ap.add_argument("--p2p", action="store_true")
    ap.add_argument("--nt", type=int, default=30)
    args = ap.parse_args()
    p = synth.make_config(1, nt=args.nt)
    p.m_true = (p.m * 0.95).astype(np.float32)
    rng = np.random.default_rng(0)
    d_obs = (rng.standard_normal((p.nt, p.rec_coords.shape[0])) * 1e-3).astype(np.float32)
    prop = sf.Propagator(dev(p.m), dev(p.damp), shape=p.shape, h=p.h, space_order=p.space_order, nt=p.nt,
                         dt=p.dt, src_coords=p.src_coords, rec_coords=p.rec_coords)
    rec1, u1, _ = prop.forward(dev(p.wavelet))
    g1, J1 = prop.gradient(dev(p.wavelet), dev(d_obs), save_every=4)
    torch.cuda.synchronize()
    rec1, u1, g1 = rec1.cpu().numpy(), u1.cpu().numpy(), g1.cpu().numpy()
    prop.close()
    del prop
    torch.cuda.empty_cache()
    r = p.space_order // 2
    group = sf.local_group_create(args.nranks)
    outs, errs = [None] * args.nranks, []

    def body(rank):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                x0, nl = sf.slab_plan(p.shape[0], p.space_order, rank, args.nranks)
                g = np.arange(x0 - r, x0 + nl + r)
                ok = (g >= 0) & (g < p.shape[0])
                m = np.ones((nl + 2 * r,) + p.shape[1:], np.float32)
                m[ok] = p.m[g[ok]]
                eta = np.zeros_like(m)
                eta[ok] = p.damp[g[ok]]
                pr = sf.Propagator(dev(m), dev(eta), shape=p.shape, h=p.h, space_order=p.space_order, nt=p.nt,
                                   dt=p.dt, src_coords=p.src_coords, rec_coords=p.rec_coords, comm=group,
                                   rank=rank, nranks=args.nranks)
                if args.p2p:
                    pr.set_option(8, 1)
                rec, u, _ = pr.forward(dev(p.wavelet))
                gg, J = pr.gradient(dev(p.wavelet), dev(d_obs), save_every=4)
                st.synchronize()
                outs[rank] = (x0, nl, rec.cpu().numpy(), u.cpu().numpy()[:, r:r + nl], gg.cpu().numpy()[r:r + nl], J)
                pr.close()
        except BaseException as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=body, args=(q,)) for q in range(args.nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    sf.local_group_destroy(group)
    assert not errs, errs
    ok = np.array_equal(sum(o[2] for o in outs), rec1)
    for x0, nl, _, u, g, J in outs:
        ok &= np.array_equal(u, u1[:, x0:x0 + nl]) and np.array_equal(g, g1[x0:x0 + nl]) and J == J1
    print(f"nranks {args.nranks} p2p {args.p2p}: {'BITWISE OK' if ok else 'MISMATCH'}")


if __name__ == "__main__":
    main()
