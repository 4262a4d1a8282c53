#!/usr/bin/env python
"""Checkpointed gradient (sf_gradient_ckpt) vs the full-snapshot gradient on the
FULL configs[2] / configs[4] grids (short record, side-stream records active): must be
bitwise equal, three repetitions each.  Run on a B200: python scripts/ckpt_check.py"""
import numpy as np, torch, sys
sys.path.insert(0, '/root/repo')
import paper_1707_03776_b200 as sf, synth
def dev(x): return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()
for cfg in (2, 4):
    p = synth.make_config(cfg, nt=20)
    rng = np.random.default_rng(0)
    d_obs = dev((rng.standard_normal((p.nt, p.rec_coords.shape[0])) * 1e-3).astype(np.float32))
    prop = sf.Propagator(dev(p.m), None if p.damp is None else dev(p.damp), shape=p.shape, h=p.h, space_order=p.space_order,
                         nt=p.nt, dt=p.dt, src_coords=p.src_coords, rec_coords=p.rec_coords)
    k = p.save_every or 2
    g0, J0 = prop.gradient(dev(p.wavelet), d_obs, save_every=k)
    g0 = g0.cpu().numpy()
    bad = 0
    for rep in range(3):
        g1, J1 = prop.gradient_ckpt(dev(p.wavelet), d_obs, save_every=k, segment=3 * k)
        torch.cuda.synchronize()
        if not (np.array_equal(g1.cpu().numpy(), g0) and J1 == J0):
            bad += 1
    print("cfg", cfg, "ckpt BAD", bad)
    prop.close()
