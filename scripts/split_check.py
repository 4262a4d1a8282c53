#!/usr/bin/env python
"""Boundary-first split schedule (SF_OPT_SPLIT, the slab schedule on one GPU: high-priority
boundary launch + concurrent interior launch) vs the single launch on the FULL configs[1]
and configs[4] grids with snapshots and side-stream records: bitwise, three repetitions.
python scripts/split_check.py"""
import numpy as np, torch, sys
sys.path.insert(0, '/root/repo')
import paper_1707_03776_b200 as sf, synth
def dev(x): return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()
for cfg in (1, 4):
    p = synth.make_config(cfg, nt=16)
    outs = []
    for split in (0, 1, 1, 1):
        prop = sf.Propagator(dev(p.m), None if p.damp is None else dev(p.damp), shape=p.shape, h=p.h,
                             space_order=p.space_order, nt=p.nt, dt=p.dt, src_coords=p.src_coords, rec_coords=p.rec_coords)
        prop.set_option(2, split)
        rec, u, snaps = prop.forward(dev(p.wavelet), save_every=2)
        torch.cuda.synchronize()
        outs.append((rec.cpu().numpy(), u.cpu().numpy(), snaps.cpu().numpy()))
        prop.close()
    bad = sum(0 if all(np.array_equal(a, b) for a, b in zip(o, outs[0])) else 1 for o in outs[1:])
    print("cfg", cfg, "split BAD", bad)
