#!/usr/bin/env python
"""The README usage snippet, runnable: python scripts/examples/readme_snippet.py (B200)."""
import sys; import os; sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), '..', '..'))
import torch, paper_1707_03776_b200 as sf, synth
p = synth.make_config(1, nt=200)                       # BASELINE configs[1] model, seeded
dev = lambda a: torch.from_numpy(a).cuda()
prop = sf.Propagator(dev(p.m), dev(p.damp), shape=p.shape, h=p.h, space_order=8,
                     nt=p.nt, dt=p.dt, src_coords=p.src_coords, rec_coords=p.rec_coords)
rec, u, _ = prop.forward(dev(p.wavelet))                # records [nt][nrec], final levels
g, J = prop.gradient(dev(p.wavelet), rec, save_every=4) # FWI gradient (zero residual here)
prop.set_option(sf.SF_OPT_SNAP_HALF, 1)                 # fp16 snapshots, etc. (include/sf.h)
print("README snippet ok", rec.shape, float(J), float(g.abs().max()))
