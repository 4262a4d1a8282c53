"""Tiny forward / adjoint / gradient runs through every kernel family (TMA 3D with fused
and standalone sparse work, generic 3D, generic 2D, split launches) for
compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1707_03776_b200 as sf  # noqa: E402
import synth  # noqa: E402


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def run(p, variant, fuse, split):
    prop = sf.Propagator(dev(p.m), None if p.damp is None else dev(p.damp), shape=p.shape, h=p.h,
                         space_order=p.space_order, nt=p.nt, dt=p.dt, src_coords=p.src_coords,
                         rec_coords=p.rec_coords)
    if len(p.shape) == 3:
        prop.set_tuning(variant, 0, 2)
    prop.set_option(3, fuse)
    prop.set_option(2, split)
    rec, u, _ = prop.forward(dev(p.wavelet))
    d_obs = (rec * 0.9).contiguous()
    g, J = prop.gradient(dev(p.wavelet), d_obs, save_every=2)
    torch.cuda.synchronize()
    prop.close()
    return float(J)


for so in (4, 8, 16):
    p = synth.random_problem(3, (14, 18, 132), so, 8, seed=so, nbl=3, nsrc=2, nrec=20)
    for variant in (1, 2):
        for fuse in (0, 256):
            for split in (0, 1):
                run(p, variant, fuse, split)
p = synth.random_problem(2, (20, 24), 4, 8, seed=1, nbl=3, nsrc=1, nrec=5)
run(p, 1, 0, 0)
print("sanitize run ok")


# separable damping (in-kernel beta) and the checkpointed gradient, TMA variant
p = synth.random_problem(3, (14, 18, 132), 8, 9, seed=5, nbl=3, nsrc=2, nrec=20)
prop = sf.Propagator(dev(p.m), None, shape=p.shape, h=p.h, space_order=8, nt=p.nt, dt=p.dt,
                     src_coords=p.src_coords, rec_coords=p.rec_coords, sigma=p.sigma)
rec, u, _ = prop.forward(dev(p.wavelet))
g, J = prop.gradient_ckpt(dev(p.wavelet), (rec * 0.9).contiguous(), save_every=2, segment=4)
torch.cuda.synchronize()
prop.close()
print("sanitize run done")
