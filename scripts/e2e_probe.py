#!/usr/bin/env python
"""Time the phases of the end-to-end forward (host buffers) on configs[1]: pinned H2D,
handle creation (sf_create), forward, D2H, destroy -- to see where e2e time goes."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1707_03776_b200 as sf  # noqa: E402
import synth  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    p = synth.make_config(cfg)
    pin = lambda x: torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).pin_memory()
    m_h, d_h, w_h = pin(p.m), pin(p.damp), pin(p.wavelet)
    rec_h = torch.empty((p.nt, p.rec_coords.shape[0]), dtype=torch.float32).pin_memory()
    for it in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        m_d, d_d, w_d = m_h.cuda(non_blocking=True), d_h.cuda(non_blocking=True), w_h.cuda(non_blocking=True)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        prop = sf.Propagator(m_d, d_d, shape=p.shape, h=p.h, space_order=p.space_order, nt=p.nt, dt=p.dt,
                             src_coords=p.src_coords, rec_coords=p.rec_coords)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        rec, u, _ = prop.forward(w_d)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        rec_h.copy_(rec)
        t4 = time.perf_counter()
        prop.close()
        torch.cuda.synchronize()
        t5 = time.perf_counter()
        sf.forward_host(m_h.numpy(), d_h.numpy(), h=p.h, space_order=p.space_order, nt=p.nt, dt=p.dt,
                        src_coords=p.src_coords, wavelet=w_h.numpy(), rec_coords=p.rec_coords,
                        rec_out=rec_h.numpy())
        t6 = time.perf_counter()
        print(f"iter {it}: h2d {1e3*(t1-t0):.1f} ms, create {1e3*(t2-t1):.1f}, forward {1e3*(t3-t2):.1f}, "
              f"d2h {1e3*(t4-t3):.1f}, destroy {1e3*(t5-t4):.1f} | forward_host {1e3*(t6-t5):.1f} ms", flush=True)


if __name__ == "__main__":
    main()
