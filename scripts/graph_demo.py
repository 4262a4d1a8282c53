#!/usr/bin/env python
"""Per-call time of sf_forward eager vs CUDA-graph replay (SF_OPT_GRAPH) on a config
(default configs[0]: 2D 141^2, so4, nt=500 -- launch-bound)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1707_03776_b200 as sf  # noqa: E402
import synth  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    p = synth.make_config(cfg)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for graph in (0, 1):
            prop = sf.Propagator(dev(p.m), None if p.damp is None else dev(p.damp), shape=p.shape, h=p.h,
                                 space_order=p.space_order, nt=p.nt, dt=p.dt, src_coords=p.src_coords,
                                 rec_coords=p.rec_coords)
            prop.set_option(5, graph)
            wav = dev(p.wavelet)
            u = prop.zeros_state()
            rec = torch.empty((p.nt, p.rec_coords.shape[0]), device="cuda")
            for _ in range(3):
                prop.forward(wav, u=u, rec=rec)
            s.synchronize()
            n = 20
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record(s)
            for _ in range(n):
                prop.forward(wav, u=u, rec=rec)
            e1.record(s)
            s.synchronize()
            wall = (time.perf_counter() - t0) / n * 1e3
            ms = e0.elapsed_time(e1) / n
            N = int(np.prod(p.shape))
            print(f"config {cfg} graph={graph}: {ms:.3f} ms/forward (device), {wall:.3f} ms wall, "
                  f"{N * (p.nt - 1) / (ms * 1e-3) / 1e9:.2f} GPts/s", flush=True)
            prop.close()


if __name__ == "__main__":
    main()
