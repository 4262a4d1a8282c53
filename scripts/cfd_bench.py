#!/usr/bin/env python
"""Timing of the f4 workloads (the paper's convection and Laplace examples) on the GPU
(CUDA events): the paper's sizes (81^2 x 100 steps; 31^2 Jacobi to l1 < 1e-4) and a large
grid for throughput.  One JSON line per case.  (The oracle is test infrastructure and is
not timed here: tests/ compare the results, bench.py times the propagator's oracle.)"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1707_03776_b200 as sf  # noqa: E402
import synth  # noqa: E402


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def timed(fn, reps=5):
    """Median of `reps` event-timed calls after a warm call; a large matmul burst before
    each call keeps the SM clocks up (tiny single-SM workloads otherwise run at idle clocks)."""
    a = torch.randn(4096, 4096, device="cuda")
    fn()
    ts = []
    for _ in range(reps):
        for _ in range(20):
            a @ a
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)), out


def main():
    for shape, nt in (((81, 81), 100), ((4096, 4096), 100)):
        q = synth.convection_problem(*shape, nt=nt)
        u0 = dev(q["u0"])
        u = torch.empty_like(u0)

        def run():
            u.copy_(u0)
            sf.convection2d(u, c=q["c"], dt=q["dt"], dx=q["dx"], dy=q["dy"], nt=q["nt"])
            return u
        ms, _ = timed(run)
        N = shape[0] * shape[1]
        print(json.dumps({"workload": f"convection2d {shape[0]}x{shape[1]}, {nt} steps", "gpu_ms": round(ms, 4),
                          "gpu_GPts": round(N * nt / (ms * 1e-3) / 1e9, 3),
                          "path": "one CTA, shared memory" if N <= 25600 else "kernel per step"}), flush=True)
    for shape in ((31, 31), (160, 160), (2048, 2048)):
        q = synth.laplace_problem(*shape)
        p0, bc = dev(q["p0"]), dev(q["bc"])
        p = torch.empty_like(p0)
        cap = 200 if shape[0] > 1000 else 100000

        def run():
            p.copy_(p0)
            return sf.laplace2d(p, bc, dx=q["dx"], dy=q["dy"], tol=1e-4, max_iter=cap)
        ms, (_, it, l1) = timed(run, reps=3)
        N = shape[0] * shape[1]
        print(json.dumps({"workload": f"laplace2d {shape[0]}x{shape[1]}, l1 < 1e-4 (cap {cap})", "sweeps": it,
                          "l1": l1, "gpu_ms": round(ms, 4), "gpu_GPts": round(N * it / (ms * 1e-3) / 1e9, 3),
                          "path": "one CTA, shared memory" if N <= 4096 else "one cooperative kernel, all SMs"}), flush=True)


if __name__ == "__main__":
    main()
