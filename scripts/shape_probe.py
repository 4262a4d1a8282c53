#!/usr/bin/env python
"""Stencil-launch time vs grid shape (constant model, random wavefield, no sparse points):
shows how the tile geometry packs a given (n1, n2) -- idle lanes of ragged z tiles, idle
SMs, warm-up planes.  Usage: python scripts/shape_probe.py [--so 8] [--nt 40] [--damp]
[--shapes 336x336x336,336x336x384]"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1707_03776_b200 as sf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--so", type=int, default=8)
    ap.add_argument("--nt", type=int, default=40)
    ap.add_argument("--damp", action="store_true")
    ap.add_argument("--vy", type=int, default=2)
    ap.add_argument("--zsplit", type=int, default=1, help="SF_OPT_ZSPLIT (narrow tiles for a z remainder)")
    ap.add_argument("--variant", type=int, default=2, help="1 generic, 2 TMA")
    ap.add_argument("--ctas", default="0", help="comma list of persistent CTA counts (0 = auto)")
    ap.add_argument("--shapes", default="336x336x336,336x336x384,336x336x320,336x336x256,336x392x336")
    args = ap.parse_args()
    for s in args.shapes.split(","):
        shape = tuple(int(x) for x in s.split("x"))
        m = torch.full(shape, 1.0 / 2.0 ** 2, device="cuda")
        eta = torch.full(shape, 0.01, device="cuda") if args.damp else None
        prop = sf.Propagator(m, eta, shape=shape, h=10.0, space_order=args.so, nt=args.nt, dt=1.0,
                             src_coords=None, rec_coords=None)
        prop.set_option(9, args.zsplit)
        N = int(np.prod(shape))
        g = torch.Generator(device="cuda").manual_seed(0)
        u0 = torch.randn((2,) + shape, device="cuda", generator=g) * 1e-3
        for ctas in [int(c) for c in args.ctas.split(",")]:
            prop.set_tuning(args.variant, args.vy if args.variant == 2 else 0, ctas)
            best = None
            for rep in range(3):
                prop.set_profiling(True)
                prop.profile(reset=True)
                prop.forward(None, u=u0.clone())
                torch.cuda.synchronize()
                pr = prop.profile(reset=True)
                ms = pr["stencil_ms"] / pr["stencil_launches"]
                best = ms if best is None else min(best, ms)
            bpp = 20 if args.damp else 16
            print(json.dumps({"shape": shape, "so": args.so, "tuning": prop.tuning(),
                              "launch_us": round(best * 1e3, 2), "ns_per_kpt": round(best * 1e6 / (N / 1e3), 4),
                              "GBps": round(bpp * N / (best * 1e-3) / 1e9, 1)}), flush=True)
        prop.close()
        del prop, m, eta, u0
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
