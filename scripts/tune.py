#!/usr/bin/env python
"""Sweep the stencil kernel's launch tuning (tile rows, persistent CTA count) on a BASELINE
config and print the average stencil-launch time and GB/s (CUDA events around every
stencil launch, recorded by libsf).  Usage: python scripts/tune.py [--config 1] [--nt 60]"""
import argparse
import itertools
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1707_03776_b200 as sf  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--nt", type=int, default=60)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--vy", default="2")
    ap.add_argument("--ctas", default="0")
    ap.add_argument("--grad", action="store_true", help="time the adjoint with fused gradient")
    ap.add_argument("--sep", action="store_true", help="separable damping profiles (16 B/pt)")
    ap.add_argument("--prefetch", default="0", help="comma list of L2 prefetch distances (planes)")
    ap.add_argument("--balance", default="0", help="comma list of SF_OPT_BALANCE values (0 chunked, 1 balanced)")
    ap.add_argument("--random-init", action="store_true",
                    help="start from a random (incompressible) wavefield instead of zeros")
    args = ap.parse_args()
    p = synth.make_config(args.config, scale=args.scale, nt=args.nt)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()
    sep = args.sep and p.sigma is not None
    prop = sf.Propagator(dev(p.m), None if (p.damp is None or sep) else dev(p.damp), shape=p.shape, h=p.h,
                         space_order=p.space_order, nt=p.nt, dt=p.dt, src_coords=p.src_coords,
                         rec_coords=p.rec_coords, sigma=p.sigma if sep else None)
    N = int(np.prod(p.shape))
    bpp = 20 if (p.damp is not None and not sep) else 16
    wav = dev(p.wavelet)
    out = []
    snaps = None
    if args.grad:
        k = p.save_every or 4
        _, _, snaps = prop.forward(wav, save_every=k)
        res = torch.randn((p.nt, p.rec_coords.shape[0]), device="cuda")
    for vy, ch, pf, bal in itertools.product([int(x) for x in args.vy.split(",")],
                                             [int(x) for x in args.ctas.split(",")],
                                             [int(x) for x in args.prefetch.split(",")],
                                             [int(x) for x in args.balance.split(",")]):
        try:
            prop.set_tuning(2, vy, ch)
            prop.set_option(1, pf)
            prop.set_option(sf.SF_OPT_BALANCE, bal)
        except sf.SfError:
            continue
        t = prop.tuning()
        for rep in range(2):
            prop.set_profiling(True)
            prop.profile(reset=True)
            if args.grad:
                prop.adjoint(res, snaps=snaps, save_every=k)
            else:
                u0 = None
                if args.random_init:
                    g = torch.Generator(device="cuda").manual_seed(0)
                    u0 = torch.randn((2,) + prop.local_shape, device="cuda", generator=g) * 1e-3
                prop.forward(wav, u=u0)
            torch.cuda.synchronize()
            pr = prop.profile(reset=True)
        ms = pr["stencil_ms"] / pr["stencil_launches"]
        extra = (4 + 12 / k) if args.grad else 0
        gbs = (bpp + extra) * N / (ms * 1e-3) / 1e9
        row = {"vy": t["vy"], "ctas": t["ctas"], "req_ctas": ch, "prefetch": pf, "balance": bal, "launch_ms": round(ms, 5),
               "interp_us": round(pr["interp_ms"] * 1e3 / max(pr["interp_launches"], 1), 2),
               "GBps": round(gbs, 1), "GPts": round(N / (ms * 1e-3) / 1e9, 2)}
        print(json.dumps(row), flush=True)
        out.append(row)
    best = min(out, key=lambda r: r["launch_ms"])
    print("BEST", json.dumps(best))


if __name__ == "__main__":
    main()
