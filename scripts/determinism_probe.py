#!/usr/bin/env python
"""Determinism probe: a BASELINE config (default configs[4]) at full grid, short record,
repeated in one process (fresh handles, optionally after a configs[3] full-grid forward),
every result compared bitwise with the first (or with a generic-kernel run,
--ref-generic).  Prints which stage diverges and where (records, state, snapshots, J,
gradient).  Found the r >= 5 slot-release race fixed in round 1."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1707_03776_b200 as sf  # noqa: E402
import synth  # noqa: E402


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=8)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--pre-c3", action="store_true")
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--ref-generic", action="store_true", help="compare every rep with a generic-kernel run")
    ap.add_argument("--detail", action="store_true")
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--vy", type=int, default=0)
    ap.add_argument("--prefetch", type=int, default=-1)
    ap.add_argument("--fuse-max", type=int, default=-1)
    ap.add_argument("--no-rec", action="store_true")
    ap.add_argument("--no-save", action="store_true")
    ap.add_argument("--save-every", type=int, default=3)
    ap.add_argument("--noise", action="store_true", help="background matmuls on another stream (staggers CTA starts)")
    ap.add_argument("--no-grad", action="store_true", help="forward only")
    ap.add_argument("--snap-half", action="store_true", help="fp16 snapshots (SF_OPT_SNAP_HALF)")
    ap.add_argument("--sep", action="store_true", help="separable damping profiles instead of the eta array")
    args = ap.parse_args()
    if args.pre_c3:
        p3 = synth.make_config(3, nt=6)
        pr3 = sf.Propagator(dev(p3.m), None, shape=p3.shape, h=p3.h, space_order=p3.space_order, nt=p3.nt,
                            dt=p3.dt, src_coords=p3.src_coords, rec_coords=p3.rec_coords)
        pr3.forward(dev(p3.wavelet))
        torch.cuda.synchronize()
        pr3.close()
        del pr3
    p = synth.make_config(args.config, nt=12)
    if args.no_rec:
        p.rec_coords = p.rec_coords[:1]
    se = 0 if args.no_save else args.save_every
    rng = np.random.default_rng(0)
    d_obs = dev((rng.standard_normal((p.nt, p.rec_coords.shape[0])) * 1e-3).astype(np.float32))
    ref = None
    bad = 0
    if args.ref_generic:
        prop = sf.Propagator(dev(p.m), None if (p.damp is None or args.sep) else dev(p.damp), sigma=p.sigma if args.sep else None, shape=p.shape, h=p.h, space_order=p.space_order, nt=p.nt,
                             dt=p.dt, src_coords=p.src_coords, rec_coords=p.rec_coords)
        prop.set_tuning(1, 0, 0)
        if args.snap_half:
            prop.set_option(7, 1)
        rec, u, snaps = prop.forward(dev(p.wavelet), save_every=se)
        if args.no_grad:
            g, J = torch.zeros(1, device="cuda"), 0.0
        else:
            g, J = prop.gradient(dev(p.wavelet), d_obs, save_every=3)
        torch.cuda.synchronize()
        ref = (rec.cpu().numpy(), u.cpu().numpy(), snaps.cpu().numpy() if snaps is not None else np.zeros(1),
               g.cpu().numpy(), J)
        prop.close()
        print("generic reference: J", J, flush=True)
    for i in range(args.reps):
        prop = sf.Propagator(dev(p.m), None if (p.damp is None or args.sep) else dev(p.damp), sigma=p.sigma if args.sep else None, shape=p.shape, h=p.h, space_order=p.space_order, nt=p.nt,
                             dt=p.dt, src_coords=p.src_coords, rec_coords=p.rec_coords)
        prop.set_tuning(args.variant, args.vy, args.ctas)
        if args.snap_half:
            prop.set_option(7, 1)
        if args.prefetch >= 0:
            prop.set_option(1, args.prefetch)
        if args.fuse_max >= 0:
            prop.set_option(3, args.fuse_max)
        wav_d = dev(p.wavelet)
        torch.cuda.synchronize()
        if args.noise:
            ns = torch.cuda.Stream()
            xa = torch.randn(1 << 22, device="cuda")
            with torch.cuda.stream(ns):
                for _ in range(3000):   # small elementwise kernels, no shared memory
                    xa = torch.tanh(xa * 0.999)
        rec, u, snaps = prop.forward(wav_d, save_every=se)
        if args.no_grad:
            g, J = torch.zeros(1, device="cuda"), 0.0
        else:
            g, J = prop.gradient(dev(p.wavelet), d_obs, save_every=3)
        torch.cuda.synchronize()
        out = (rec.cpu().numpy(), u.cpu().numpy(), snaps.cpu().numpy() if snaps is not None else np.zeros(1),
               g.cpu().numpy(), J)
        prop.close()
        if ref is None:
            ref = out
            print("rep 0: J", J, flush=True)
            continue
        names = ("rec", "u", "snaps", "grad")
        diffs = [n for n, a, b in zip(names, out[:4], ref[:4]) if not np.array_equal(a, b)]
        if out[4] != ref[4]:
            diffs.append("J")
        if diffs:
            bad += 1
            for n, a, b in zip(names, out[:4], ref[:4]):
                if not np.array_equal(a, b):
                    d = np.argwhere(a != b)
                    print(f"rep {i}: {n} differs at {len(d)} entries, first {d[:3].tolist()} "
                          f"rel {np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30):.3e}", flush=True)
                    if args.detail and n == "snaps":
                        slots = np.unique(d[:, 0])
                        s0 = int(slots[0])
                        dd = d[d[:, 0] == s0][:, 1:]
                        print(f"   first bad slot {s0} (of {a.shape[0]}): {len(dd)} points, x {np.unique(dd[:, 0]).tolist()[:12]} "
                              f"y {np.unique(dd[:, 1]).tolist()[:30]} z {np.unique(dd[:, 2]).tolist()[:12]}", flush=True)
                        for k in dd[:4]:
                            kk = (s0,) + tuple(int(v) for v in k)
                            print(f"     {kk}: {a[kk]!r} vs {b[kk]!r}", flush=True)
                    if args.detail and a.ndim >= 3:
                        sp = d[:, -3:]
                        print(f"   x {np.unique(sp[:, 0]).tolist()[:20]} y {np.unique(sp[:, 1]).tolist()[:40]} "
                              f"z {np.unique(sp[:, 2]).tolist()[:20]}", flush=True)
                        k = tuple(d[0])
                        print(f"   at {k}: {a[k]!r} vs {b[k]!r}", flush=True)
            print(f"rep {i}: J {out[4]} vs {ref[4]}", flush=True)
        else:
            print(f"rep {i}: identical", flush=True)
    print("BAD", bad)


if __name__ == "__main__":
    main()
