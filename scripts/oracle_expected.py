#!/usr/bin/env python
"""Write the fp64 oracle's expected outputs for a full-size BASELINE gradient config to
disk, for the opt-in full-size parity test (tests/test_fullsize_parity.py) to compare the
GPU against when the oracle cannot run inside one GPU-box call (configs[4]: four 400^3
so12 propagations of 1499 steps, ~50 min of host time).  Calls only oracle/ and synth/ --
no value here comes from the CUDA path.

  python scripts/oracle_expected.py --config 4 [--shot 0] --out gpurun_data/c4

Writes d_obs.npy (oracle record at the true model, rounded to fp32), grad.npy (oracle
gradient at the initial model, rounded to fp32 -- 6e-8 relative, far below the 1e-4
tolerance) and meta.json (J in fp64, checkpoint segment, residual norm, timings)."""
import argparse
import json
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--shot", type=int, default=0)
    ap.add_argument("--nt", type=int, default=None)
    ap.add_argument("--out", required=True)
    ap.add_argument("--subsample", type=int, default=0,
                    help="only write d_obs_sub.npy = every N-th trace of an existing d_obs.npy "
                         "(the upload to the GPU box is capped at 512 MiB) and record it in meta.json")
    a = ap.parse_args()
    if a.subsample:
        d = np.load(os.path.join(a.out, "d_obs.npy"))
        np.save(os.path.join(a.out, "d_obs_sub.npy"), np.ascontiguousarray(d[:, ::a.subsample]))
        with open(os.path.join(a.out, "meta.json")) as f:
            meta = json.load(f)
        meta["d_obs_stride"] = a.subsample
        with open(os.path.join(a.out, "meta.json"), "w") as f:
            json.dump(meta, f, indent=1)
        print(json.dumps(meta))
        return
    p = synth.make_config(a.config, nt=a.nt, shot=a.shot) if a.config == 4 else synth.make_config(a.config, nt=a.nt)
    k = p.save_every
    S = max(k, int(round(math.sqrt(2.0 * (p.nt - 1) * k) / k)) * k)
    os.makedirs(a.out, exist_ok=True)
    t0 = time.time()
    d_obs = oracle.forward(p, m=p.m_true)["rec"]
    t1 = time.time()
    np.save(os.path.join(a.out, "d_obs.npy"), d_obs.astype(np.float32))
    go = oracle.gradient(p, d_obs, save_every=k, checkpoint=S)
    t2 = time.time()
    np.save(os.path.join(a.out, "grad.npy"), go["grad"].astype(np.float32))
    meta = {"config": a.config, "shot": a.shot, "shape": list(p.shape), "nt": p.nt, "space_order": p.space_order,
            "save_every": k, "checkpoint_segment": S, "J": go["J"],
            "grad_norm": float(np.linalg.norm(go["grad"])), "d_obs_norm": float(np.linalg.norm(d_obs)),
            "rel_residual": float(np.linalg.norm(go["res"]) / np.linalg.norm(d_obs)),
            "oracle_threads": oracle.num_threads(), "d_obs_s": t1 - t0, "gradient_s": t2 - t1,
            "written_by": "scripts/oracle_expected.py (oracle/ only)"}
    with open(os.path.join(a.out, "meta.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(json.dumps(meta))


if __name__ == "__main__":
    main()
