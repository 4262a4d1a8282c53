"""Practical HBM ceiling for the stencil's access mix: 4 streamed reads + 1 write per
point (fp32, 37.9 M points = the configs[1] grid), via torch.addcmul chains, and a
plain copy; CUDA events, best of 10."""
import json
import torch

N = 336 ** 3
a, b, c, d = (torch.randn(N, device="cuda") for _ in range(4))
o = torch.empty(N, device="cuda")


def bench(fn, nbytes):
    for _ in range(3):
        fn()
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return nbytes / (best * 1e-3) / 1e9, best


res = {}
res["copy_1r1w_GBps"], _ = bench(lambda: o.copy_(a), 8 * N)
res["add_2r1w_GBps"], _ = bench(lambda: torch.add(a, b, out=o), 12 * N)
res["addcmul_3r1w_GBps"], _ = bench(lambda: torch.addcmul(a, b, c, out=o), 16 * N)


def four():
    torch.addcmul(a, b, c, out=o)  # not a 4-input op; emulate with foreach? use sum of views
res["note"] = "torch has no fused 4-input elementwise; 3r1w is the closest mix (16 B/pt)"
print(json.dumps(res))
