import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import synth, paper_1707_03776_b200 as sf
p = synth.make_config(1, nt=200)
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()
for recs in (True, False, True, False):
    pr = sf.Propagator(dev(p.m), dev(p.damp), shape=p.shape, h=p.h, space_order=8, nt=p.nt, dt=p.dt,
                       src_coords=p.src_coords, rec_coords=p.rec_coords if recs else None)
    w = dev(p.wavelet)
    for _ in range(2): pr.forward(w)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): pr.forward(w)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print("records" if recs else "no records", round(ms, 3), "ms/forward", round(p.npoints * (p.nt - 1) / (ms * 1e-3) / 1e9, 1), "GPts/s")
    pr.close()
