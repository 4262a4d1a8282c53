"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic (no stencil, no interpolation,
no injection, no gradient): it only draws the *inputs* the paper's seismic
example feeds to its operators -- square slowness m, damping eta, Ricker source
signatures and source/receiver coordinates -- with the shapes, value ranges and
structure of the workloads in BASELINE.json ``configs``.

Citations: ``P:n`` = /root/reference/PAPER.md line n (not read at run time).
  * m = 1/v^2 "square slowness", eta "spatially varying dampening factor used to
    implement an absorbing boundary condition" -- P:479-485 (acoustic wave eq.).
  * Ricker source -- P:629-633 ("Create source with Ricker wavelet"); formula is
    reading C10.
  * Model utility providing m, eta and coordinates -- P:617-627 (internals elided);
    our geometry/damping readings C7, C8, C16, C17 are listed in DESIGN.md.

Everything is SI: metres, seconds, m/s; m in s^2/m^2.  Arrays are float32
(the GPU consumes fp32; the oracle receives float64 copies of the same values).
Grid layout: 3D ``[x][y][z]`` (z = depth, fastest), 2D ``[x][z]``.
Coordinates are metres from computational index 0 (the padding is included).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

__all__ = [
    "ricker", "damping_profile", "damping_profiles_1d", "pad_edge", "convection_problem",
    "laplace_problem", "Problem", "make_config",
    "random_problem", "CONFIG_NAMES",
]


def ricker(nt: int, dt: float, f0: float, t0: Optional[float] = None) -> np.ndarray:
    """Ricker wavelet w(t) = (1 - 2 pi^2 f^2 (t-t0)^2) exp(-pi^2 f^2 (t-t0)^2),
    t0 = 1/f, sampled at t_n = n*dt (reading C10; P:629-633 names it only)."""
    if t0 is None:
        t0 = 1.0 / f0
    t = np.arange(nt, dtype=np.float64) * dt
    a = (math.pi * f0 * (t - t0)) ** 2
    return ((1.0 - 2.0 * a) * np.exp(-a)).astype(np.float32)


def pad_edge(v: np.ndarray, nbl: int, axes=None) -> np.ndarray:
    """Edge-replicate a physical model by nbl points on the given axes (reading C8:
    the absorbing layer lies OUTSIDE the stated grid, like Devito's Model padding)."""
    if nbl == 0:
        return v.copy()
    axes = range(v.ndim) if axes is None else axes
    pw = [(nbl, nbl) if a in axes else (0, 0) for a in range(v.ndim)]
    return np.pad(v, pw, mode="edge")


def damping_profiles_1d(shape_comp, nbl: int, h: float, vmax: float) -> list:
    """Per-axis damping profiles sigma_a(i) = sigma_max (d_a/nbl)^2 [1/s], d_a = points
    beyond the physical region on axis a (0 inside), sigma_max = 3 vmax ln(1e3)/(2 nbl h)
    (reading C7), rounded to fp32: the separable damping input (sf_desc.sigma)."""
    out = []
    for n in shape_comp:
        if nbl == 0:
            out.append(np.zeros(n, dtype=np.float32))
            continue
        smax = 3.0 * vmax * math.log(1e3) / (2.0 * nbl * h)
        i = np.arange(n, dtype=np.float64)
        d = np.maximum(np.maximum(nbl - i, i - (n - 1 - nbl)), 0.0)
        out.append((smax * (d / nbl) ** 2).astype(np.float32))
    return out


def damping_profile(shape_comp, nbl: int, h: float, vmax: float) -> np.ndarray:
    """sigma(x) = sum_axes sigma_a(x_a) (the fp32 1D profiles above, summed in fp64);
    eta = m * sigma is formed by the caller.  Returns sigma in 1/s."""
    sig = np.zeros(shape_comp, dtype=np.float64)
    for a, prof in enumerate(damping_profiles_1d(shape_comp, nbl, h, vmax)):
        sh = [1] * len(shape_comp)
        sh[a] = len(prof)
        sig = sig + prof.astype(np.float64).reshape(sh)
    return sig


@dataclass
class Problem:
    """One acoustic problem instance (all arrays fp32, computational grid)."""
    name: str
    ndim: int
    shape: tuple
    h: float
    space_order: int
    nt: int
    dt: float
    m: np.ndarray                      # [N] s^2/m^2, shape `shape`
    damp: Optional[np.ndarray]         # eta, same shape, or None (== 0)
    src_coords: np.ndarray             # [nsrc][ndim] metres from comp index 0
    wavelet: np.ndarray                # [nt][nsrc]
    rec_coords: np.ndarray             # [nrec][ndim]
    save_every: int = 0
    nbl: int = 0
    m_true: Optional[np.ndarray] = None  # gradient configs: model generating d_obs
    extra: dict = field(default_factory=dict)
    sigma: Optional[list] = None       # separable form of damp: damp = m * sum_a sigma[a]

    @property
    def npoints(self) -> int:
        return int(np.prod(self.shape))


CONFIG_NAMES = ["C1_2d_fwd", "C2_3d_fwd", "C3_3d_grad", "C4_3d_slab", "C5_multishot"]


def _dt(h: float, vmax: float) -> float:
    # Reading C16: dt = 0.4 h / vmax over all models of the run (BASELINE configs[0]).
    return 0.4 * h / vmax


def _scaled(n: int, scale: float, lo: int = 8) -> int:
    return max(lo, int(round(n * scale)))


def make_config(i: int, scale: float = 1.0, nt: Optional[int] = None, shot: int = 0) -> Problem:
    """BASELINE.json configs[i] as read in SURVEY.md §8.0 (readings in DESIGN.md).

    ``scale`` < 1 shrinks the physical grid and padding (test sizes that keep the
    same structure); ``nt`` overrides the number of time samples.
    """
    if i == 0:
        # 2D 101x101, h=10, v=1500, so4, nt=500, 10 Hz Ricker at (500,20) m,
        # 101 receivers at depth 20 m, 20-pt quadratic damping layer (outside).
        nphys = _scaled(101, scale)
        nbl = _scaled(20, scale, lo=4)
        h = 10.0
        v = np.full((nphys, nphys), 1500.0)
        vp = pad_edge(v, nbl)
        shape = vp.shape
        vmax = 1500.0
        dt = _dt(h, vmax)
        ntt = nt if nt is not None else _scaled(500, scale, lo=20)
        m = (1.0 / vp ** 2)
        sig = damping_profile(shape, nbl, h, vmax)
        damp = m * sig
        xs = min(500.0, (nphys - 1) * h / 2)
        src = np.array([[xs + nbl * h, 20.0 + nbl * h]])
        nrec = nphys
        rec = np.stack([np.arange(nrec) * h * (nphys - 1) / (nrec - 1) + nbl * h,
                        np.full(nrec, 20.0 + nbl * h)], axis=1)
        wav = ricker(ntt, dt, 10.0)[:, None]
        p0 = Problem("C1_2d_fwd", 2, shape, h, 4, ntt, dt, m.astype(np.float32),
                     damp.astype(np.float32), src.astype(np.float32), wav,
                     rec.astype(np.float32), 0, nbl)
        p0.sigma = damping_profiles_1d(shape, nbl, h, vmax)
        return p0
    if i in (1, 2):
        nphys = _scaled(256, scale)
        nbl = _scaled(40, scale, lo=4)
        h = 10.0
        zc = np.arange(nphys) * h
        if i == 1:
            # two-layer: 1.5 km/s above z=1280 m, 2.5 km/s below (tie -> deeper, C17)
            vz = np.where(zc < 1280.0 * scale, 1500.0, 2500.0)
            v = np.broadcast_to(vz, (nphys, nphys, nphys)).astype(np.float64)
            vtrue = None
            vmax = float(v.max())
        else:
            layers = np.array([1500.0, 2000.0, 2500.0, 3000.0, 3500.0])
            k = np.arange(nphys)
            vz = layers[np.minimum((5 * k) // nphys, 4)]
            g = np.arange(nphys) * h
            c = (nphys - 1) * h / 2.0
            sig_a = 200.0 * scale
            r2 = ((g[:, None, None] - c) ** 2 + (g[None, :, None] - c) ** 2
                  + (g[None, None, :] - c) ** 2)
            vtrue = np.broadcast_to(vz, (nphys,) * 3) + 300.0 * np.exp(-r2 / (2 * sig_a ** 2))
            from scipy.ndimage import gaussian_filter
            v = gaussian_filter(vtrue, 10 * scale, mode="nearest", truncate=4.0)
            vmax = float(max(vtrue.max(), v.max()))
        vp = pad_edge(v, nbl)
        shape = vp.shape
        dt = _dt(h, vmax)
        ntt = nt if nt is not None else _scaled(1000, scale, lo=20)
        m = 1.0 / vp ** 2
        damp = m * damping_profile(shape, nbl, h, vmax)
        cphys = (nphys - 1) * h / 2.0
        src = np.array([[cphys + nbl * h, cphys + nbl * h, nbl * h]])
        ii, jj = np.meshgrid(np.arange(nphys), np.arange(nphys), indexing="ij")
        rec = np.stack([(ii.ravel() + nbl) * h, (jj.ravel() + nbl) * h,
                        np.full(ii.size, nbl * h)], axis=1)
        wav = ricker(ntt, dt, 15.0)[:, None]
        p = Problem(CONFIG_NAMES[i], 3, shape, h, 8, ntt, dt, m.astype(np.float32),
                    damp.astype(np.float32), src.astype(np.float32), wav,
                    rec.astype(np.float32), 4 if i == 2 else 0, nbl)
        p.sigma = damping_profiles_1d(shape, nbl, h, vmax)
        if i == 2:
            p.m_true = (1.0 / pad_edge(vtrue, nbl) ** 2).astype(np.float32)
        return p
    if i == 3:
        # 1024x512x512, h=10, random 8-layer 1.5-4.5 km/s with seed-drawn interfaces
        # +-50 m, so16, nt=500, single Ricker, no damping layer (reading C8).
        n0, n1, n2 = _scaled(1024, scale), _scaled(512, scale), _scaled(512, scale)
        h = 10.0
        vals = np.linspace(1500.0, 4500.0, 8)
        delta = np.random.default_rng(4).uniform(-50.0, 50.0, 7)
        depth = np.arange(n2) * h / max(scale, 1e-9) if scale != 1.0 else np.arange(n2) * h
        j = np.arange(1, 8)
        idx = (depth[:, None] >= (640.0 * j + delta)[None, :]).sum(axis=1)
        vz = vals[idx]
        v = np.broadcast_to(vz, (n0, n1, n2))
        vmax = 4500.0
        dt = _dt(h, vmax)
        ntt = nt if nt is not None else _scaled(500, scale, lo=20)
        m = np.ascontiguousarray(1.0 / v ** 2)
        src = np.array([[(n0 - 1) * h / 2.0, (n1 - 1) * h / 2.0, 0.0]])
        nrec = n0
        rec = np.stack([np.arange(nrec) * h, np.full(nrec, (n1 - 1) * h / 2.0),
                        np.zeros(nrec)], axis=1)
        wav = ricker(ntt, dt, 15.0)[:, None]
        return Problem("C4_3d_slab", 3, (n0, n1, n2), h, 16, ntt, dt, m.astype(np.float32),
                       None, src.astype(np.float32), wav, rec.astype(np.float32), 0, 0)
    if i == 4:
        n = _scaled(400, scale)
        h = 12.5
        L = (n - 1) * h
        vals = np.linspace(1500.0, 4500.0, 6)
        k = np.arange(n)
        vz = vals[np.minimum((6 * k) // n, 5)]
        cen = np.random.default_rng(5).uniform(0.25, 0.75, (3, 3)) * L
        g = np.arange(n) * h
        sig_a = 200.0 * max(scale, 0.05)
        vtrue = np.broadcast_to(vz, (n, n, n)).astype(np.float64).copy()
        for c in cen:
            r2 = ((g[:, None, None] - c[0]) ** 2 + (g[None, :, None] - c[1]) ** 2
                  + (g[None, None, :] - c[2]) ** 2)
            vtrue += 300.0 * np.exp(-r2 / (2 * sig_a ** 2))
        from scipy.ndimage import gaussian_filter
        vinit = gaussian_filter(vtrue, 10 * scale, mode="nearest", truncate=4.0)
        vmax = float(max(vtrue.max(), vinit.max()))
        dt = _dt(h, vmax)
        ntt = nt if nt is not None else _scaled(1500, scale, lo=20)
        xs = (shot + 0.5) * L / 8.0
        src = np.array([[xs, L / 2.0, 0.0]])
        ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
        rec = np.stack([ii.ravel() * h, jj.ravel() * h, np.zeros(ii.size)], axis=1)
        wav = ricker(ntt, dt, 10.0)[:, None]
        p = Problem("C5_multishot", 3, (n, n, n), h, 12, ntt, dt,
                    (1.0 / vinit ** 2).astype(np.float32), None, src.astype(np.float32),
                    wav, rec.astype(np.float32), 3, 0)
        p.m_true = (1.0 / vtrue ** 2).astype(np.float32)
        p.extra["shot"] = shot
        return p
    raise ValueError(f"no config {i}")


def random_problem(ndim: int, shape, space_order: int, nt: int, *, seed: int = 0,
                   h: float = 10.0, nbl: int = 0, nsrc: int = 2, nrec: int = 7,
                   courant: float = 0.4, vmin: float = 1500.0, vmax: float = 2300.0,
                   damp: bool = True, f0: float = 15.0,
                   random_wavelet: bool = False) -> Problem:
    """Small random problem (tests): random velocity in [vmin, vmax], an interior
    damping ring of width nbl (sources/receivers placed where eta == 0, reading C9),
    off-node sources and receivers."""
    rng = np.random.default_rng(seed)
    shape = tuple(int(s) for s in shape)
    v = rng.uniform(vmin, vmax, size=shape)
    m = 1.0 / v ** 2
    dt = courant * h / vmax
    if damp and nbl > 0:
        inner = tuple(s - 2 * nbl for s in shape)
        sig = damping_profile(shape, nbl, h, vmax)
        del inner
        eta = m * sig
    else:
        eta = None
    lo = np.array([nbl + 0.5] * ndim) * h
    hi = (np.array(shape) - 1 - nbl - 1.5) * h

    def pts(n):
        return lo + rng.uniform(0, 1, size=(n, ndim)) * (hi - lo)

    src = pts(nsrc)
    rec = pts(nrec)
    if random_wavelet:
        wav = rng.standard_normal((nt, nsrc)).astype(np.float32)
    else:
        wav = np.stack([ricker(nt, dt, f0) for _ in range(nsrc)], axis=1)
    pr = Problem(f"rand{ndim}d", ndim, shape, h, space_order, nt, dt,
                 m.astype(np.float32), None if eta is None else eta.astype(np.float32),
                 src.astype(np.float32), wav.astype(np.float32), rec.astype(np.float32),
                 0, nbl)
    if eta is not None:
        pr.sigma = damping_profiles_1d(shape, nbl, h, vmax)
    return pr


# ------------------------------------------------------------------ other paper workloads (f4)
def convection_problem(nx: int = 81, ny: int = 81, nt: int = 100, sigma: float = 0.2, c: float = 1.0):
    """Linear convection example (the CFD tutorial's step 5 it reproduces):
    domain [0, 2]^2, u = 2 on [0.5, 1]^2 and 1 elsewhere, dt = sigma dx.  Returns a dict
    (u0 [nx][ny] float32, c, dt, dx, dy, nt)."""
    dx = 2.0 / (nx - 1)
    dy = 2.0 / (ny - 1)
    x = np.arange(nx) * dx
    y = np.arange(ny) * dy
    u0 = np.ones((nx, ny), dtype=np.float32)
    u0[np.ix_((x >= 0.5) & (x <= 1.0), (y >= 0.5) & (y <= 1.0))] = 2.0
    return {"u0": u0, "c": c, "dt": sigma * dx, "dx": dx, "dy": dy, "nt": nt}


def laplace_problem(nx: int = 31, ny: int = 31):
    """Laplace example (the CFD tutorial's step 9): domain [0, 2] x [0, 1],
    bc = linspace(0, 1, nx), initial p = 0 with the listing's boundary expressions
    applied (figure 'initial condition of pn.data').  Returns a dict (p0, bc, dx, dy)."""
    dx = 2.0 / (nx - 1)
    dy = 1.0 / (ny - 1)
    bc = np.linspace(0.0, 1.0, nx).astype(np.float32)
    p0 = np.zeros((nx, ny), dtype=np.float32)
    p0[:, 0] = 0.0
    p0[:, ny - 1] = bc
    p0[0, :] = p0[1, :]
    p0[nx - 1, :] = p0[nx - 2, :]
    return {"p0": p0, "bc": bc, "dx": dx, "dy": dy}
