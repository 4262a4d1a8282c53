"""ORACLE -- plain fp64 CPU implementation of the acoustic FD path (test infrastructure).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  It never imports the CUDA
product package (``paper_1707_03776_b200``) and shares no code with it.

Thin ctypes wrapper over ``sf_oracle.c`` (see that file's header for what each
function computes and the PAPER.md passages it follows).  ``gradient`` below is
plumbing over ``forward``/``adjoint``: J = 1/2 sum (d_syn - d_obs)^2 (reading C13).

Parity status: every function here is pinned by tests in
``tests/test_oracle_pins.py`` (closed forms, analytic Green's functions,
convergence orders, dot test, Taylor test, invariants).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sf_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile sf_oracle.c -> liboracle.so with gcc (fp64, OpenMP, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-fno-fast-math", "-ffp-contract=off", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i, d = ctypes.c_int, ctypes.c_double
        L.or_fd_weights.argtypes = [i, P]
        L.or_laplacian.argtypes = [i, P, d, i, P, P]
        L.or_point_stencil.argtypes = [i, P, d, P, P, P]
        L.or_interpolate.argtypes = [i, P, d, i, P, P, P]
        L.or_inject.argtypes = [i, P, d, i, P, P, P, d, P]
        L.or_forward.argtypes = [i, P, d, i, i, d, P, P, i, P, P, i, P, P, P, i, P]
        L.or_adjoint.argtypes = [i, P, d, i, i, d, P, P, i, P, P, i, P, P, P, i, P, P]
        L.or_convection2d.argtypes = [P, d, d, d, d, i, P]
        L.or_laplace2d.argtypes = [P, d, d, P, d, i, P, P, P]
        for f in (L.or_fd_weights, L.or_laplacian, L.or_point_stencil, L.or_interpolate,
                  L.or_inject, L.or_forward, L.or_adjoint, L.or_num_threads, L.or_convection2d,
                  L.or_laplace2d):
            f.restype = ctypes.c_int
        _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _shape(shape):
    return np.ascontiguousarray(shape, dtype=np.int64)


def _chk(code, what):
    if code != 0:
        raise OracleError(f"{what} failed with code {code}")


def num_threads() -> int:
    return _load().or_num_threads()


def fd_weights(space_order: int) -> np.ndarray:
    """[w_0, w_1, ..., w_r] of the centred 2nd derivative (times h^2)."""
    w = np.zeros(space_order // 2 + 1)
    _chk(_load().or_fd_weights(space_order, _p(w)), "fd_weights")
    return w


def laplacian(u, h: float, space_order: int) -> np.ndarray:
    u = _f64(u)
    out = np.empty_like(u)
    sh = _shape(u.shape)
    _chk(_load().or_laplacian(u.ndim, _p(sh), h, space_order, _p(u), _p(out)), "laplacian")
    return out


def point_stencil(shape, h: float, coord):
    sh = _shape(shape)
    nd = len(shape)
    idx = np.zeros(1 << nd, dtype=np.int64)
    W = np.zeros(1 << nd)
    c = _f64(coord)
    _chk(_load().or_point_stencil(nd, _p(sh), h, _p(c), _p(idx), _p(W)), "point_stencil")
    return idx, W


def interpolate(coords, u, h: float) -> np.ndarray:
    u = _f64(u)
    c = _f64(coords).reshape(-1, u.ndim)
    out = np.zeros(c.shape[0])
    sh = _shape(u.shape)
    _chk(_load().or_interpolate(u.ndim, _p(sh), h, c.shape[0], _p(c), _p(u), _p(out)),
         "interpolate")
    return out


def inject(coords, vals, u, h: float, m=None, dt: float = 1.0) -> np.ndarray:
    """Return u + P^T(vals * dt^2/m) (or P^T vals when m is None) -- new array."""
    u = _f64(u).copy()
    c = _f64(coords).reshape(-1, u.ndim)
    v = _f64(vals).ravel()
    mm = _f64(m)
    sh = _shape(u.shape)
    _chk(_load().or_inject(u.ndim, _p(sh), h, c.shape[0], _p(c), _p(v), _p(mm), dt, _p(u)),
         "inject")
    return u


def forward(prob=None, *, m=None, damp=None, shape=None, h=None, space_order=None, nt=None,
            dt=None, src_coords=None, wavelet=None, rec_coords=None, u_state=None,
            save_every: int = 0):
    """Forward propagation.  Returns dict(rec [nt][nrec], u_state [2][*shape],
    snaps [nsnap][*shape] or None).  ``prob`` is a synth.Problem; keywords override."""
    if prob is not None:
        m = prob.m if m is None else m
        damp = prob.damp if damp is None else damp
        shape, h = prob.shape, prob.h
        space_order = prob.space_order if space_order is None else space_order
        nt = prob.nt if nt is None else nt
        dt = prob.dt if dt is None else dt
        src_coords = prob.src_coords if src_coords is None else src_coords
        wavelet = prob.wavelet if wavelet is None else wavelet
        rec_coords = prob.rec_coords if rec_coords is None else rec_coords
    shape = tuple(int(s) for s in shape)
    nd = len(shape)
    N = int(np.prod(shape))
    m64, d64 = _f64(m).reshape(shape), _f64(damp)
    sc = _f64(src_coords).reshape(-1, nd) if src_coords is not None else np.zeros((0, nd))
    rc = _f64(rec_coords).reshape(-1, nd) if rec_coords is not None else np.zeros((0, nd))
    nsrc, nrec = sc.shape[0], rc.shape[0]
    wav = _f64(wavelet).reshape(nt, nsrc) if nsrc else np.zeros((nt, 1))
    rec = np.zeros((nt, max(nrec, 1)))
    st = np.zeros((2,) + shape) if u_state is None else _f64(u_state).reshape((2,) + shape).copy()
    snaps = None
    if save_every > 0:
        snaps = np.zeros(((nt - 1) // save_every + 1,) + shape)
    sh = _shape(shape)
    _chk(_load().or_forward(nd, _p(sh), h, space_order, nt, dt, _p(m64), _p(d64),
                            nsrc, _p(sc), _p(wav), nrec, _p(rc), _p(rec), _p(st),
                            save_every, _p(snaps)), "forward")
    del N
    return {"rec": rec[:, :nrec], "u_state": st, "snaps": snaps}


def adjoint(prob=None, *, res=None, m=None, damp=None, shape=None, h=None, space_order=None,
            nt=None, dt=None, src_coords=None, rec_coords=None, v_state=None,
            save_every: int = 0, snaps=None, grad=None):
    """Adjoint propagation: injects ``res`` [nt][nrec] at the receivers,
    interpolates srca [nt][nsrc] at the sources.  If ``snaps`` is given, accumulates
    the gradient (reading C13/C14).  Returns dict(srca, v_state, grad)."""
    if prob is not None:
        m = prob.m if m is None else m
        damp = prob.damp if damp is None else damp
        shape, h = prob.shape, prob.h
        space_order = prob.space_order if space_order is None else space_order
        nt = prob.nt if nt is None else nt
        dt = prob.dt if dt is None else dt
        src_coords = prob.src_coords if src_coords is None else src_coords
        rec_coords = prob.rec_coords if rec_coords is None else rec_coords
    shape = tuple(int(s) for s in shape)
    nd = len(shape)
    m64, d64 = _f64(m).reshape(shape), _f64(damp)
    sc = _f64(src_coords).reshape(-1, nd) if src_coords is not None else np.zeros((0, nd))
    rc = _f64(rec_coords).reshape(-1, nd) if rec_coords is not None else np.zeros((0, nd))
    nsrc, nrec = sc.shape[0], rc.shape[0]
    r64 = _f64(res).reshape(nt, nrec) if nrec else np.zeros((nt, 1))
    srca = np.zeros((nt, max(nsrc, 1)))
    st = np.zeros((2,) + shape) if v_state is None else _f64(v_state).reshape((2,) + shape).copy()
    g = None
    s64 = None
    if snaps is not None:
        s64 = _f64(snaps)
        g = np.zeros(shape) if grad is None else _f64(grad).reshape(shape).copy()
    sh = _shape(shape)
    _chk(_load().or_adjoint(nd, _p(sh), h, space_order, nt, dt, _p(m64), _p(d64),
                            nrec, _p(rc), _p(r64), nsrc, _p(sc), _p(srca), _p(st),
                            save_every, _p(s64), _p(g)), "adjoint")
    return {"srca": srca[:, :nsrc], "v_state": st, "grad": g}


def _snap_round(snaps, snap_dtype):
    if snap_dtype == "float16":
        return snaps.astype(np.float32).astype(np.float16).astype(np.float64)
    if snap_dtype is not None:
        raise ValueError(f"snap_dtype {snap_dtype!r}")
    return snaps


def gradient(prob, d_obs, m=None, save_every: int = 1, snap_dtype=None, checkpoint: int = 0):
    """FWI gradient at model m (default prob.m): forward with snapshots, residual
    res = d_syn - d_obs, J = 1/2 sum res^2, adjoint with correlation (C13/C14).
    snap_dtype='float16': the snapshots are stored in IEEE half precision before the
    correlation (reading C23: u^n -> fp32 -> fp16, round to nearest even at both steps,
    numpy's conversions; widened exactly).  Returns dict(grad, J, res, d_syn, srca).

    checkpoint = S > 0 (a multiple of save_every): checkpoint-recompute (SURVEY §8(c)
    item 4), for runs whose fp64 snapshots do not fit host memory.  The forward runs in
    time windows [c, c + S] (c = 0, S, 2S, ...; the last one ragged), each restarted from
    the state pair (u^{c-1}, u^c) the previous window ended with, which is kept as the
    window's checkpoint; the record rows are the windows' rows (row c of a window is P u^c
    again).  The backward sweep takes the windows last to first: it recomputes the
    window's forward from its checkpoint with snapshots every k (levels c, c+k, ..., all
    in the window because S % k == 0), then runs the adjoint over the same window
    -- adjoint time steps t = c+S .. c+1 on res[c : c+S+1], continuing the (v^{t+1}, v^t)
    pair of the later window -- which adds that window's correlation terms.  Every level,
    record row and gradient term is computed by the same operations as in the stored-
    snapshot run, so the result is bitwise identical (pinned in tests/test_oracle_pins.py).
    Memory: 2 N (nt-1)/S checkpoint floats + N (S/k + 1) snapshot floats."""
    mm = prob.m if m is None else m
    if checkpoint:
        return _gradient_ckpt(prob, d_obs, mm, save_every, snap_dtype, int(checkpoint))
    fw = forward(prob, m=mm, save_every=save_every)
    res = fw["rec"] - _f64(d_obs)
    J = 0.5 * float(np.sum(res * res))
    snaps = _snap_round(fw["snaps"], snap_dtype)
    ad = adjoint(prob, res=res, m=mm, save_every=save_every, snaps=snaps)
    return {"grad": ad["grad"], "J": J, "res": res, "d_syn": fw["rec"], "srca": ad["srca"]}


def _gradient_ckpt(prob, d_obs, mm, k, snap_dtype, S):
    if k < 1 or S < 1 or S % k:
        raise ValueError(f"checkpoint {S} must be a positive multiple of save_every {k}")
    nt = prob.nt
    shape = tuple(int(s) for s in prob.shape)
    nsrc = len(prob.src_coords) if prob.src_coords is not None else 0
    nrec = len(prob.rec_coords) if prob.rec_coords is not None else 0
    wav = _f64(prob.wavelet).reshape(nt, -1) if nsrc else None
    windows = [(c, min(c + S, nt - 1)) for c in range(0, nt - 1, S)]
    # forward sweep: record rows and one checkpoint (u^{c-1}, u^c) per window
    rec = np.zeros((nt, nrec))
    ckpt = []
    st = np.zeros((2,) + shape)
    for c, e in windows:
        ckpt.append(st)
        fw = forward(prob, m=mm, nt=e - c + 1, wavelet=None if wav is None else wav[c:e + 1],
                     u_state=st)
        rec[c:e + 1] = fw["rec"]
        st = fw["u_state"]
    res = rec - _f64(d_obs)
    J = 0.5 * float(np.sum(res * res))
    # backward sweep: recompute each window's snapshots, adjoint over the same window
    grad = np.zeros(shape)
    srca = np.zeros((nt, nsrc))
    vst = np.zeros((2,) + shape)
    for (c, e), st in zip(reversed(windows), reversed(ckpt)):
        L = e - c + 1
        fw = forward(prob, m=mm, nt=L, wavelet=None if wav is None else wav[c:e + 1],
                     u_state=st, save_every=k)
        ad = adjoint(prob, res=res[c:e + 1], m=mm, nt=L, v_state=vst, save_every=k,
                     snaps=_snap_round(fw["snaps"], snap_dtype), grad=grad)
        grad = ad["grad"]
        vst = ad["v_state"]
        srca[c:e + 1] = ad["srca"]
    return {"grad": grad, "J": J, "res": res, "d_syn": rec, "srca": srca}


# ------------------------------------------------------------------ other paper workloads (f4)
def convection2d(u0, *, c: float, dt: float, dx: float, dy: float, nt: int) -> np.ndarray:
    """Linear 2D convection, Eq. 2, nt forward-Euler / upwind steps from u0
    ([n0][n1]); edges keep their initial values (reading C21).  fp64."""
    u = _f64(u0).copy()
    n = _shape(u.shape)
    _chk(_load().or_convection2d(_p(n), float(c), float(dt), float(dx), float(dy), int(nt), _p(u)),
         "or_convection2d")
    return u


def laplace2d(p0, bc, *, dx: float, dy: float, tol: float = 1e-4, max_iter: int = 100000):
    """Laplace equation by Jacobi sweeps, Eq. 4 with the boundary expressions of
    P:411-414 and the l1 stopping rule of P:433-447 (reading C22).  Returns (p, iterations,
    last l1).  fp64."""
    p = _f64(p0).copy()
    n = _shape(p.shape)
    b = _f64(bc)
    it = ctypes.c_int()
    l1 = ctypes.c_double()
    _chk(_load().or_laplace2d(_p(n), float(dx), float(dy), _p(b), float(tol), int(max_iter), _p(p),
                              ctypes.byref(it), ctypes.byref(l1)), "or_laplace2d")
    return p, it.value, l1.value
