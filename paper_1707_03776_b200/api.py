"""Thin Python binding of libsf.so (same names as the C-ABI; marshalling only).

torch is used for device memory and streams; every computation happens in the
library's CUDA kernels.  Arrays:
  * grid arrays: torch.float32 CUDA tensors, contiguous, shape = grid shape
    ([x][y][z], 2D [x][z]); wavefield state u/v: shape (2, *grid);
  * sparse series: (nt, npoint) float32 CUDA tensors (time-major, reading C12);
  * coordinates: host arrays (npoint, ndim), metres from computational index 0.
"""
from __future__ import annotations

import ctypes
import functools
from typing import Optional

import numpy as np
import torch

from ._lib import SfDesc, SfError, check, lib

__all__ = ["Propagator", "fd_weights", "forward_host", "slab_plan", "slab_halo_plan", "sparse_owner", "SfError",
           "nccl_unique_id", "nccl_comm_init", "nccl_comm_destroy", "allreduce_gradient",
           "local_group_create", "local_group_destroy", "convection2d", "laplace2d"]


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _dev(t: torch.Tensor, name: str, shape=None):
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
        raise TypeError(f"{name}: expected a contiguous float32 CUDA tensor")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: shape {tuple(t.shape)} != {tuple(shape)}")
    return t


def fd_weights(space_order: int) -> np.ndarray:
    w = np.zeros(space_order // 2 + 1)
    check(lib().sf_fd_weights(space_order, w.ctypes.data_as(ctypes.c_void_p)))
    return w


def slab_plan(n0: int, space_order: int, rank: int, nranks: int):
    x0, nl = ctypes.c_int64(), ctypes.c_int64()
    check(lib().sf_slab_plan(n0, space_order, rank, nranks, ctypes.byref(x0), ctypes.byref(nl)))
    return x0.value, nl.value


def slab_halo_plan(n0: int, space_order: int, rank: int, nranks: int) -> dict:
    """The per-step halo exchange of a slab rank (sf_slab_halo_plan), in local planes."""
    plan = (ctypes.c_int64 * 7)()
    check(lib().sf_slab_halo_plan(n0, space_order, rank, nranks, plan))
    return {"send_left": plan[0], "recv_left": plan[1], "send_right": plan[2], "recv_right": plan[3],
            "planes": plan[4], "has_left": bool(plan[5]), "has_right": bool(plan[6])}


def sparse_owner(n0: int, space_order: int, nranks: int, h: float, coord0: float) -> int:
    o = ctypes.c_int()
    check(lib().sf_sparse_owner(n0, space_order, nranks, h, coord0, ctypes.byref(o)))
    return o.value


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    check(lib().sf_nccl_unique_id(buf))
    return buf.raw


def nccl_comm_init(uid: bytes, nranks: int, rank: int) -> int:
    c = ctypes.c_void_p()
    check(lib().sf_nccl_comm_init(ctypes.create_string_buffer(uid, 128), nranks, rank, ctypes.byref(c)))
    return c.value


def nccl_comm_destroy(comm: int):
    check(lib().sf_nccl_comm_destroy(ctypes.c_void_p(comm)))


def nccl_comm_info(comm: int):
    """sf_nccl_comm_info: (nranks, rank) of an NCCL communicator."""
    n, r = ctypes.c_int(), ctypes.c_int()
    check(lib().sf_nccl_comm_info(ctypes.c_void_p(comm), ctypes.byref(n), ctypes.byref(r)))
    return n.value, r.value


def nccl_check(comm: int):
    """sf_nccl_check: raises SfError(SF_ERR_NCCL) if the communicator reported an
    asynchronous error."""
    check(lib().sf_nccl_check(ctypes.c_void_p(comm)))


def _ondev(fn):
    """Run a Propagator method with the handle's device current: the library allocates,
    launches and creates streams on the current device."""
    @functools.wraps(fn)
    def w(self, *a, **k):
        with torch.cuda.device(self.device):
            return fn(self, *a, **k)
    return w


class Propagator:
    """One acoustic problem bound to a device handle (sf_create / sf_create_slab).

    ``shape`` is the (global) computational grid.  In slab mode (``comm`` given,
    nranks > 1) ``m``/``damp`` are the rank's local arrays with r halo planes on
    axis 0 ([n0_loc + 2r][n1][n2]) and every wavefield array is local likewise.
    ``sigma``: optional separable damping (sf_desc.sigma) -- one host 1D float32 array per
    axis of the GLOBAL grid, eta = m * (sigma_x + sigma_y (+ sigma_z)); exclusive with damp.
    """

    def __init__(self, m: torch.Tensor, damp: Optional[torch.Tensor], *, shape, h: float,
                 space_order: int, nt: int, dt: float, src_coords=None, rec_coords=None,
                 comm: Optional[int] = None, rank: int = 0, nranks: int = 1, sigma=None):
        self.shape = tuple(int(s) for s in shape)
        self.ndim = len(self.shape)
        self.h, self.space_order, self.nt, self.dt = float(h), int(space_order), int(nt), float(dt)
        self.r = self.space_order // 2
        self.nranks, self.rank = int(nranks), int(rank)
        if self.nranks > 1:
            self.x0, self.n0_loc = slab_plan(self.shape[0], self.space_order, rank, nranks)
            self.local_shape = (self.n0_loc + 2 * self.r,) + self.shape[1:]
        else:
            self.x0, self.n0_loc = 0, self.shape[0]
            self.local_shape = self.shape
        _dev(m, "m", self.local_shape)
        if damp is not None:
            _dev(damp, "damp", self.local_shape)
        self._src = np.zeros((0, self.ndim)) if src_coords is None else \
            np.ascontiguousarray(np.asarray(src_coords, dtype=np.float64).reshape(-1, self.ndim))
        self._rec = np.zeros((0, self.ndim)) if rec_coords is None else \
            np.ascontiguousarray(np.asarray(rec_coords, dtype=np.float64).reshape(-1, self.ndim))
        self.nsrc, self.nrec = self._src.shape[0], self._rec.shape[0]
        d = SfDesc()
        d.ndim = self.ndim
        for a in range(3):
            d.shape[a] = self.shape[a] if a < self.ndim else 1
        d.h, d.space_order, d.nt, d.dt = self.h, self.space_order, self.nt, self.dt
        d.m = m.data_ptr()
        d.damp = damp.data_ptr() if damp is not None else None
        d.nsrc = self.nsrc
        d.src_coords = self._src.ctypes.data if self.nsrc else None
        d.nrec = self.nrec
        d.rec_coords = self._rec.ctypes.data if self.nrec else None
        self._sigma = None
        if sigma is not None:
            self._sigma = [np.ascontiguousarray(np.asarray(sa, dtype=np.float32).reshape(-1)) for sa in sigma]
            if len(self._sigma) != self.ndim or any(sa.size != n for sa, n in zip(self._sigma, self.shape)):
                raise ValueError("sigma: one profile per axis of the global grid")
            for a, sa in enumerate(self._sigma):
                d.sigma[a] = sa.ctypes.data
        self._desc = d
        hnd = ctypes.c_void_p()
        self.device = m.device
        with torch.cuda.device(self.device):
            torch.cuda.synchronize()
            if comm is not None or self.nranks > 1:
                check(lib().sf_create_slab(ctypes.byref(d), ctypes.c_void_p(comm), rank, nranks,
                                           ctypes.byref(hnd)))
            else:
                check(lib().sf_create(ctypes.byref(d), ctypes.byref(hnd)))
        self._h = hnd
        self.snap_dtype = torch.float32

    # -------------------------------------------------------------- lifetime
    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().sf_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -------------------------------------------------------------- helpers
    def nsnap(self, save_every: int) -> int:
        return (self.nt - 1) // save_every + 1

    def _check_snaps(self, snaps: torch.Tensor, save_every: int):
        shape = (self.nsnap(save_every),) + self.local_shape
        if not (isinstance(snaps, torch.Tensor) and snaps.is_cuda and snaps.dtype == self.snap_dtype
                and snaps.is_contiguous() and tuple(snaps.shape) == shape):
            raise TypeError(f"snaps: expected a contiguous {self.snap_dtype} CUDA tensor of shape {shape}")

    def zeros_state(self):
        return torch.zeros((2,) + self.local_shape, device=self.device, dtype=torch.float32)

    @_ondev
    def set_tuning(self, variant: int = 0, vy: int = 0, ctas: int = 0):
        """sf_set_tuning: variant (0 auto, 1 generic, 2 TMA), rows per thread (0 auto, 1, 2),
        persistent CTAs (0 = one per SM)."""
        check(lib().sf_set_tuning(self._h, variant, vy, ctas))

    @_ondev
    def set_option(self, option: int, value: int):
        """sf_set_option: 1 L2 prefetch distance, 2 split boundary launches, 3 fuse-max points,
        4 SMs left free by the split interior launch, 5 CUDA-graph replay of whole calls,
        7 fp16 snapshots, 8 peer-store halo exchange in slab mode."""
        check(lib().sf_set_option(self._h, int(option), int(value)))
        if int(option) == 7:
            self.snap_dtype = torch.float16 if value else torch.float32

    @_ondev
    def tuning(self):
        v, b, c = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        check(lib().sf_get_tuning(self._h, ctypes.byref(v), ctypes.byref(b), ctypes.byref(c)))
        out = {"variant": v.value, "vy": b.value, "ctas": c.value}
        g, b0, b1 = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        if hasattr(lib(), "sf_get_tuning_modes"):  # (A/B builds of older revisions lack it)
            check(lib().sf_get_tuning_modes(self._h, ctypes.byref(g), ctypes.byref(b0), ctypes.byref(b1)))
            out.update(vy_grad=g.value, balance=b0.value, balance_grad=b1.value)
        return out

    @_ondev
    def set_profiling(self, on: bool = True):
        check(lib().sf_set_profiling(self._h, 1 if on else 0))

    @_ondev
    def autotune(self, steps: int = 8, stream=None) -> dict:
        """sf_autotune: time every feasible launch configuration on a scratch state and keep
        the fastest (same bits either way; GRAD-mode steps get their own layout, tuning()
        reports it as vy_grad).  Returns {variant, vy, zsplit, ms_per_step}."""
        u = torch.zeros((2,) + self.local_shape, device=self.device)
        ch = (ctypes.c_int * 3)()
        ms = ctypes.c_float()
        check(lib().sf_autotune(self._h, _ptr(u), int(steps), ch, ctypes.byref(ms), _stream(stream)))
        return {"variant": ch[0], "vy": ch[1], "zsplit": ch[2], "ms_per_step": ms.value}

    @_ondev
    def debug_probe(self, dst: Optional[torch.Tensor]) -> int:
        """sf_debug_probe: set (or clear) the one-launch test probe buffer; returns the
        number of steps run with the one-launch schedule so far."""
        n = ctypes.c_longlong()
        check(lib().sf_debug_probe(self._h, _ptr(dst) if dst is not None else None, ctypes.byref(n)))
        return n.value

    @_ondev
    def profile(self, reset: bool = True):
        """Summed in-stream kernel times (CUDA events) and launch counts since the last
        reset, by kind: stencil / inject / interp / other."""
        ms = (ctypes.c_double * 4)()
        cnt = (ctypes.c_longlong * 4)()
        check(lib().sf_get_profile_detail(self._h, ms, cnt, 1 if reset else 0))
        kinds = ("stencil", "inject", "interp", "other")
        out = {f"{k}_ms": ms[i] for i, k in enumerate(kinds)}
        out.update({f"{k}_launches": cnt[i] for i, k in enumerate(kinds)})
        out["launches"] = sum(cnt)
        return out

    # -------------------------------------------------------------- the path
    @_ondev
    def forward(self, wavelet: Optional[torch.Tensor], *, u: Optional[torch.Tensor] = None,
                rec: Optional[torch.Tensor] = None, save_every: int = 0,
                snaps: Optional[torch.Tensor] = None, stream=None):
        """sf_forward.  Returns (rec [nt][nrec], u (u^{nt-2}, u^{nt-1}), snaps)."""
        if self.nsrc:
            _dev(wavelet, "wavelet", (self.nt, self.nsrc))
        u = self.zeros_state() if u is None else _dev(u, "u", (2,) + self.local_shape)
        if self.nrec:
            rec = torch.empty((self.nt, self.nrec), device=self.device) if rec is None else \
                _dev(rec, "rec", (self.nt, self.nrec))
        else:
            rec = None
        if save_every > 0 and snaps is None:
            snaps = torch.empty((self.nsnap(save_every),) + self.local_shape, device=self.device,
                                dtype=self.snap_dtype)
        if snaps is not None:
            self._check_snaps(snaps, save_every)
        check(lib().sf_forward(self._h, _ptr(wavelet) if self.nsrc else None, _ptr(rec), _ptr(u),
                               _ptr(snaps), int(save_every), _stream(stream)))
        return rec, u, snaps

    @_ondev
    def adjoint(self, res: Optional[torch.Tensor], *, v: Optional[torch.Tensor] = None,
                srca: Optional[torch.Tensor] = None, snaps: Optional[torch.Tensor] = None,
                save_every: int = 0, grad: Optional[torch.Tensor] = None, stream=None):
        """sf_adjoint.  Returns (srca [nt][nsrc], v (v^1, v^0), grad)."""
        if self.nrec:
            _dev(res, "res", (self.nt, self.nrec))
        v = self.zeros_state() if v is None else _dev(v, "v", (2,) + self.local_shape)
        if self.nsrc:
            srca = torch.empty((self.nt, self.nsrc), device=self.device) if srca is None else \
                _dev(srca, "srca", (self.nt, self.nsrc))
        else:
            srca = None
        if snaps is not None:
            self._check_snaps(snaps, save_every)
            if grad is None:
                grad = torch.zeros(self.local_shape, device=self.device)
        if grad is not None:
            _dev(grad, "grad", self.local_shape)
        check(lib().sf_adjoint(self._h, _ptr(res) if self.nrec else None, _ptr(srca), _ptr(v),
                               _ptr(snaps), int(save_every), _ptr(grad), _stream(stream)))
        return srca, v, grad

    @_ondev
    def residual(self, d_syn: torch.Tensor, d_obs: torch.Tensor, res: Optional[torch.Tensor] = None,
                 stream=None):
        _dev(d_syn, "d_syn", (self.nt, self.nrec))
        _dev(d_obs, "d_obs", (self.nt, self.nrec))
        res = torch.empty_like(d_syn) if res is None else _dev(res, "res", (self.nt, self.nrec))
        J = ctypes.c_double()
        check(lib().sf_residual(self._h, _ptr(d_syn), _ptr(d_obs), _ptr(res), ctypes.byref(J),
                                _stream(stream)))
        return res, J.value

    def gradient_workspace_bytes(self, save_every: int) -> int:
        return int(lib().sf_gradient_workspace_bytes(self._h, int(save_every)))

    @_ondev
    def gradient(self, wavelet: torch.Tensor, d_obs: torch.Tensor, *, save_every: int = 1,
                 grad: Optional[torch.Tensor] = None, ws: Optional[torch.Tensor] = None, stream=None):
        """sf_gradient: returns (grad [local grid], J)."""
        _dev(d_obs, "d_obs", (self.nt, self.nrec))
        if self.nsrc:
            _dev(wavelet, "wavelet", (self.nt, self.nsrc))
        nbytes = self.gradient_workspace_bytes(save_every)
        if ws is None or ws.numel() * ws.element_size() < nbytes:
            ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        grad = torch.empty(self.local_shape, device=self.device) if grad is None else \
            _dev(grad, "grad", self.local_shape)
        J = ctypes.c_double()
        check(lib().sf_gradient(self._h, _ptr(wavelet) if self.nsrc else None, _ptr(d_obs), _ptr(grad),
                                ctypes.byref(J), ctypes.c_void_p(ws.data_ptr()), nbytes,
                                int(save_every), _stream(stream)))
        return grad, J.value

    def gradient_ckpt_workspace_bytes(self, save_every: int, segment: int) -> int:
        return int(lib().sf_gradient_ckpt_workspace_bytes(self._h, int(save_every), int(segment)))

    @_ondev
    def gradient_ckpt(self, wavelet: torch.Tensor, d_obs: torch.Tensor, *, save_every: int = 1,
                      segment: int, grad: Optional[torch.Tensor] = None, ws: Optional[torch.Tensor] = None,
                      stream=None):
        """sf_gradient_ckpt (checkpoint-recompute, `segment` steps per checkpoint): returns
        (grad, J), bitwise equal to gradient()."""
        _dev(d_obs, "d_obs", (self.nt, self.nrec))
        if self.nsrc:
            _dev(wavelet, "wavelet", (self.nt, self.nsrc))
        nbytes = self.gradient_ckpt_workspace_bytes(save_every, segment)
        if nbytes == 0:
            raise ValueError("segment must be a positive multiple of save_every")
        if ws is None or ws.numel() * ws.element_size() < nbytes:
            ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        grad = torch.empty(self.local_shape, device=self.device) if grad is None else \
            _dev(grad, "grad", self.local_shape)
        J = ctypes.c_double()
        check(lib().sf_gradient_ckpt(self._h, _ptr(wavelet) if self.nsrc else None, _ptr(d_obs), _ptr(grad),
                                     ctypes.byref(J), ctypes.c_void_p(ws.data_ptr()), nbytes,
                                     int(save_every), int(segment), _stream(stream)))
        return grad, J.value

    @_ondev
    def allreduce_gradient(self, comm: int, grad: torch.Tensor, J: Optional[float] = None, rank: int = 0,
                           stream=None):
        return allreduce_gradient(comm, grad, J, handle=self, rank=rank, stream=stream)


def allreduce_gradient(comm: int, grad: torch.Tensor, J: Optional[float] = None, handle=None,
                       rank: int = 0, stream=None):
    """sf_allreduce_gradient: in-place sum of grad (and J) over the communicator (NCCL or
    a local group; `rank` = the caller's rank, needed by the local group only)."""
    _dev(grad, "grad")
    Jc = ctypes.c_double(0.0 if J is None else J)
    check(lib().sf_allreduce_gradient(handle._h if handle is not None else None, ctypes.c_void_p(comm),
                                      _ptr(grad), grad.numel(),
                                      ctypes.byref(Jc) if J is not None else None, int(rank),
                                      _stream(stream)))
    return grad, (Jc.value if J is not None else None)


def local_group_create(nranks: int) -> int:
    """sf_local_group_create: an in-process transport for `nranks` rank threads on one device
    (testing the slab / multi-shot paths without NCCL); pass it as `comm`."""
    g = ctypes.c_void_p()
    check(lib().sf_local_group_create(int(nranks), ctypes.byref(g)))
    return g.value


def local_group_destroy(group: int):
    check(lib().sf_local_group_destroy(ctypes.c_void_p(group)))


def forward_host(m: np.ndarray, damp: Optional[np.ndarray], *, h: float, space_order: int, nt: int,
                 dt: float, src_coords, wavelet: np.ndarray, rec_coords, rec_out: Optional[np.ndarray] = None,
                 u_out: Optional[np.ndarray] = None, stream=None, sigma=None) -> np.ndarray:
    """sf_forward_host: end-to-end forward with HOST (numpy / pinned) buffers."""
    shape = m.shape
    nd = len(shape)
    src = np.ascontiguousarray(np.asarray(src_coords, np.float64).reshape(-1, nd))
    rec = np.ascontiguousarray(np.asarray(rec_coords, np.float64).reshape(-1, nd))
    d = SfDesc()
    d.ndim = nd
    for a in range(3):
        d.shape[a] = shape[a] if a < nd else 1
    d.h, d.space_order, d.nt, d.dt = h, space_order, nt, dt
    assert m.dtype == np.float32 and m.flags.c_contiguous
    d.m = m.ctypes.data
    if damp is not None:
        assert damp.dtype == np.float32 and damp.flags.c_contiguous
        d.damp = damp.ctypes.data
    d.nsrc, d.src_coords = src.shape[0], src.ctypes.data if src.shape[0] else None
    d.nrec, d.rec_coords = rec.shape[0], rec.ctypes.data if rec.shape[0] else None
    sig = None
    if sigma is not None:
        sig = [np.ascontiguousarray(np.asarray(sa, dtype=np.float32).reshape(-1)) for sa in sigma]
        for a, sa in enumerate(sig):
            d.sigma[a] = sa.ctypes.data
    wav = np.ascontiguousarray(wavelet, dtype=np.float32)
    if rec_out is None:
        rec_out = np.empty((nt, rec.shape[0]), np.float32)
    check(lib().sf_forward_host(ctypes.byref(d), wav.ctypes.data_as(ctypes.c_void_p),
                                rec_out.ctypes.data_as(ctypes.c_void_p),
                                None if u_out is None else u_out.ctypes.data_as(ctypes.c_void_p),
                                _stream(stream)))
    return rec_out


# ------------------------------------------------------------------ other paper workloads (f4)
def convection2d(u: torch.Tensor, *, c: float, dt: float, dx: float, dy: float, nt: int, stream=None):
    """sf_convection2d: nt steps of Eq. 2 on the device [n0][n1] tensor u, in place."""
    _dev(u, "u")
    if u.dim() != 2:
        raise ValueError("u: expected a 2D [n0][n1] tensor")
    work = None if u.numel() <= 25600 else torch.empty_like(u)
    check(lib().sf_convection2d(_ptr(u), _ptr(work), u.shape[0], u.shape[1], float(c), float(dt), float(dx),
                                float(dy), int(nt), _stream(stream)))
    return u


def laplace2d(p: torch.Tensor, bc: torch.Tensor, *, dx: float, dy: float, tol: float = 1e-4,
              max_iter: int = 100000, stream=None):
    """sf_laplace2d: Jacobi sweeps of Eq. 4 with the P:411-414 boundary rows until the l1 rule
    of P:433-447 holds; p (device [n0][n1]) in place.  Returns (p, sweeps, last l1)."""
    _dev(p, "p")
    _dev(bc, "bc", (p.shape[0],))
    work = None if p.numel() <= 4096 else torch.empty_like(p)
    it, l1 = ctypes.c_int(), ctypes.c_double()
    check(lib().sf_laplace2d(_ptr(p), _ptr(work), _ptr(bc), p.shape[0], p.shape[1], float(dx), float(dy),
                             float(tol), int(max_iter), ctypes.byref(it), ctypes.byref(l1), _stream(stream)))
    return p, it.value, l1.value
