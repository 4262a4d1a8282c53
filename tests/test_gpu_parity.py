"""GPU parity: the CUDA path (through the C-ABI) vs the fp64 oracle on the same seeded
inputs.  Tolerance: relative L2 <= 1e-4 on records, final wavefields and gradients
(BASELINE north_star); bitwise where the operation is exact (integer/index work,
zero-in/zero-out, constant preservation, determinism, variant equivalence).
"""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-4


def sf():
    import paper_1707_03776_b200 as m
    return m


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def make_prop(p, m=None, **kw):
    m = p.m if m is None else m
    return sf().Propagator(dev(m), None if p.damp is None else dev(p.damp), shape=p.shape, h=p.h,
                           space_order=p.space_order, nt=p.nt, dt=p.dt,
                           src_coords=p.src_coords.astype(np.float64),
                           rec_coords=p.rec_coords.astype(np.float64), **kw)


def gpu_forward(p, variant=0, ctas=0, vy=0, save_every=0, wavelet=None):
    prop = make_prop(p)
    prop.set_tuning(variant, vy, ctas)
    rec, u, snaps = prop.forward(dev(p.wavelet if wavelet is None else wavelet), save_every=save_every)
    torch.cuda.synchronize()
    out = (rec.cpu().numpy(), u.cpu().numpy(), None if snaps is None else snaps.cpu().numpy())
    prop.close()
    return out


def oracle_forward(p, save_every=0, wavelet=None):
    o = oracle.forward(p, save_every=save_every, wavelet=wavelet)
    return o["rec"], o["u_state"], o["snaps"]


# ------------------------------------------------------------------- forward parity
@pytest.mark.parametrize("so", [2, 4, 6, 8, 10, 12, 14, 16])
def test_forward_3d_all_orders_both_variants(so):
    """3D, damping on, ragged tiles in every axis (n2 = 132: one full + one partial
    128-column tile; n1 = 45: ragged 14- and 7-row tiles; 37 planes).  The persistent TMA
    kernel runs with one CTA per SM and with 1, 3 and 7 CTAs, so that CTA runs start and
    end mid-column and span several tile columns (segments)."""
    p = synth.random_problem(3, (37, 45, 132), so, 60, seed=so, nbl=6, nsrc=2, nrec=9)
    ro, uo, _ = oracle_forward(p)
    results = {}
    for variant, vy, ctas in ((1, 0, 0), (2, 2, 0), (2, 2, 1), (2, 2, 3), (2, 2, 7), (2, 1, 0), (2, 1, 5)):
        rg, ug, _ = gpu_forward(p, variant=variant, vy=vy, ctas=ctas)
        assert rel(rg, ro) <= TOL, (variant, vy, ctas, rel(rg, ro))
        assert rel(ug[1], uo[1]) <= TOL and rel(ug[0], uo[0]) <= TOL
        results[(variant, vy, ctas)] = (rg, ug)
    # every variant evaluates the same per-point expression in the same order: identical bits
    base = results[(1, 0, 0)]
    for k, v in results.items():
        assert np.array_equal(v[0], base[0]) and np.array_equal(v[1], base[1]), k


@pytest.mark.parametrize("vy", [1, 2])
def test_forward_3d_tma_rows_per_thread(vy):
    p = synth.random_problem(3, (30, 50, 64), 8, 40, seed=7, nbl=5)
    ro, uo, _ = oracle_forward(p)
    rg, ug, _ = gpu_forward(p, variant=2, vy=vy, ctas=2)
    assert rel(rg, ro) <= TOL and rel(ug[1], uo[1]) <= TOL


def test_forward_3d_generic_when_n2_not_multiple_of_4():
    p = synth.random_problem(3, (21, 23, 27), 4, 50, seed=3, nbl=4)
    prop = make_prop(p)
    assert prop.tuning()["variant"] == 1
    prop.close()
    ro, uo, _ = oracle_forward(p)
    rg, ug, _ = gpu_forward(p)
    assert rel(rg, ro) <= TOL and rel(ug[1], uo[1]) <= TOL


@pytest.mark.parametrize("so", [2, 4, 8, 16])
def test_forward_2d(so):
    p = synth.random_problem(2, (61, 47), so, 150, seed=so + 1, nbl=8, nsrc=2, nrec=11)
    ro, uo, _ = oracle_forward(p)
    rg, ug, _ = gpu_forward(p)
    assert rel(rg, ro) <= TOL and rel(ug[1], uo[1]) <= TOL and rel(ug[0], uo[0]) <= TOL


def test_config0_full_size_vs_oracle_and_green():
    """BASELINE configs[0] at its full size (141^2 comp grid, so4, nt=500)."""
    p = synth.make_config(0)
    ro, uo, _ = oracle_forward(p)
    rg, ug, _ = gpu_forward(p)
    assert rel(rg, ro) <= TOL
    assert rel(ug[1], uo[1]) <= TOL


def test_config1_reduced_vs_oracle():
    """configs[1] structure (two layers, 40-pt layer scaled, surface receiver grid,
    source off-node at the surface centre) at scale 1/4: 84^3, nt 250."""
    p = synth.make_config(1, scale=0.25, nt=250)
    ro, uo, _ = oracle_forward(p)
    rg, ug, _ = gpu_forward(p)
    assert rel(rg, ro) <= TOL and rel(ug[1], uo[1]) <= TOL


def test_config1_full_grid_short_run_bench_launch():
    """configs[1] at its FULL grid (336^3, so8, damping) in the launch configuration
    bench.py times (auto tuning: TMA variant), short record (nt = 24) so the oracle
    finishes; every receiver row and both final levels compared."""
    p = synth.make_config(1, nt=24)
    prop = make_prop(p)
    assert prop.tuning()["variant"] == 2
    prop.close()
    ro, uo, _ = oracle_forward(p)
    rg, ug, _ = gpu_forward(p)
    assert rel(rg, ro) <= TOL
    assert rel(ug[1], uo[1]) <= TOL and rel(ug[0], uo[0]) <= TOL


def test_config3_full_grid_restart_bench_launch():
    """configs[3] at its FULL grid (1024 x 512 x 512, so16, no damping layer, 8-layer model)
    in the launch configuration bench.py times (persistent TMA kernel), restarted from a
    seeded random state so that every point of the grid -- tile edges, ragged 14-row tiles,
    chunk boundaries, the zero halo on all six faces -- carries signal; nt = 6 so the fp64
    oracle finishes.  Records and both final levels compared over the whole grid."""
    p = synth.make_config(3, nt=6)
    rng = np.random.default_rng(33)
    u0 = rng.standard_normal((2,) + tuple(p.shape), dtype=np.float32) * np.float32(1e-3)
    o = oracle.forward(p, u_state=u0)
    prop = make_prop(p)
    assert prop.tuning()["variant"] == 2
    u = dev(u0)
    rec, u, _ = prop.forward(dev(p.wavelet), u=u)
    torch.cuda.synchronize()
    rg, ug = rec.cpu().numpy(), u.cpu().numpy()
    prop.close()
    assert rel(rg, o["rec"]) <= TOL, rel(rg, o["rec"])
    assert rel(ug[1], o["u_state"][1]) <= TOL and rel(ug[0], o["u_state"][0]) <= TOL


def test_config4_full_grid_short_gradient():
    """configs[4] (one shot) at its FULL grid (400^3, so12, no damping, layered model +
    3 anomalies, 400 x 400 surface receivers incl. the clamped last node, save every 3) in
    the bench launch configuration; short record nt = 12, observed data from a 15 %
    perturbed model (well-conditioned residual)."""
    p = synth.make_config(4, nt=12)
    d_obs = oracle.forward(p, m=(p.m * 0.85).astype(np.float32))["rec"].astype(np.float32)
    go = oracle.gradient(p, d_obs, save_every=3)
    prop = make_prop(p)
    g, J = prop.gradient(dev(p.wavelet), dev(d_obs), save_every=3)
    torch.cuda.synchronize()
    prop.close()
    assert rel(g.cpu().numpy(), go["grad"]) <= TOL, rel(g.cpu().numpy(), go["grad"])
    assert abs(J - go["J"]) <= 1e-4 * go["J"]


def test_config3_shape_so16_no_damping_reduced():
    """configs[3] structure (so16, no damping layer, layered model) at scale 1/8."""
    p = synth.make_config(3, scale=0.125, nt=80)
    ro, uo, _ = oracle_forward(p)
    rg, ug, _ = gpu_forward(p)
    assert rel(rg, ro) <= TOL and rel(ug[1], uo[1]) <= TOL


# ------------------------------------------------------------------- snapshots / adjoint
def test_forward_snapshots():
    p = synth.random_problem(3, (26, 30, 64), 8, 41, seed=9, nbl=5)
    ro, uo, so_ = oracle_forward(p, save_every=4)
    rg, ug, sg = gpu_forward(p, save_every=4)
    assert sg.shape == so_.shape
    assert np.all(sg[0] == 0)
    for k in range(1, sg.shape[0]):
        assert rel(sg[k], so_[k]) <= TOL, k


@pytest.mark.parametrize("ndim,shape,so", [(2, (51, 44), 4), (3, (28, 26, 64), 8), (3, (24, 22, 20), 6),
                                         (3, (30, 28, 144), 12), (3, (26, 24, 64), 16)])
def test_adjoint_parity(ndim, shape, so):
    p = synth.random_problem(ndim, shape, so, 70, seed=21, nbl=5, nsrc=2, nrec=8)
    res = np.random.default_rng(1).standard_normal((p.nt, 8)).astype(np.float32)
    ad = oracle.adjoint(p, res=res)
    prop = make_prop(p)
    srca, v, _ = prop.adjoint(dev(res))
    torch.cuda.synchronize()
    assert rel(srca.cpu().numpy(), ad["srca"]) <= TOL
    assert rel(v.cpu().numpy()[1], ad["v_state"][1]) <= TOL


@pytest.mark.parametrize("ndim,shape,so", [(2, (45, 41), 4), (3, (30, 28, 64), 8)])
def test_dot_product_gpu_fp32(ndim, shape, so):
    """<F x, y> = <x, F^T y> for the fp32 GPU operators: <= 1e-4."""
    p = synth.random_problem(ndim, shape, so, 90, seed=4, nbl=6, nsrc=2, nrec=7, random_wavelet=True)
    rng = np.random.default_rng(8)
    y = rng.standard_normal((p.nt, 7)).astype(np.float32)
    prop = make_prop(p)
    rec, _, _ = prop.forward(dev(p.wavelet))
    srca, _, _ = prop.adjoint(dev(y))
    torch.cuda.synchronize()
    a = float(np.sum(rec.cpu().numpy().astype(np.float64) * y))
    b = float(np.sum(p.wavelet.astype(np.float64) * srca.cpu().numpy()))
    assert abs(a - b) / abs(a) <= 1e-4


# ------------------------------------------------------------------- gradient
def _grad_problem(ndim=3):
    if ndim == 3:
        p = synth.make_config(2, scale=0.125, nt=120)   # 32^3 + 5-pt layer, 5 layers + anomaly
    else:
        p = synth.random_problem(2, (50, 44), 4, 150, seed=2, nbl=6, nsrc=1, nrec=12)
        p.m_true = (p.m * 0.97).astype(np.float32)
    d_obs = oracle.forward(p, m=p.m_true)["rec"].astype(np.float32)
    return p, d_obs


@pytest.mark.parametrize("k", [1, 3, 4])
def test_gradient_parity_3d(k):
    p, d_obs = _grad_problem(3)
    go = oracle.gradient(p, d_obs, save_every=k)
    prop = make_prop(p)
    g, J = prop.gradient(dev(p.wavelet), dev(d_obs), save_every=k)
    torch.cuda.synchronize()
    assert rel(g.cpu().numpy(), go["grad"]) <= TOL, rel(g.cpu().numpy(), go["grad"])
    assert abs(J - go["J"]) <= 1e-4 * go["J"]


def test_gradient_parity_2d_and_components():
    p, d_obs = _grad_problem(2)
    go = oracle.gradient(p, d_obs, save_every=2)
    prop = make_prop(p)
    # component calls: forward with snapshots, residual, adjoint with correlation
    rec, _, snaps = prop.forward(dev(p.wavelet), save_every=2)
    res, J = prop.residual(rec, dev(d_obs))
    _, _, g = prop.adjoint(res, snaps=snaps, save_every=2)
    torch.cuda.synchronize()
    assert rel(res.cpu().numpy(), go["res"]) <= TOL
    assert rel(g.cpu().numpy(), go["grad"]) <= TOL
    g2, J2 = prop.gradient(dev(p.wavelet), dev(d_obs), save_every=2)
    assert np.array_equal(g2.cpu().numpy(), g.cpu().numpy()) and J2 == J


def test_residual_objective_fp64():
    p = synth.random_problem(2, (20, 20), 4, 300, seed=1, nbl=0, nrec=50, damp=False)
    prop = make_prop(p)
    rng = np.random.default_rng(0)
    a = rng.standard_normal((300, 50)).astype(np.float32)
    b = rng.standard_normal((300, 50)).astype(np.float32)
    res, J = prop.residual(dev(a), dev(b))
    r = (a - b).astype(np.float64)   # the kernel squares the fp32 residual in fp64
    assert np.array_equal(res.cpu().numpy(), (a - b))
    assert abs(J - 0.5 * np.sum(r * r)) <= 1e-12 * J


# ------------------------------------------------------------------- invariants / edges
def test_zero_in_zero_out_and_determinism():
    p = synth.make_config(1, scale=0.25, nt=60)
    rg, ug, _ = gpu_forward(p, wavelet=np.zeros_like(p.wavelet))
    assert not rg.any() and not ug.any()
    a = gpu_forward(p)
    b = gpu_forward(p)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_constant_preserved_bitwise_interior():
    """eta = 0, no source: a constant field is annihilated exactly by the difference-form
    Laplacian (reading C15) -> bitwise constant away from the zero halo."""
    n, so, nt = 40, 8, 5
    p = synth.random_problem(3, (n, n, 64), so, nt, seed=3, nbl=0, damp=False)
    prop = make_prop(p)
    u0 = torch.full((2, n, n, 64), 0.7311, device="cuda")
    _, u, _ = prop.forward(torch.zeros((nt, 2), device="cuda"), u=u0)
    k = (so // 2) * nt
    core = u.cpu().numpy()[1][k:-k, k:-k, k:-k]
    assert np.all(core == np.float32(0.7311))


def test_single_step_and_no_sparse_points():
    p = synth.random_problem(3, (20, 21, 32), 4, 2, seed=5, nbl=0)
    ro, uo, _ = oracle_forward(p)
    rg, ug, _ = gpu_forward(p)
    assert rel(rg, ro) <= TOL and rel(ug[1], uo[1]) <= TOL
    # no sources, no receivers, nonzero initial state
    st = np.random.default_rng(2).standard_normal((2, 20, 21, 32)).astype(np.float32)
    o = oracle.forward(m=p.m, damp=p.damp, shape=p.shape, h=p.h, space_order=4, nt=9, dt=p.dt,
                       src_coords=None, wavelet=None, rec_coords=None, u_state=st)
    prop = sf().Propagator(dev(p.m), None if p.damp is None else dev(p.damp), shape=p.shape, h=p.h,
                           space_order=4, nt=9, dt=p.dt)
    _, u, _ = prop.forward(None, u=dev(st))
    assert rel(u.cpu().numpy(), o["u_state"]) <= TOL


def test_receivers_on_last_node_clamp():
    p = synth.random_problem(3, (16, 18, 20), 4, 30, seed=6, nbl=0)
    n = np.array(p.shape)
    p.rec_coords = np.array([(n - 1) * p.h, [0.0, 0.0, 0.0], [(n[0] - 1) * p.h, 0.0, 3.5 * p.h]],
                            dtype=np.float32)
    ro, _, _ = oracle_forward(p)
    rg, _, _ = gpu_forward(p)
    assert rel(rg, ro) <= TOL


def test_errors():
    p = synth.random_problem(3, (16, 16, 16), 4, 10, seed=0, nbl=0)
    S = sf()
    with pytest.raises(S.SfError) as e:
        S.Propagator(dev(p.m), None, shape=p.shape, h=p.h, space_order=4, nt=10, dt=p.dt,
                     rec_coords=np.array([[0.0, 0.0, 15.01 * p.h]]))
    assert e.value.status == "SF_ERR_OUT_OF_DOMAIN"
    with pytest.raises(S.SfError) as e:
        S.Propagator(dev(p.m), None, shape=p.shape, h=p.h, space_order=4, nt=10, dt=p.dt * 2.0)
    assert e.value.status == "SF_ERR_CFL"
    with pytest.raises(S.SfError) as e:
        S.Propagator(dev(p.m), None, shape=p.shape, h=p.h, space_order=5, nt=10, dt=p.dt)
    assert e.value.status == "SF_ERR_ORDER"
    bad = p.m.copy()
    bad[3, 3, 3] = -1.0
    with pytest.raises(S.SfError) as e:
        S.Propagator(dev(bad), None, shape=p.shape, h=p.h, space_order=4, nt=10, dt=p.dt)
    assert e.value.status == "SF_ERR_INVALID_ARG"


def test_forward_host_matches_device():
    p = synth.make_config(1, scale=0.2, nt=50)
    rg, ug, _ = gpu_forward(p)
    u = np.empty((2,) + p.shape, np.float32)
    rh = sf().forward_host(p.m, p.damp, h=p.h, space_order=p.space_order, nt=p.nt, dt=p.dt,
                           src_coords=p.src_coords, wavelet=p.wavelet, rec_coords=p.rec_coords,
                           u_out=u)
    assert np.array_equal(rh, rg) and np.array_equal(u, ug)


def test_profiling_counts():
    p = synth.make_config(1, scale=0.2, nt=30)
    prop = make_prop(p)
    prop.set_profiling(True)
    prop.forward(dev(p.wavelet))
    prof = prop.profile()
    assert prof["stencil_launches"] == p.nt - 1 and prof["stencil_ms"] > 0 and prof["interp_launches"] >= 1
    assert prof["launches"] >= p.nt - 1


@pytest.mark.parametrize("k", [1, 4])
def test_gradient_parity_tma_variant(k):
    """Gradient through the TMA kernel's fused GRAD mode (n2 % 4 == 0), damping on."""
    p = synth.random_problem(3, (30, 28, 64), 8, 100, seed=12, nbl=5, nsrc=1, nrec=20)
    rng = np.random.default_rng(3)
    p.m_true = (p.m * rng.uniform(0.9, 1.1, p.m.shape)).astype(np.float32)
    d_obs = oracle.forward(p, m=p.m_true)["rec"].astype(np.float32)
    go = oracle.gradient(p, d_obs, save_every=k)
    prop = make_prop(p)
    assert prop.tuning()["variant"] == 2
    g, J = prop.gradient(dev(p.wavelet), dev(d_obs), save_every=k)
    torch.cuda.synchronize()
    assert rel(g.cpu().numpy(), go["grad"]) <= TOL, rel(g.cpu().numpy(), go["grad"])
    assert abs(J - go["J"]) <= 1e-4 * go["J"]
    # generic variant: identical bits
    prop.set_tuning(1, 0, 0)
    g1, J1 = prop.gradient(dev(p.wavelet), dev(d_obs), save_every=k)
    assert np.array_equal(g1.cpu().numpy(), g.cpu().numpy()) and J1 == J


def test_config2_full_grid_short_gradient():
    """configs[2] at its FULL grid (336^3: true = 5 layers + anomaly, init = smoothed,
    damping), save every 4, in the bench launch configuration; short record nt = 64.
    Observed data come from a uniformly 15 % perturbed model so that the residual is
    well conditioned (|res| ~ |d|) within the short record."""
    p = synth.make_config(2, nt=64)
    d_obs = oracle.forward(p, m=(p.m * 0.85).astype(np.float32))["rec"].astype(np.float32)
    go = oracle.gradient(p, d_obs, save_every=4)
    prop = make_prop(p)
    g, J = prop.gradient(dev(p.wavelet), dev(d_obs), save_every=4)
    torch.cuda.synchronize()
    assert rel(g.cpu().numpy(), go["grad"]) <= TOL, rel(g.cpu().numpy(), go["grad"])
    assert abs(J - go["J"]) <= 1e-4 * go["J"]


def test_fused_sparse_epilogue_mixed_receivers():
    """TMA kernel's fused injection + interpolation epilogue: on-node surface receivers
    (fused), receivers straddling planes/tiles (left to k_interp_list) and sources on
    tile boundaries -- vs the oracle and bitwise vs the generic (unfused) variant."""
    p = synth.make_config(1, scale=0.25, nt=90)
    rng = np.random.default_rng(5)
    n = np.array(p.shape)
    extra = rng.uniform(0.5, 1.0, (40, 3)) * (n - 1) * p.h * 0.9
    extra[:5, 1] = 15.5 * p.h          # y straddles the BY=16 tile boundary
    extra[5:10, 2] = 127.5 * p.h if n[2] > 128 else extra[5:10, 2]
    # <= 256 points so the TMA kernel interpolates them in-kernel (SF_FUSE_MAX)
    p.rec_coords = np.concatenate([p.rec_coords[::71][:100], extra.astype(np.float32)])
    p.src_coords = np.array([[40.0 * p.h, 16.0 * p.h, 40.3 * p.h], [20.5 * p.h, 31.5 * p.h, 60.0 * p.h]],
                            dtype=np.float32)
    p.wavelet = np.stack([p.wavelet[:, 0], 0.5 * p.wavelet[:, 0]], axis=1)
    ro, uo, _ = oracle_forward(p)
    rg, ug, _ = gpu_forward(p, variant=2)
    assert rel(rg, ro) <= TOL and rel(ug[1], uo[1]) <= TOL
    rg1, ug1, _ = gpu_forward(p, variant=1)
    assert np.array_equal(rg, rg1) and np.array_equal(ug, ug1)


@pytest.mark.parametrize("variant", [1, 2])
def test_split_boundary_launches_bitwise(variant):
    """SF_OPT_SPLIT (the slab-mode schedule: boundary planes + their injection first, then
    the interior, optionally on fewer persistent CTAs, SF_OPT_COMM_SMS) reorders work only: forward records/state and adjoint+gradient are
    bitwise identical to the single launch (fused small-set and standalone large-set
    sparse paths, sources and receivers in the boundary planes)."""
    p = synth.random_problem(3, (26, 30, 64), 8, 50, seed=31, nbl=5, nsrc=3, nrec=300)
    h = p.h
    p.src_coords[0, 0] = 1.5 * h            # in the left boundary planes (r = 4)
    p.src_coords[1, 0] = (p.shape[0] - 2.3) * h   # in the right boundary planes
    p.rec_coords[:50, 0] = 2.0 * h
    p.m_true = (p.m * 0.93).astype(np.float32)
    d_obs = oracle.forward(p, m=p.m_true)["rec"].astype(np.float32)
    out = {}
    for split in (0, 1, 2):
        for fuse in (256, 0):
            prop = make_prop(p)
            prop.set_tuning(variant, 0, 0)
            prop.set_option(2, min(split, 1))
            prop.set_option(3, fuse)
            if split == 2:
                prop.set_option(4, 60)  # interior launch leaves 60 SMs free (SF_OPT_COMM_SMS)
            rec, u, _ = prop.forward(dev(p.wavelet))
            g, J = prop.gradient(dev(p.wavelet), dev(d_obs), save_every=3)
            torch.cuda.synchronize()
            out[(split, fuse)] = (rec.cpu().numpy(), u.cpu().numpy(), g.cpu().numpy(), J)
            prop.close()
    base = out[(0, 256)]
    for k, v in out.items():
        assert all(np.array_equal(a, b) for a, b in zip(v[:3], base[:3])) and v[3] == base[3], k
    go = oracle.gradient(p, d_obs, save_every=3)
    assert rel(base[2], go["grad"]) <= TOL


# ------------------------------------------------------------ separable damping (16 B/pt)
def make_prop_sep(p, m=None, **kw):
    """Same problem, damping given as the separable profiles (sf_desc.sigma) instead of
    the eta array: beta regenerated in-kernel, c3 hoisted from m and the profiles."""
    m = p.m if m is None else m
    return sf().Propagator(dev(m), None, shape=p.shape, h=p.h, space_order=p.space_order, nt=p.nt,
                           dt=p.dt, src_coords=p.src_coords.astype(np.float64),
                           rec_coords=p.rec_coords.astype(np.float64), sigma=p.sigma, **kw)


@pytest.mark.parametrize("so", [4, 8, 16])
def test_separable_damping_forward(so):
    """Separable damping (reading C7 structure): both variants vs the oracle fed
    the equivalent eta array; TMA and generic bitwise equal (one sf_beta_sep); close to
    the beta-array path (the two differ only by fp32 rounding of eta and of beta)."""
    p = synth.random_problem(3, (37, 45, 132), so, 60, seed=40 + so, nbl=6, nsrc=2, nrec=9)
    ro, uo, _ = oracle_forward(p)
    out = {}
    for variant, vy, ctas in ((1, 0, 0), (2, 2, 0), (2, 2, 3), (2, 1, 0)):
        prop = make_prop_sep(p)
        prop.set_tuning(variant, vy, ctas)
        rec, u, _ = prop.forward(dev(p.wavelet))
        torch.cuda.synchronize()
        out[(variant, vy, ctas)] = (rec.cpu().numpy(), u.cpu().numpy())
        prop.close()
        assert rel(out[(variant, vy, ctas)][0], ro) <= TOL
        assert rel(out[(variant, vy, ctas)][1][1], uo[1]) <= TOL
    base = out[(1, 0, 0)]
    for k, v in out.items():
        assert np.array_equal(v[0], base[0]) and np.array_equal(v[1], base[1]), k
    ra, ua, _ = gpu_forward(p)
    assert rel(base[0], ra) <= 1e-5 and rel(base[1][1], ua[1]) <= 1e-5


def test_separable_damping_2d_and_gradient():
    """2D (generic kernel, sigma_x and sigma_z) forward, and the 3D gradient (SAVE and
    GRAD modes of the TMA kernel) with separable damping, vs the oracle."""
    p2 = synth.random_problem(2, (90, 110), 8, 120, seed=5, nbl=10, nsrc=2, nrec=11)
    ro, uo, _ = oracle_forward(p2)
    prop = make_prop_sep(p2)
    rec, u, _ = prop.forward(dev(p2.wavelet))
    torch.cuda.synchronize()
    assert rel(rec.cpu().numpy(), ro) <= TOL and rel(u.cpu().numpy()[1], uo[1]) <= TOL
    prop.close()
    p = synth.random_problem(3, (30, 34, 64), 8, 60, seed=6, nbl=5, nsrc=2, nrec=25)
    p.m_true = (p.m * 0.9).astype(np.float32)
    d_obs = oracle.forward(p, m=p.m_true)["rec"].astype(np.float32)
    go = oracle.gradient(p, d_obs, save_every=3)
    for variant in (2, 1):
        prop = make_prop_sep(p)
        prop.set_tuning(variant, 0, 0)
        g, J = prop.gradient(dev(p.wavelet), dev(d_obs), save_every=3)
        torch.cuda.synchronize()
        assert rel(g.cpu().numpy(), go["grad"]) <= TOL, (variant, rel(g.cpu().numpy(), go["grad"]))
        assert abs(J - go["J"]) <= 1e-4 * go["J"]
        prop.close()


def test_separable_damping_errors():
    p = synth.random_problem(3, (16, 16, 16), 4, 10, seed=0, nbl=3)
    S = sf()
    kw = dict(shape=p.shape, h=p.h, space_order=4, nt=10, dt=p.dt)
    with pytest.raises(S.SfError) as e:      # damp and sigma are exclusive
        S.Propagator(dev(p.m), dev(p.damp), sigma=p.sigma, **kw)
    assert e.value.status == "SF_ERR_INVALID_ARG"
    bad = [s.copy() for s in p.sigma]
    bad[1][2] = -1.0
    with pytest.raises(S.SfError) as e:      # negative profile value
        S.Propagator(dev(p.m), None, sigma=bad, **kw)
    assert e.value.status == "SF_ERR_INVALID_ARG"
    with pytest.raises(ValueError):          # wrong number / length of profiles
        S.Propagator(dev(p.m), None, sigma=p.sigma[:2], **kw)


# ------------------------------------------------------------ checkpointed gradient (f3)
@pytest.mark.parametrize("ndim,k,segment", [(3, 3, 6), (3, 1, 7), (3, 4, 400), (2, 2, 10)])
def test_gradient_checkpointed_bitwise(ndim, k, segment):
    """sf_gradient_ckpt (checkpoint-recompute) == sf_gradient bit for bit (deterministic
    kernels; the recomputed forward starts from the exact checkpointed state pair), for
    segments that divide nt-1, leave a ragged last segment, or exceed the record."""
    shape = (30, 34, 64) if ndim == 3 else (80, 96)
    p = synth.random_problem(ndim, shape, 8, 61, seed=70 + k, nbl=5, nsrc=2, nrec=20)
    p.m_true = (p.m * 0.9).astype(np.float32)
    d_obs = oracle.forward(p, m=p.m_true)["rec"].astype(np.float32)
    prop = make_prop(p)
    g, J = prop.gradient(dev(p.wavelet), dev(d_obs), save_every=k)
    gc, Jc = prop.gradient_ckpt(dev(p.wavelet), dev(d_obs), save_every=k, segment=segment)
    torch.cuda.synchronize()
    assert np.array_equal(g.cpu().numpy(), gc.cpu().numpy()) and J == Jc
    full = prop.gradient_workspace_bytes(k)
    ck = prop.gradient_ckpt_workspace_bytes(k, segment)
    if k == 1:   # every step saved: 9 checkpoints + 8 snapshots instead of 61 snapshots
        assert ck < 0.6 * full
    with pytest.raises(ValueError):
        prop.gradient_ckpt(dev(p.wavelet), dev(d_obs), save_every=3, segment=4)
    prop.close()


# ------------------------------------------------------------ slab path on one device
def _run_ranks(nranks, fn):
    """Run fn(rank) for every rank in its own thread (and CUDA stream); re-raise errors."""
    import threading
    out, err = [None] * nranks, []

    def body(rank):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                out[rank] = fn(rank)
                s.synchronize()
        except BaseException as e:  # noqa: BLE001
            err.append(e)

    ts = [threading.Thread(target=body, args=(q,)) for q in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    assert not err, err
    return out


def _slab_inputs(p, rank, nranks):
    S = sf()
    r = p.space_order // 2
    x0, nl = S.slab_plan(p.shape[0], p.space_order, rank, nranks)
    g = np.arange(x0 - r, x0 + nl + r)
    ok = (g >= 0) & (g < p.shape[0])
    m = np.ones((nl + 2 * r,) + tuple(p.shape[1:]), np.float32)
    m[ok] = p.m[g[ok]]
    eta = None
    if p.damp is not None:
        eta = np.zeros_like(m)
        eta[ok] = p.damp[g[ok]]
    return x0, nl, m, eta


@pytest.mark.parametrize("nranks,variant,p2p,dense", [(2, 2, 0, 0), (3, 2, 0, 0), (3, 1, 0, 0), (2, 2, 1, 0),
                                                      (3, 2, 1, 0), (3, 1, 1, 0), (2, 2, 0, 1), (3, 2, 1, 1)])
def test_slab_decomposition_bitwise_local_transport(nranks, variant, p2p, dense):
    """The multi-GPU slab path (local [n0_loc + 2r] buffers, split boundary/interior
    launches with the persistent-kernel SM reservation, per-step halo exchange, owner-only
    injection and records, record all-reduce inside the gradient) run as rank threads on
    ONE device through the in-process transport (same planes as the NCCL exchange): the
    records, the owned planes of both final levels and of the gradient, and J are bitwise
    those of the single-domain run (reading C18).  Sources and receivers straddle the slab
    boundaries.  p2p = 1: SF_OPT_P2P -- the boundary kernel stores the boundary planes
    straight into the neighbours' halos and the streams order on counters -- with
    the TMA kernel, from the single persistent launch of each step (one-launch schedule); the
    transport then only runs once per call (the initial halo).  dense = 1: 20 receivers
    inside one grid cell at a rank boundary, so their 8 corners get 20 contributions each
    and the adjoint injection takes the CSR path (no ELL table) in the split launches."""
    S = sf()
    p = synth.random_problem(3, (41, 30, 64), 8, 50, seed=91, nbl=5, nsrc=3, nrec=40)
    h = p.h
    p.src_coords[0, 0] = 13.5 * h          # on / across the rank boundaries (41 planes)
    p.src_coords[1, 0] = 20.2 * h
    p.rec_coords[:20, 0] = np.linspace(8 * h, 33 * h, 20)
    if dense:
        cell = np.array([13.0, 14.0, 30.0]) * h
        p.rec_coords[20:] = (cell + np.random.default_rng(5).uniform(0.1, 0.9, (20, 3)) * h).astype(np.float32)
    p.m_true = (p.m * 0.92).astype(np.float32)
    d_obs = oracle.forward(p, m=p.m_true)["rec"].astype(np.float32)
    prop = make_prop(p)
    prop.set_tuning(variant, 0, 0)
    rec1, u1, _ = prop.forward(dev(p.wavelet))
    g1, J1 = prop.gradient(dev(p.wavelet), dev(d_obs), save_every=3)
    torch.cuda.synchronize()
    rec1, u1, g1 = rec1.cpu().numpy(), u1.cpu().numpy(), g1.cpu().numpy()
    prop.close()
    group = S.local_group_create(nranks)
    r = p.space_order // 2

    def rank_fn(rank):
        x0, nl, m, eta = _slab_inputs(p, rank, nranks)
        pr = S.Propagator(dev(m), None if eta is None else dev(eta), shape=p.shape, h=p.h,
                          space_order=p.space_order, nt=p.nt, dt=p.dt,
                          src_coords=p.src_coords.astype(np.float64),
                          rec_coords=p.rec_coords.astype(np.float64), comm=group, rank=rank, nranks=nranks)
        pr.set_tuning(variant, 0, 0)
        if p2p:
            pr.set_option(8, 1)
        pr.set_profiling(True)
        pr.profile(reset=True)
        rec, u, _ = pr.forward(dev(p.wavelet))
        torch.cuda.current_stream().synchronize()
        other = pr.profile(reset=True)["other_launches"]
        pr.set_profiling(False)
        # transport exchanges: one per step, or only the initial one with peer stores
        assert (other <= 2) if p2p else (other >= p.nt - 1), other
        if p2p and variant == 2:
            # peer stores from the ONE persistent TMA launch per step (SF_OPT_ONE_LAUNCH +
            # SF_OPT_P2P: boundary planes stored into the neighbours' halos by the stencil
            # kernel itself) on every forward step
            assert pr.debug_probe(None) == p.nt - 1
        g, J = pr.gradient(dev(p.wavelet), dev(d_obs), save_every=3)
        torch.cuda.current_stream().synchronize()
        res = (x0, nl, rec.cpu().numpy(), u.cpu().numpy()[:, r:r + nl], g.cpu().numpy()[r:r + nl], J)
        pr.close()
        return res

    try:
        outs = _run_ranks(nranks, rank_fn)
    finally:
        S.local_group_destroy(group)
    rec_sum = sum(o[2] for o in outs)
    assert np.array_equal(rec_sum, rec1)
    for x0, nl, _, u, g, J in outs:
        assert np.array_equal(u, u1[:, x0:x0 + nl]), (x0, nl)
        assert np.array_equal(g, g1[x0:x0 + nl]), (x0, nl)
        assert J == J1


def test_multishot_allreduce_local_transport():
    """Multi-shot FWI (one shot per rank) + sf_allreduce_gradient over the in-process
    transport: the summed gradient and J equal the sequential sum of the shots'."""
    S = sf()
    shots = []
    for s in range(2):
        p = synth.random_problem(3, (26, 30, 64), 8, 40, seed=95 + s, nbl=5, nsrc=1, nrec=30)
        p.m = shots[0].m if shots else p.m
        p.damp = shots[0].damp if shots else p.damp
        p.m_true = (p.m * 0.9).astype(np.float32)
        shots.append(p)
    gs, Js = [], []
    for p in shots:
        d_obs = oracle.forward(p, m=p.m_true)["rec"].astype(np.float32)
        pr = make_prop(p)
        g, J = pr.gradient(dev(p.wavelet), dev(d_obs), save_every=2)
        torch.cuda.synchronize()
        gs.append(g.cpu().numpy())
        Js.append(J)
        p.d_obs = d_obs
        pr.close()
    group = S.local_group_create(2)

    def rank_fn(rank):
        p = shots[rank]
        pr = make_prop(p)
        g, J = pr.gradient(dev(p.wavelet), dev(p.d_obs), save_every=2)
        g, J = pr.allreduce_gradient(group, g, J, rank=rank)
        torch.cuda.current_stream().synchronize()
        out = (g.cpu().numpy(), J)
        pr.close()
        return out

    try:
        outs = _run_ranks(2, rank_fn)
    finally:
        S.local_group_destroy(group)
    gsum = (gs[0] + gs[1]).astype(np.float32)
    for g, J in outs:
        assert np.array_equal(g, gsum)
        assert J == Js[0] + Js[1]


# ------------------------------------------------------------ CUDA graph replay
@pytest.mark.parametrize("cfg", [0, 1, "narrow"])
def test_graph_replay_bitwise(cfg):
    """SF_OPT_GRAPH: the first call runs eagerly, the second identical call is captured as
    one CUDA graph (on the handle's stream, event-ordered after the caller's stream) and
    replayed afterwards: records, states and gradients bitwise those of eager calls; a
    tuning change drops the graph; a restart state (same buffers, new contents) is honoured."""
    if cfg == "narrow":  # so12 with a 16-column z remainder: two stencil launches per step
        p = synth.random_problem(3, (40, 44, 144), 12, 40, seed=3, nbl=5, nsrc=2, nrec=9)
    else:
        p = synth.make_config(cfg, scale=1.0 if cfg == 0 else 0.15, nt=60)
    p.m_true = (p.m * 0.9).astype(np.float32)
    d_obs = oracle.forward(p, m=p.m_true)["rec"].astype(np.float32)
    ref = make_prop(p)
    r0, u0, _ = ref.forward(dev(p.wavelet))
    g0, J0 = ref.gradient(dev(p.wavelet), dev(d_obs), save_every=2)
    torch.cuda.synchronize()
    r0, u0, g0 = r0.cpu().numpy(), u0.cpu().numpy(), g0.cpu().numpy()
    ref.close()
    prop = make_prop(p)
    prop.set_option(5, 1)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        wav, dob = dev(p.wavelet), dev(d_obs)
        u = prop.zeros_state()
        rec = torch.empty((p.nt, p.rec_coords.shape[0]), device="cuda")
        ws = torch.empty(prop.gradient_workspace_bytes(2), dtype=torch.uint8, device="cuda")
        grad = torch.empty(prop.local_shape, device="cuda")
        for it in range(4):
            if it == 3:
                prop.set_tuning(0, 0, 0)   # drops the graphs: eager again
            u.zero_()
            prop.forward(wav, u=u, rec=rec)
            s.synchronize()
            assert np.array_equal(rec.cpu().numpy(), r0) and np.array_equal(u.cpu().numpy(), u0), it
            g, J = prop.gradient(wav, dob, save_every=2, grad=grad, ws=ws)
            s.synchronize()
            assert np.array_equal(g.cpu().numpy(), g0) and J == J0, it
    prop.close()


# ------------------------------------------------------------ f4: convection, Laplace
@pytest.mark.parametrize("shape", [(81, 81), (200, 170)])
def test_convection2d_parity(shape):
    """Eq. 2 on the GPU (one-CTA shared-memory loop at the paper's 81^2, per-step kernels
    above 25 600 points) vs the fp64 oracle: relative L2 <= 1e-5 after 100 steps; edges
    bitwise unchanged."""
    q = synth.convection_problem(*shape, nt=100)
    ref = oracle.convection2d(q["u0"], c=q["c"], dt=q["dt"], dx=q["dx"], dy=q["dy"], nt=q["nt"])
    u = dev(q["u0"])
    sf().convection2d(u, c=q["c"], dt=q["dt"], dx=q["dx"], dy=q["dy"], nt=q["nt"])
    torch.cuda.synchronize()
    g = u.cpu().numpy()
    assert rel(g, ref) <= 1e-5, rel(g, ref)
    for sl in (np.s_[0, :], np.s_[-1, :], np.s_[:, 0], np.s_[:, -1]):
        assert np.array_equal(g[sl], q["u0"][sl])


@pytest.mark.parametrize("shape", [(31, 31), (190, 150)])
def test_laplace2d_parity(shape):
    """Jacobi sweeps of Eq. 4 with the listing's boundary rows: (a) a fixed sweep count
    (tol < 0) vs the oracle, relative L2 <= 1e-5; (b) the paper's l1 < 1e-4 loop stops
    within one sweep of the oracle's count, and the field equals the oracle run for the
    GPU's count."""
    q = synth.laplace_problem(*shape)
    kw = dict(dx=q["dx"], dy=q["dy"])
    n = 300 if shape[0] < 100 else 40
    ref, _, _ = oracle.laplace2d(q["p0"], q["bc"], tol=-1.0, max_iter=n, **kw)
    p, it, l1 = sf().laplace2d(dev(q["p0"]), dev(q["bc"]), tol=-1.0, max_iter=n, **kw)
    assert it == n and rel(p.cpu().numpy(), ref) <= 1e-5
    if shape[0] < 100:
        ro, ito, _ = oracle.laplace2d(q["p0"], q["bc"], tol=1e-4, **kw)
        p, it, l1 = sf().laplace2d(dev(q["p0"]), dev(q["bc"]), tol=1e-4, **kw)
        assert abs(it - ito) <= 1 and l1 <= 1e-4
        ref, _, _ = oracle.laplace2d(q["p0"], q["bc"], tol=-1.0, max_iter=it, **kw)
        assert rel(p.cpu().numpy(), ref) <= 1e-5


# ------------------------------------------------------------ fp16 snapshots (C23)
def test_fp16_snapshots_forward_and_gradient():
    """SF_OPT_SNAP_HALF: saved snapshots are exactly the fp32 snapshots rounded to fp16
    (bitwise vs torch's conversion); the gradient (TMA and generic, full and checkpointed)
    matches the oracle with fp16 snapshots (rel. L2 <= 1e-4); TMA == generic == checkpointed
    bitwise; within the quantisation bound of the fp32-snapshot gradient."""
    p = synth.random_problem(3, (26, 30, 64), 8, 61, seed=33, nbl=5, nsrc=2, nrec=30)
    p.m_true = (p.m * 0.9).astype(np.float32)
    d_obs = oracle.forward(p, m=p.m_true)["rec"].astype(np.float32)
    go16 = oracle.gradient(p, d_obs, save_every=3, snap_dtype="float16")
    prop = make_prop(p)
    _, _, s32 = prop.forward(dev(p.wavelet), save_every=3)
    g32, _ = prop.gradient(dev(p.wavelet), dev(d_obs), save_every=3)
    prop.set_option(7, 1)
    _, _, s16 = prop.forward(dev(p.wavelet), save_every=3)
    torch.cuda.synchronize()
    assert s16.dtype == torch.float16 and torch.equal(s16, s32.half())
    out = []
    for variant in (2, 1):
        prop.set_tuning(variant, 0, 0)
        g, J = prop.gradient(dev(p.wavelet), dev(d_obs), save_every=3)
        gc, Jc = prop.gradient_ckpt(dev(p.wavelet), dev(d_obs), save_every=3, segment=9)
        torch.cuda.synchronize()
        out.append(g.cpu().numpy())
        assert np.array_equal(g.cpu().numpy(), gc.cpu().numpy()) and J == Jc
        assert rel(g.cpu().numpy(), go16["grad"]) <= TOL, rel(g.cpu().numpy(), go16["grad"])
        assert abs(J - go16["J"]) <= 1e-4 * go16["J"]
    assert np.array_equal(out[0], out[1])
    assert rel(out[0], g32.cpu().numpy()) < 2.0 ** -11 * 4
    assert prop.gradient_workspace_bytes(3) < make_prop(p).gradient_workspace_bytes(3)
    prop.close()


def test_p2p_option_errors():
    """SF_OPT_P2P needs a slab handle whose every rank owns more than 2r planes."""
    S = sf()
    p = synth.random_problem(3, (20, 16, 32), 8, 10, seed=5, nbl=0, nsrc=1, nrec=2)
    prop = make_prop(p)
    with pytest.raises(S.SfError):
        prop.set_option(8, 1)           # single-domain handle
    prop.close()
    group = S.local_group_create(3)

    def rank_fn(rank):
        x0, nl, m, eta = _slab_inputs(p, rank, 3)
        pr = S.Propagator(dev(m), None if eta is None else dev(eta), shape=p.shape, h=p.h,
                          space_order=p.space_order, nt=p.nt, dt=p.dt,
                          src_coords=p.src_coords.astype(np.float64),
                          rec_coords=p.rec_coords.astype(np.float64), comm=group, rank=rank, nranks=3)
        try:
            pr.set_option(8, 1)        # 20 planes / 3 ranks: 6-7 planes <= 2r = 8
            return None
        except S.SfError as e:
            return e.status
        finally:
            pr.close()

    try:
        outs = _run_ranks(3, rank_fn)
    finally:
        S.local_group_destroy(group)
    assert outs == ["SF_ERR_SHAPE"] * 3, outs


def test_nccl_single_rank_transport():
    """The NCCL plumbing on the box: libnccl resolved at run time (the copy torch loaded),
    communicator from an ncclUniqueId, the in-stream gradient all-reduce (fp32 + fp64 J)
    -- on one rank the sum is the identity, bitwise."""
    import socket

    import torch.distributed as dist
    S = sf()
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        comm = S.nccl_comm_init(S.nccl_unique_id(), 1, 0)
        p = synth.random_problem(3, (20, 18, 32), 4, 20, seed=8, nbl=3, nsrc=1, nrec=5)
        prop = make_prop(p)
        g = torch.randn(p.shape, device="cuda")
        g0 = g.clone()
        g, J = prop.allreduce_gradient(comm, g, 1.25, rank=0)
        torch.cuda.synchronize()
        assert torch.equal(g, g0) and J == 1.25
        prop.close()
        S.nccl_comm_destroy(comm)
    finally:
        dist.destroy_process_group()


def test_tma_bitwise_with_concurrent_records():
    """Regression: the TMA kernel's slot releases under contention.  configs[4] at its full
    grid (r = 6) with 160 000 surface receivers, every level saved and the source injected
    by the standalone kernel: the side-stream record kernels then run concurrently with the
    persistent stencil and their small blocks share its SMs.  Per-thread slot releases
    gave wrong values in ~1 of 2 runs here; every repetition must equal the generic
    kernel bit for bit."""
    p = synth.make_config(4, nt=10)
    outs = []
    for variant in (1, 2, 2, 2, 2):
        prop = make_prop(p)
        prop.set_tuning(variant, 0, 0)
        prop.set_option(3, 0)          # standalone injection
        rec, u, snaps = prop.forward(dev(p.wavelet), save_every=1)
        torch.cuda.synchronize()
        outs.append((rec.cpu().numpy(), u.cpu().numpy(), snaps.cpu().numpy()))
        prop.close()
        del rec, u, snaps
    for o in outs[1:]:
        for a, b in zip(o, outs[0]):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("shape,so", [((34, 30, 144), 10), ((30, 60, 144), 12), ((26, 22, 192), 16),
                                      ((22, 58, 296), 14)])
def test_z_remainder_narrow_tiles_bitwise(shape, so):
    """SF_OPT_ZSPLIT (space order >= 10): n2 = 128 k + rem (rem 16 / 16 / 64 / 40) -> 128-column tiles over the
    first 128 k columns, then narrow 56 x 32 tiles over the rest.  Forward (records, state,
    snapshots) and gradient are bitwise equal to the unsplit launch and within 1e-4 of the
    oracle; a source and receivers sit in the remainder columns, rows span several narrow
    tiles (ragged last tile)."""
    p = synth.random_problem(3, shape, so, 60, seed=31, nbl=5, nsrc=2, nrec=12)
    n2 = shape[2]
    p.src_coords[1, 2] = (n2 - 8.3) * p.h
    p.rec_coords[0, 2] = (n2 - 7.4) * p.h
    p.rec_coords[1, 2] = (n2 - 9.0) * p.h
    rng = np.random.default_rng(5)
    m_true = (p.m * rng.uniform(0.9, 1.1, p.m.shape)).astype(np.float32)
    d_obs = oracle.forward(p, m=m_true)["rec"].astype(np.float32)
    ro, uo, sno = oracle_forward(p, save_every=4)
    go = oracle.gradient(p, d_obs, save_every=4)
    outs = []
    for z in (1, 0):
        prop = make_prop(p)
        prop.set_option(9, z)
        assert prop.tuning()["variant"] == 2
        prop.set_profiling(True)
        prop.profile(reset=True)
        rec, u, snaps = prop.forward(dev(p.wavelet), save_every=4)
        torch.cuda.synchronize()
        launches = prop.profile(reset=True)["other_launches"]
        prop.set_profiling(False)
        g, J = prop.gradient(dev(p.wavelet), dev(d_obs), save_every=4)
        torch.cuda.synchronize()
        outs.append((rec.cpu().numpy(), u.cpu().numpy(), snaps.cpu().numpy(), g.cpu().numpy(), J, launches))
        prop.close()
    on, off = outs
    for a, b in zip(on[:4], off[:4]):
        assert np.array_equal(a, b)
    assert on[4] == off[4]
    assert on[5] >= off[5] + (p.nt - 1)  # one narrow launch per step
    assert rel(on[0], ro) <= TOL and rel(on[1], uo) <= TOL and rel(on[2], sno) <= TOL
    assert rel(on[3], go["grad"]) <= TOL, rel(on[3], go["grad"])


@pytest.mark.parametrize("shape,so", [((5, 3, 8), 2), ((17, 15, 4), 8), ((9, 31, 132), 16),
                                      ((3, 4, 136), 12), ((40, 4, 16), 4)])
def test_tma_small_and_ragged_extents(shape, so):
    """Edge shapes through the TMA kernel: fewer planes / rows than the radius or than one
    tile, four rows, n2 = 4 (one lane), 128 k + 4 / + 8 columns (narrow-tile remainder at
    r >= 5).  Records and state bitwise equal to the generic kernel and within 1e-4 of the
    oracle; constant-free random wavefield start (restart form)."""
    p = synth.random_problem(3, shape, so, 12, seed=41, nbl=0, nsrc=1, nrec=3, damp=False)
    rng = np.random.default_rng(9)
    u0 = rng.standard_normal((2,) + shape).astype(np.float32)
    o = oracle.forward(p, u_state=u0)
    outs = []
    for variant in (1, 2):
        prop = make_prop(p)
        prop.set_tuning(variant, 0, 0)
        assert prop.tuning()["variant"] == variant
        rec, u, _ = prop.forward(dev(p.wavelet), u=dev(u0))
        torch.cuda.synchronize()
        outs.append((rec.cpu().numpy(), u.cpu().numpy()))
        prop.close()
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    assert rel(outs[1][0], o["rec"]) <= TOL and rel(outs[1][1], o["u_state"]) <= TOL


def test_bench_json_contract():
    """bench.py prints one JSON line with the contract's keys (short run: nt = 20)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--nt", "20", "--steps", "1",
                          "--warmup", "3", "--cpu-seconds", "1"], capture_output=True, text=True,
                         timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "gpu_launches", "clocks"):
        assert k in d, k
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["gpu_launches"] > 0
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"], k
    assert 0 < d["roofline"]["frac"] < 1.2
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in d["cpu_baseline"], k
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"], k
    assert "workload" in d["config"]


@pytest.mark.parametrize("so", [12, 16])
def test_gradient_high_order_damped_tma(so):
    """GRAD mode at the tightest shared-memory plans (r = 6 / 8 with the beta array: the u
    ring shrinks to its minimum depth and two coefficient stages of five planes): gradient
    and J vs the oracle, and bitwise equal to the generic kernel; adjoint source records
    too."""
    p = synth.random_problem(3, (34, 30, 64), so, 60, seed=17, nbl=6, nsrc=1, nrec=16)
    rng = np.random.default_rng(8)
    p.m_true = (p.m * rng.uniform(0.88, 1.12, p.m.shape)).astype(np.float32)
    d_obs = oracle.forward(p, m=p.m_true)["rec"].astype(np.float32)
    go = oracle.gradient(p, d_obs, save_every=2)
    outs = []
    for variant in (2, 1):
        prop = make_prop(p)
        prop.set_tuning(variant, 0, 0)
        assert prop.tuning()["variant"] == variant
        g, J = prop.gradient(dev(p.wavelet), dev(d_obs), save_every=2)
        torch.cuda.synchronize()
        outs.append((g.cpu().numpy(), J))
        prop.close()
    assert np.array_equal(outs[0][0], outs[1][0]) and outs[0][1] == outs[1][1]
    assert rel(outs[0][0], go["grad"]) <= TOL, rel(outs[0][0], go["grad"])
    assert abs(outs[0][1] - go["J"]) <= 1e-4 * go["J"]
    # adjoint source records: GPU forward snapshots + GRAD-mode adjoint driven by the
    # oracle's residual, vs the oracle's srca (and gradient), both variants bitwise
    sr = []
    for variant in (2, 1):
        prop = make_prop(p)
        prop.set_tuning(variant, 0, 0)
        _, _, snaps = prop.forward(dev(p.wavelet), save_every=2)
        srca, _, g = prop.adjoint(dev(go["res"]), snaps=snaps, save_every=2,
                                  grad=torch.zeros(p.shape, device="cuda"))
        torch.cuda.synchronize()
        sr.append((srca.cpu().numpy(), g.cpu().numpy()))
        prop.close()
    assert np.array_equal(sr[0][0], sr[1][0]) and np.array_equal(sr[0][1], sr[1][1])
    assert rel(sr[0][0], go["srca"]) <= TOL, rel(sr[0][0], go["srca"])
    assert rel(sr[0][1], go["grad"]) <= TOL


# ------------------------------------------------------------------- receiver surfaces
def _surface_problem(shape, so, nt, zs, seed, nbl=4, damp=True):
    """Receivers on every grid node of the plane z = zs inside an absorbing ring (> 256
    targets, one contribution each, like the configs' surface receiver grids); the source
    two cells below the receiver plane so records and residuals carry signal."""
    p = synth.random_problem(3, shape, so, nt, seed=seed, nbl=nbl if damp else 0, nsrc=1, nrec=4,
                             damp=damp)
    h = p.h
    lo = nbl + 1 if damp else 1
    ii, jj = np.meshgrid(np.arange(lo, shape[0] - lo), np.arange(lo, shape[1] - lo), indexing="ij")
    p.rec_coords = np.stack([ii.ravel() * h, jj.ravel() * h, np.full(ii.size, zs * h)], 1).astype(np.float32)
    zsrc = zs + 2.3 if zs + 3 < shape[2] else zs - 2.3
    p.src_coords = np.array([[shape[0] / 2.0 * h + 0.3 * h, shape[1] / 2.0 * h - 0.4 * h, zsrc * h]],
                            dtype=np.float32)
    return p


@pytest.mark.parametrize("shape,so,zs,damp", [((30, 44, 64), 8, 9, True), ((26, 30, 144), 12, 7, False),
                                              ((26, 30, 144), 12, 135, False), ((30, 30, 132), 4, 129, True)])
def test_receiver_surface_adjoint_gradient(shape, so, zs, damp):
    """Adjoint injection of a receiver surface (every node of z = zs: > 256 targets, the
    standalone injection kernel between stencil steps): adjoint source records, final
    levels and the fused gradient (GRAD mode + the injection's correlation patch) are bitwise
    equal between the TMA and generic kernels and match the oracle.  r = 4 (unrolled loop,
    combined Laplacian form) and r = 6 with the narrow-tile z split (zs in the 128-column
    tiles and in the remainder), ragged tiles, the last z columns."""
    p = _surface_problem(shape, so, 60, zs, seed=41, damp=damp)
    assert p.rec_coords.shape[0] > 256
    rng = np.random.default_rng(2)
    p.m_true = (p.m * rng.uniform(0.9, 1.1, p.m.shape)).astype(np.float32)
    d_obs = oracle.forward(p, m=p.m_true)["rec"].astype(np.float32)
    go = oracle.gradient(p, d_obs, save_every=2)
    assert np.linalg.norm(go["srca"]) > 1e-6 * np.abs(go["res"]).max()
    outs = []
    for variant in (2, 1):
        prop = make_prop(p)
        prop.set_tuning(variant, 0, 0)
        _, _, snaps = prop.forward(dev(p.wavelet), save_every=2)
        srca, v, g = prop.adjoint(dev(go["res"]), snaps=snaps, save_every=2,
                                  grad=torch.zeros(p.shape, device="cuda"))
        srca0, v0, _ = prop.adjoint(dev(go["res"]))          # PLAIN-mode adjoint
        gg, J = prop.gradient(dev(p.wavelet), dev(d_obs), save_every=2)
        torch.cuda.synchronize()
        outs.append([x.cpu().numpy() for x in (srca, v, g, srca0, v0, gg)] + [J])
        prop.close()
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)
    assert rel(outs[0][0], go["srca"]) <= TOL and rel(outs[0][3], go["srca"]) <= TOL
    assert rel(outs[0][2], go["grad"]) <= TOL and rel(outs[0][5], go["grad"]) <= TOL
    assert abs(outs[0][6] - go["J"]) <= 1e-4 * go["J"]


def test_many_sources_forward_save():
    """Forward injection of a large SOURCE surface (320 sources on the nodes of z = 5, the
    standalone kernel) in SAVE mode: the snapshots hold the post-injection values, bitwise
    equal between the TMA and generic kernels, and records, final level and snapshots match
    the oracle."""
    p = synth.random_problem(3, (24, 28, 64), 8, 40, seed=5, nbl=3, nsrc=1, nrec=6)
    h = p.h
    ii, jj = np.meshgrid(np.arange(4, 20), np.arange(4, 24), indexing="ij")
    p.src_coords = np.stack([ii.ravel() * h, jj.ravel() * h, np.full(ii.size, 5 * h)], 1).astype(np.float32)
    ns = p.src_coords.shape[0]
    p.wavelet = np.random.default_rng(3).standard_normal((p.nt, ns)).astype(np.float32)
    ro, uo, so_ = oracle_forward(p, save_every=3)
    outs = []
    for variant in (2, 1):
        prop = make_prop(p)
        prop.set_tuning(variant, 0, 0)
        rec, u, snaps = prop.forward(dev(p.wavelet), save_every=3)
        torch.cuda.synchronize()
        outs.append((rec.cpu().numpy(), u.cpu().numpy(), snaps.cpu().numpy()))
        prop.close()
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)
    assert rel(outs[0][0], ro) <= TOL and rel(outs[0][1][1], uo[1]) <= TOL
    for k in range(1, so_.shape[0]):
        assert rel(outs[0][2][k], so_[k]) <= TOL


@pytest.mark.parametrize("nranks", [2, 3])
def test_receiver_surface_slab_bitwise(nranks):
    """Slab path (split boundary / interior launches, local transport) with a receiver
    surface injected by the split-list kernels: gradient, J and the owned planes bitwise
    equal to the single-domain run."""
    S = sf()
    p = _surface_problem((41, 30, 64), 8, 40, 9, seed=44)
    p.m_true = (p.m * 0.93).astype(np.float32)
    d_obs = oracle.forward(p, m=p.m_true)["rec"].astype(np.float32)
    prop = make_prop(p)
    g1, J1 = prop.gradient(dev(p.wavelet), dev(d_obs), save_every=3)
    torch.cuda.synchronize()
    g1 = g1.cpu().numpy()
    prop.close()
    group = S.local_group_create(nranks)
    r = p.space_order // 2

    def rank_fn(rank):
        x0, nl, m, eta = _slab_inputs(p, rank, nranks)
        pr = S.Propagator(dev(m), None if eta is None else dev(eta), shape=p.shape, h=p.h,
                          space_order=p.space_order, nt=p.nt, dt=p.dt,
                          src_coords=p.src_coords.astype(np.float64),
                          rec_coords=p.rec_coords.astype(np.float64), comm=group, rank=rank, nranks=nranks)
        g, J = pr.gradient(dev(p.wavelet), dev(d_obs), save_every=3)
        torch.cuda.current_stream().synchronize()
        res = (x0, nl, g.cpu().numpy()[r:r + nl], J)
        pr.close()
        return res

    try:
        outs = _run_ranks(nranks, rank_fn)
    finally:
        S.local_group_destroy(group)
    for x0, nl, g, J in outs:
        assert np.array_equal(g, g1[x0:x0 + nl]), (x0, nl)
        assert J == J1


# ------------------------------------------------------------------- one-launch schedule
@pytest.mark.parametrize("so,shape,plane", [(8, (58, 30, 64), True), (16, (60, 26, 64), False), (4, (40, 44, 128), True)])
def test_one_launch_schedule_bitwise(so, shape, plane):
    """The one-launch slab schedule (SF_OPT_ONE_LAUNCH, emulated on one GPU with
    SF_OPT_SPLIT): one persistent launch per step whose last x-chunk of every tile streams
    DOWNWARD, fused source lists walked backwards there, plane injection pipelined
    downward, boundary ranges signalled on device counters that the comm stream waits on.
    Forward records / final levels / snapshots and the gradient (its adjoint with a receiver
    surface on the two-launch split) are bitwise those of the plain single launch; every step took the
    one-launch path; and the probe copy the comm stream takes as soon as the counters fire
    holds the final boundary planes of the last level (a counter firing before every CTA
    had stored its boundary planes would capture stale values)."""
    S = sf()
    if plane:
        p = _surface_problem(shape, so, 40, 5, seed=61)
    else:
        p = synth.random_problem(3, shape, so, 40, seed=61, nbl=4, nsrc=3, nrec=9)
    h, r = p.h, so // 2
    # sources in the first and the last x-chunk (fused lists, walked both ways)
    p.src_coords[0, 0] = 3.5 * h
    p.src_coords[-1, 0] = (shape[0] - 4.3) * h
    p.m_true = (p.m * 0.94).astype(np.float32)
    d_obs = oracle.forward(p, m=p.m_true)["rec"].astype(np.float32)
    outs = []
    for one in (0, 2):
        prop = make_prop(p)
        prop.set_tuning(2, 0, 0)
        if one:
            prop.set_option(S.SF_OPT_SPLIT, 1)
            prop.set_option(S.SF_OPT_ONE_LAUNCH, 2)
            probe = torch.full((2 * r,) + tuple(shape[1:]), float("nan"), device="cuda")
            prop.debug_probe(probe)
        rec, u, snaps = prop.forward(dev(p.wavelet), save_every=3)
        torch.cuda.synchronize()
        o = [rec.cpu().numpy(), u.cpu().numpy(), snaps.cpu().numpy()]
        if one:
            pr = probe.cpu().numpy()
            assert np.array_equal(pr[:r], o[1][1][:r]) and np.array_equal(pr[r:], o[1][1][-r:])
        g, J = prop.gradient(dev(p.wavelet), dev(d_obs), save_every=3)
        torch.cuda.synchronize()
        o += [g.cpu().numpy(), J]
        if one:
            n1 = prop.debug_probe(None)
            # the forward and the gradient's forward; the gradient's adjoint only on its non-
            # correlation steps with a small receiver set (GRAD-mode injection stays standalone
            # -> the two-launch split there; a receiver surface is never fused)
            na = 0 if plane else (p.nt - 1) - (p.nt - 1) // 3
            assert n1 == 2 * (p.nt - 1) + na, n1
        outs.append(o)
        prop.close()
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)
    ro = oracle.forward(p)["rec"]
    assert rel(outs[1][0], ro) <= TOL


def test_pdl_launches_bitwise():
    """SF_OPT_PDL (programmatic dependent launches of the stencil and standalone injection
    kernels: each launch overlaps the previous kernel's tail and waits for its writes with
    griddepcontrol.wait): forward records, final levels and the gradient with a receiver
    surface (standalone injection between every adjoint step) are bitwise those of plain
    launches, for r = 4 and r = 6 (narrow-tile z split: two launches per step)."""
    for shape, so in (((30, 44, 64), 8), ((26, 30, 144), 12)):
        p = _surface_problem(shape, so, 40, 7, seed=52, damp=(so == 8))
        p.m_true = (p.m * 0.95).astype(np.float32)
        d_obs = oracle.forward(p, m=p.m_true)["rec"].astype(np.float32)
        outs = []
        for pdl in (0, 1):
            prop = make_prop(p)
            prop.set_option(sf().SF_OPT_PDL, pdl)
            assert prop.tuning()["variant"] == 2
            rec, u, _ = prop.forward(dev(p.wavelet))
            g, J = prop.gradient(dev(p.wavelet), dev(d_obs), save_every=2)
            torch.cuda.synchronize()
            outs.append((rec.cpu().numpy(), u.cpu().numpy(), g.cpu().numpy(), J))
            prop.close()
        for a, b in zip(outs[0], outs[1]):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("shape,so", [((40, 44, 128), 8), ((26, 30, 144), 12)])
def test_autotune_picks_a_configuration_same_bits(shape, so):
    """sf_autotune (setup-time tuning): times every feasible launch configuration
    on a scratch state, keeps the fastest; the forward after it is bitwise the forward with
    the default tuning (every configuration computes the same bits); so is the gradient,
    whose GRAD-mode steps run the layout autotune picked for them (vy_grad)."""
    p = synth.random_problem(3, shape, so, 30, seed=71, nbl=4, nsrc=2, nrec=9)
    d_obs = (np.random.default_rng(3).standard_normal((p.nt, 9)) * 1e-3).astype(np.float32)
    ref = gpu_forward(p)
    prop = make_prop(p)
    g0, J0 = prop.gradient(dev(p.wavelet), dev(d_obs), save_every=2)
    g0 = g0.cpu().numpy()
    t = prop.autotune(steps=4)
    assert t["variant"] in (1, 2) and t["ms_per_step"] > 0
    tun = prop.tuning()
    assert tun["variant"] == t["variant"]
    assert tun["vy_grad"] in ((2, 4) if t["variant"] == 2 else (0,))
    assert tun["balance"] in (0, 1) and tun["balance_grad"] in (0, 1)
    rec, u, _ = prop.forward(dev(p.wavelet))
    g, J = prop.gradient(dev(p.wavelet), dev(d_obs), save_every=2)
    torch.cuda.synchronize()
    assert np.array_equal(rec.cpu().numpy(), ref[0]) and np.array_equal(u.cpu().numpy(), ref[1])
    assert np.array_equal(g.cpu().numpy(), g0) and J == J0
    prop.set_tuning(2, 4, 0)  # explicit layouts apply to every mode
    assert prop.tuning()["vy_grad"] == 4
    prop.close()


@pytest.mark.parametrize("so", [10, 12, 14, 16])
def test_wide_layout_bitwise(so):
    """The wide TMA layout (tuning vy = 3, r >= 5: 2 rows x 2 z per thread, 11 consumer warps,
    22 x 64 tiles): forward records / final levels / snapshots (SAVE), the gradient (GRAD, with
    the fused source lists in the forward) are bitwise those of the default layout and of the
    generic kernel, and match the oracle.  Ragged tiles in y (45 rows) and z (132 columns)."""
    p = synth.random_problem(3, (37, 45, 132), so, 40, seed=83, nbl=5, nsrc=2, nrec=9)
    p.m_true = (p.m * 0.93).astype(np.float32)
    d_obs = oracle.forward(p, m=p.m_true)["rec"].astype(np.float32)
    outs = []
    for variant, vy in ((2, 3), (2, 2), (1, 0)):
        prop = make_prop(p)
        prop.set_tuning(variant, vy, 0)
        assert prop.tuning()["vy"] == (vy if variant == 2 else 0)
        rec, u, snaps = prop.forward(dev(p.wavelet), save_every=3)
        g, J = prop.gradient(dev(p.wavelet), dev(d_obs), save_every=3)
        torch.cuda.synchronize()
        outs.append((rec.cpu().numpy(), u.cpu().numpy(), snaps.cpu().numpy(), g.cpu().numpy(), J))
        prop.close()
    for o in outs[1:]:
        for a, b in zip(outs[0], o):
            assert np.array_equal(a, b)
    ro, uo, _ = oracle_forward(p)
    assert rel(outs[0][0], ro) <= TOL and rel(outs[0][1][1], uo[1]) <= TOL


@pytest.mark.parametrize("so,shape", [(2, (23, 45, 132)), (4, (37, 45, 200)), (8, (37, 45, 132)),
                                      (8, (29, 33, 256)), (12, (37, 45, 132)), (12, (31, 40, 200)),
                                      (16, (37, 45, 132)), (16, (30, 17, 128))])
def test_ws_layout_bitwise(so, shape):
    """The warp-specialised TMA layout (tuning vy = 4: 8 consumer warps x 2 rows x 4 z, 16 x 128
    tiles, a producer warpgroup handing its registers to the consumers with setmaxnreg):
    forward records / final levels / snapshots (SAVE), the gradient (GRAD) and the adjoint's
    source records are bitwise those of the default layout and of the generic kernel, and
    match the oracle.  Ragged tiles in y; n2 = 132 puts a 4-column remainder on the narrow
    64 x 32 tiles at r >= 5; n2 = 200 / 256 keep the fused source lists of the forward."""
    p = synth.random_problem(3, shape, so, 40, seed=97 + so, nbl=5, nsrc=2, nrec=9)
    p.m_true = (p.m * 0.93).astype(np.float32)
    d_obs = oracle.forward(p, m=p.m_true)["rec"].astype(np.float32)
    res = np.random.default_rng(so).standard_normal((p.nt, 9)).astype(np.float32)
    outs = []
    for variant, vy in ((2, 4), (2, 2), (1, 0)):
        prop = make_prop(p)
        prop.set_tuning(variant, vy, 0)
        assert prop.tuning()["vy"] == (vy if variant == 2 else 0)
        rec, u, snaps = prop.forward(dev(p.wavelet), save_every=3)
        g, J = prop.gradient(dev(p.wavelet), dev(d_obs), save_every=3)
        srca, v, _ = prop.adjoint(dev(res))
        torch.cuda.synchronize()
        outs.append((rec.cpu().numpy(), u.cpu().numpy(), snaps.cpu().numpy(), g.cpu().numpy(), J,
                     srca.cpu().numpy(), v.cpu().numpy()))
        prop.close()
    for o in outs[1:]:
        for a, b in zip(outs[0], o):
            assert np.array_equal(a, b)
    ro, uo, _ = oracle_forward(p)
    assert rel(outs[0][0], ro) <= TOL and rel(outs[0][1][1], uo[1]) <= TOL


@pytest.mark.parametrize("so,shape,vy,ctas", [(4, (37, 45, 200), 2, 0), (8, (29, 33, 256), 4, 5),
                                              (12, (37, 45, 132), 4, 0), (12, (31, 40, 200), 2, 7),
                                              (16, (30, 17, 128), 4, 3), (16, (41, 45, 132), 2, 0)])
def test_balanced_split_bitwise(so, shape, vy, ctas):
    """SF_OPT_BALANCE = 1 (each persistent CTA streams an equal contiguous run of the tile-major
    (tile, plane) sequence, cut at tile boundaries) gives the bits of the chunked split (0):
    forward records / levels / snapshots with fused sources, the gradient and the adjoint;
    CTA counts that put segment starts mid-tile (ctas 3, 5, 7), narrow remainder tiles
    (n2 = 132, r >= 5); and it matches the oracle."""
    p = synth.random_problem(3, shape, so, 36, seed=131 + so, nbl=5, nsrc=2, nrec=9)
    p.m_true = (p.m * 0.93).astype(np.float32)
    d_obs = oracle.forward(p, m=p.m_true)["rec"].astype(np.float32)
    res = np.random.default_rng(so).standard_normal((p.nt, 9)).astype(np.float32)
    outs = []
    for bal in (1, 0):
        prop = make_prop(p)
        prop.set_tuning(2, vy, ctas)
        prop.set_option(sf().SF_OPT_BALANCE, bal)
        rec, u, snaps = prop.forward(dev(p.wavelet), save_every=3)
        g, J = prop.gradient(dev(p.wavelet), dev(d_obs), save_every=3)
        srca, v, _ = prop.adjoint(dev(res))
        torch.cuda.synchronize()
        outs.append((rec.cpu().numpy(), u.cpu().numpy(), snaps.cpu().numpy(), g.cpu().numpy(), J,
                     srca.cpu().numpy(), v.cpu().numpy()))
        prop.close()
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)
    ro, uo, _ = oracle_forward(p)
    assert rel(outs[0][0], ro) <= TOL and rel(outs[0][1][1], uo[1]) <= TOL


@pytest.mark.parametrize("so,sep", [(4, False), (8, False), (4, True), (16, False)])
def test_loop2d_bitwise(so, sep):
    """SF_OPT_LOOP2D (a small 2D grid runs its whole forward / adjoint time loop in one CTA,
    both levels in shared memory): records, final levels and the adjoint's source records
    are bitwise those of the per-step kernels, and the forward matches the oracle.  Damping
    as the beta array or as separable profiles; ragged extents."""
    p = synth.random_problem(2, (61, 47), so, 80, seed=91, nbl=6, nsrc=2, nrec=9)
    res = np.random.default_rng(4).standard_normal((p.nt, 9)).astype(np.float32)
    outs = []
    for loop in (1, 0):
        prop = sf().Propagator(dev(p.m), None if sep else dev(p.damp), shape=p.shape, h=p.h,
                               space_order=p.space_order, nt=p.nt, dt=p.dt,
                               src_coords=p.src_coords.astype(np.float64),
                               rec_coords=p.rec_coords.astype(np.float64), sigma=p.sigma if sep else None)
        prop.set_option(sf().SF_OPT_LOOP2D, loop)
        prop.set_profiling(True)
        prop.profile(reset=True)
        rec, u, _ = prop.forward(dev(p.wavelet))
        srca, v, _ = prop.adjoint(dev(res))
        torch.cuda.synchronize()
        n = prop.profile(reset=True)["stencil_launches"]
        assert n == (2 if loop else 2 * (p.nt - 1)), n
        outs.append([x.cpu().numpy() for x in (rec, u, srca, v)])
        prop.close()
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)
    if not sep:
        ro, uo, _ = oracle_forward(p)
        assert rel(outs[0][0], ro) <= TOL and rel(outs[0][1][1], uo[1]) <= TOL


@pytest.mark.parametrize("so,damp,shape,nt", [
    (8, True, (30, 21, 252), 41),    # 3 z tiles (the last 12 columns), 3 y tiles (ragged), odd step count
    (8, False, (25, 17, 132), 40),   # no damping array, even step count (ends with one single step)
    (6, True, (22, 33, 256), 27),
    (4, True, (19, 26, 248), 31),
    (2, True, (14, 9, 124), 20),
    (8, True, (12, 10, 120), 3),     # one two-step launch
    (8, True, (12, 10, 120), 2),     # one single step only
])
def test_tblock_bitwise(so, damp, shape, nt):
    """SF_OPT_TBLOCK (two time steps per launch, stencil_tb2.cuh): records and final levels
    bitwise those of the single-step path, sources in many tiles (random wavelets, sources
    on the grown tiles' halos), and the forward matches the oracle."""
    p = synth.random_problem(3, shape, so, nt, seed=so + nt, nbl=2 if damp else 0, nsrc=12, nrec=9,
                             damp=damp, random_wavelet=True)
    outs = []
    for tb in (1, 0):
        prop = make_prop(p)
        if tb:
            prop.set_option(sf().SF_OPT_TBLOCK, 1)
        prop.set_profiling(True)
        prop.profile(reset=True)
        rec, u, _ = prop.forward(dev(p.wavelet))
        torch.cuda.synchronize()
        n = prop.profile(reset=True)["stencil_launches"]
        if tb:
            assert n == (nt - 1) // 2 + (nt - 1) % 2, n
        outs.append([x.cpu().numpy() for x in (rec, u)])
        prop.close()
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)
    ro, uo, _ = oracle_forward(p)
    assert rel(outs[0][0], ro) <= TOL and rel(outs[0][1][1], uo[1]) <= TOL


def test_tblock_rejects_unsupported():
    """SF_OPT_TBLOCK needs space order <= 8, 3D, n_z % 4 == 0: an error, not a fallback."""
    p = synth.random_problem(3, (12, 10, 64), 10, 5, seed=1, nbl=2)
    prop = make_prop(p)
    with pytest.raises(sf().SfError):
        prop.set_option(sf().SF_OPT_TBLOCK, 1)
    prop.close()
