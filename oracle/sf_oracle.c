/*
 * sf_oracle.c -- ORACLE: plain, slow, obviously-correct fp64 CPU implementation of
 * the acoustic finite-difference path of Lange et al., "Optimised finite difference
 * computation from symbolic equations" (Devito, SciPy 2017, arxiv 1707.03776).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant generator with the CUDA path (paper_1707_03776_b200/),
 * and never imports it.
 *
 * Citations: P:n = PAPER.md line n (section "Seismic Inversion Example" P:455-680);
 * C1..C20 = the readings of silent/ambiguous points listed in DESIGN.md §3.
 *
 * What is computed (every function follows its definition literally, fp64 throughout):
 *   or_fd_weights  : centred 2nd-derivative FD weights of order `so` by Fornberg's
 *                    recursion (space order parameterisable: P:544).
 *   or_laplacian   : L_h u = sum_axes sum_{k=-r..r} w_|k| u(p + k e_a) / h^2, zero
 *                    ghost halo of width r (reading C6); `u.laplace`.
 *   or_point_stencil / or_interpolate / or_inject :
 *                    linear (bi/tri-linear) interpolation between sparse points and
 *                    the grid, and its transpose (reading C11).
 *   or_forward     : for n = 0..nt-2
 *                      u^{n+1} = [2 m u^n - (m - eta dt/2) u^{n-1} + dt^2 L_h u^n] / (m + eta dt/2)
 *                      (= solve(m*u.dt2 - u.laplace + eta*u.dt, u.forward), P:547-549,
 *                       centred u.dt: reading C1)
 *                      u^{n+1}[c] += W_{s,c} * wavelet[n][s] * dt^2 / m[c]   (src.inject; C3)
 *                      rec[n+1][r] = sum_c W_{r,c} u^{n+1}[c]                (rec.interpolate; C4)
 *                    rec[0] = P u^0; optional snapshots u^n, n % k == 0 (BASELINE north_star).
 *   or_adjoint     : for n = nt-1..1
 *                      v^{n-1} = [2 m v^n - (m - eta dt/2) v^{n+1} + dt^2 L_h v^n] / (m + eta dt/2)
 *                      (= solve(m*v.dt2 - v.laplace - eta*v.dt, v.backward); C2)
 *                      v^{n-1}[c] += W_{r,c} * res[n][r] * dt^2 / m[c]        (rec.inject)
 *                      srca[n-1][s] = sum_c W_{s,c} v^{n-1}[c]                (srca.interpolate)
 *                    srca[nt-1] = P v^{nt-1}.  Optional gradient (not in the paper; north_star
 *                    "g += v * u_tt", readings C13/C14):
 *                      g -= k * u^n * (v^{n+1} - 2 v^n + v^{n-1}) / dt^2  for n % k == 0, n >= 1.
 *
 * The paper's two other example workloads (readings C21/C22 in DESIGN.md):
 *   or_convection2d : linear 2D convection, forward Euler in time, backward (upwind) in
 *                     space, Eq. 2:
 *                       u^{n+1}_ij = u^n_ij - c dt/dx (u^n_ij - u^n_{i-1,j}) - c dt/dy (u^n_ij - u^n_{i,j-1})
 *                     on the interior 1 <= i < n0-1, 1 <= j < n1-1; edge points keep their
 *                     initial values (Dirichlet, C21).
 *   or_laplace2d    : Laplace equation by Jacobi sweeps, Eq. 4:
 *                       p_ij = (dy^2 (pn_{i+1,j} + pn_{i-1,j}) + dx^2 (pn_{i,j+1} + pn_{i,j-1}))
 *                              / (2 (dx^2 + dy^2))
 *                     on the interior, then the boundary expressions in the listing's order
 *                     (P:411-414): p[x,0] = 0; p[x,n1-1] = bc[x]; p[0,y] = p[1,y];
 *                     p[n0-1,y] = p[n0-2,y]; buffers swap every sweep; after each sweep
 *                     l1 = sum(|p| - |pn|) / sum(|pn|); stop when l1 <= tol (C22).
 *
 * Layout: row-major [n0][n1][n2] (2D: [n0][n1]), last axis fastest.  Sparse data are
 * time-major [nt][npoint] (reading C12).  Coordinates in metres from index 0.
 * Return codes: 0 ok, 1 invalid argument, 5 sparse point out of domain.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_MAXR 8

/* ---------------------------------------------------------------------------------
 * Fornberg, "Generation of finite difference formulas on arbitrarily spaced grids"
 * (Math. Comp. 1988): weights c[j] for the M-th derivative at x0 on nodes x[0..N-1].
 * Textbook recursion, O(N^2 M), fp64.
 * ------------------------------------------------------------------------------- */
static void fornberg(int M, double x0, const double *x, int N, double *out)
{
    /* delta[m][n][nu], m <= M, n < N, nu <= n */
    double *d = (double *)calloc((size_t)(M + 1) * N * N, sizeof(double));
#define D(m, n, nu) d[((size_t)(m) * N + (n)) * N + (nu)]
    D(0, 0, 0) = 1.0;
    double c1 = 1.0;
    for (int n = 1; n < N; ++n) {
        double c2 = 1.0;
        for (int nu = 0; nu < n; ++nu) {
            double c3 = x[n] - x[nu];
            c2 *= c3;
            for (int m = 0; m <= (n < M ? n : M); ++m) {
                double prev = (m > 0) ? D(m - 1, n - 1, nu) : 0.0;
                D(m, n, nu) = ((x[n] - x0) * D(m, n - 1, nu) - m * prev) / c3;
            }
        }
        for (int m = 0; m <= (n < M ? n : M); ++m) {
            double prev = (m > 0) ? D(m - 1, n - 1, n - 1) : 0.0;
            D(m, n, n) = c1 / c2 * (m * prev - (x[n - 1] - x0) * D(m, n - 1, n - 1));
        }
        c1 = c2;
    }
    for (int j = 0; j < N; ++j) out[j] = D(M, N - 1, j);
#undef D
    free(d);
}

/* w[0..r]: w[0] = centre weight, w[k] = weight at offsets +-k (units 1/h^2 omitted). */
int or_fd_weights(int so, double *w)
{
    if (so < 2 || so > 2 * OR_MAXR || (so & 1) || !w) return 1;
    int r = so / 2, N = so + 1;
    double x[2 * OR_MAXR + 1], c[2 * OR_MAXR + 1];
    for (int j = 0; j < N; ++j) x[j] = (double)(j - r);
    fornberg(2, 0.0, x, N, c);
    for (int k = 0; k <= r; ++k) w[k] = c[r + k];
    return 0;
}

static int64_t npts(int ndim, const int64_t *n)
{
    int64_t N = 1;
    for (int a = 0; a < ndim; ++a) N *= n[a];
    return N;
}

/* L_h u at the point with multi-index p and flat offset off (reading C6: zero ghost halo):
 * sum over axes a and offsets k = -r..r of w_|k| u(p + k e_a), divided by h^2. */
static double lap_point(const double *u, int ndim, const int64_t *n, const int64_t *stride,
                        const int64_t *p, int64_t off, const double *w, int r, double h)
{
    double acc = 0.0;
    for (int a = 0; a < ndim; ++a) {
        for (int k = -r; k <= r; ++k) {
            const int64_t q = p[a] + k;
            const double val = (q < 0 || q >= n[a]) ? 0.0 : u[off + k * stride[a]];
            acc += w[k < 0 ? -k : k] * val;
        }
    }
    return acc / (h * h);
}

static void strides_of(int ndim, const int64_t *n, int64_t *stride)
{
    stride[ndim - 1] = 1;
    for (int a = ndim - 2; a >= 0; --a) stride[a] = stride[a + 1] * n[a + 1];
}

static void unravel(int ndim, const int64_t *n, int64_t off, int64_t *p)
{
    for (int a = ndim - 1; a >= 0; --a) {
        p[a] = off % n[a];
        off /= n[a];
    }
}

int or_laplacian(int ndim, const int64_t *n, double h, int so, const double *u, double *out)
{
    if (ndim < 1 || ndim > 3) return 1;
    double w[OR_MAXR + 1];
    if (or_fd_weights(so, w)) return 1;
    int r = so / 2;
    int64_t N = npts(ndim, n), stride[3];
    strides_of(ndim, n, stride);
#pragma omp parallel for schedule(static)
    for (int64_t off = 0; off < N; ++off) {
        int64_t p[3];
        unravel(ndim, n, off, p);
        out[off] = lap_point(u, ndim, n, stride, p, off, w, r, h);
    }
    return 0;
}

/* Reading C11: pos = x/h; base = min(floor(pos), n-2); xi = pos - base; corner
 * weights = prod over axes of (1-xi) or xi; corners ordered last-axis fastest.
 * Out of [0, n-1] on any axis -> error 5 (never clipped). */
int or_point_stencil(int ndim, const int64_t *n, double h, const double *coord,
                     int64_t *idx, double *W)
{
    int64_t base[3];
    double xi[3];
    for (int a = 0; a < ndim; ++a) {
        double pos = coord[a] / h;
        if (!(pos >= 0.0) || pos > (double)(n[a] - 1)) return 5;
        int64_t b = (int64_t)floor(pos);
        if (b > n[a] - 2) b = n[a] - 2;
        base[a] = b;
        xi[a] = pos - (double)b;
    }
    int nc = 1 << ndim;
    for (int c = 0; c < nc; ++c) {
        double wt = 1.0;
        int64_t off = 0;
        for (int a = 0; a < ndim; ++a) {
            int bit = (c >> (ndim - 1 - a)) & 1;
            wt *= bit ? xi[a] : (1.0 - xi[a]);
            off = off * n[a] + base[a] + bit;
        }
        idx[c] = off;
        W[c] = wt;
    }
    return 0;
}

/* out[p] = sum_c W_{p,c} u[c]   (pt.interpolate) */
int or_interpolate(int ndim, const int64_t *n, double h, int np, const double *coords,
                   const double *u, double *out)
{
    for (int p = 0; p < np; ++p) {
        int64_t idx[8];
        double W[8];
        int e = or_point_stencil(ndim, n, h, coords + (size_t)p * ndim, idx, W);
        if (e) return e;
        double acc = 0.0;
        for (int c = 0; c < (1 << ndim); ++c) acc += W[c] * u[idx[c]];
        out[p] = acc;
    }
    return 0;
}

/* u[c] += W_{p,c} * vals[p] * (m ? dt^2/m[c] : 1)   (pt.inject) */
int or_inject(int ndim, const int64_t *n, double h, int np, const double *coords,
              const double *vals, const double *m, double dt, double *u)
{
    for (int p = 0; p < np; ++p) {
        int64_t idx[8];
        double W[8];
        int e = or_point_stencil(ndim, n, h, coords + (size_t)p * ndim, idx, W);
        if (e) return e;
        for (int c = 0; c < (1 << ndim); ++c) {
            double s = m ? dt * dt / m[idx[c]] : 1.0;
            u[idx[c]] += W[c] * vals[p] * s;
        }
    }
    return 0;
}

/* one explicit leapfrog update: nxt = [2 m cur - (m - eta dt/2) prv + dt^2 L_h cur] / (m + eta dt/2) */
static void leapfrog(int ndim, const int64_t *n, double h, const double *w, int r, double dt,
                     const double *m, const double *damp, const double *cur, const double *prv,
                     double *nxt)
{
    int64_t stride[3];
    strides_of(ndim, n, stride);
    const int64_t rows = npts(ndim, n) / n[ndim - 1];  /* all axes but the last */
    const int64_t nl = n[ndim - 1];
#pragma omp parallel for schedule(static)
    for (int64_t row = 0; row < rows; ++row) {
        int64_t p[3];
        unravel(ndim, n, row * nl, p);
        for (int64_t i = 0; i < nl; ++i) {
            const int64_t off = row * nl + i;
            p[ndim - 1] = i;
            double L = lap_point(cur, ndim, n, stride, p, off, w, r, h);
            double eta = damp ? damp[off] : 0.0;
            double mm = m[off];
            nxt[off] = (2.0 * mm * cur[off] - (mm - 0.5 * eta * dt) * prv[off] + dt * dt * L)
                       / (mm + 0.5 * eta * dt);
        }
    }
}

static int check_common(int ndim, const int64_t *n, double h, int so, int nt, double dt,
                        const double *m)
{
    if (ndim < 2 || ndim > 3 || !n || !m) return 1;
    if (so < 2 || so > 16 || (so & 1)) return 1;
    if (nt < 2 || !(dt > 0.0) || !(h > 0.0)) return 1;
    for (int a = 0; a < ndim; ++a)
        if (n[a] < 2) return 1;
    return 0;
}

/*
 * u_state [2][N]: in (u^{-1}, u^0), out (u^{nt-2}, u^{nt-1}).
 * rec [nt][nrec] (may be NULL if nrec == 0); snaps [floor((nt-1)/k)+1][N] or NULL.
 */
int or_forward(int ndim, const int64_t *n, double h, int so, int nt, double dt,
               const double *m, const double *damp,
               int nsrc, const double *src_coords, const double *wavelet,
               int nrec, const double *rec_coords, double *rec,
               double *u_state, int save_every, double *snaps)
{
    int e = check_common(ndim, n, h, so, nt, dt, m);
    if (e) return e;
    double w[OR_MAXR + 1];
    or_fd_weights(so, w);
    int r = so / 2;
    int64_t N = npts(ndim, n);
    double *prv = (double *)malloc(sizeof(double) * N);
    double *cur = (double *)malloc(sizeof(double) * N);
    double *nxt = (double *)malloc(sizeof(double) * N);
    memcpy(prv, u_state, sizeof(double) * N);
    memcpy(cur, u_state + N, sizeof(double) * N);
    double *sv = (double *)malloc(sizeof(double) * (nsrc > 0 ? nsrc : 1));
    if (nrec > 0) {
        e = or_interpolate(ndim, n, h, nrec, rec_coords, cur, rec);
        if (e) goto done;
    }
    if (snaps && save_every > 0) memcpy(snaps, cur, sizeof(double) * N);
    for (int t = 0; t <= nt - 2; ++t) {
        leapfrog(ndim, n, h, w, r, dt, m, damp, cur, prv, nxt);
        if (nsrc > 0) {
            for (int s = 0; s < nsrc; ++s) sv[s] = wavelet[(size_t)t * nsrc + s];
            e = or_inject(ndim, n, h, nsrc, src_coords, sv, m, dt, nxt);
            if (e) goto done;
        }
        if (nrec > 0) {
            e = or_interpolate(ndim, n, h, nrec, rec_coords, nxt, rec + (size_t)(t + 1) * nrec);
            if (e) goto done;
        }
        if (snaps && save_every > 0 && (t + 1) % save_every == 0)
            memcpy(snaps + (size_t)((t + 1) / save_every) * N, nxt, sizeof(double) * N);
        double *tmp = prv;
        prv = cur;
        cur = nxt;
        nxt = tmp;
    }
    memcpy(u_state, prv, sizeof(double) * N);
    memcpy(u_state + N, cur, sizeof(double) * N);
done:
    free(prv); free(cur); free(nxt); free(sv);
    return e;
}

/*
 * v_state [2][N]: in (v^{nt}, v^{nt-1}), out (v^1, v^0).
 * res [nt][nrec] injected at the receivers; srca [nt][nsrc] interpolated at the sources.
 * If grad != NULL: snaps holds u^n for n % k == 0 (slot n/k) and
 *   grad -= k * u^n * (v^{n+1} - 2 v^n + v^{n-1}) / dt^2  for every n % k == 0, 1 <= n <= nt-1.
 */
int or_adjoint(int ndim, const int64_t *n, double h, int so, int nt, double dt,
               const double *m, const double *damp,
               int nrec, const double *rec_coords, const double *res,
               int nsrc, const double *src_coords, double *srca,
               double *v_state, int save_every, const double *snaps, double *grad)
{
    int e = check_common(ndim, n, h, so, nt, dt, m);
    if (e) return e;
    if (grad && (!snaps || save_every < 1)) return 1;
    double w[OR_MAXR + 1];
    or_fd_weights(so, w);
    int r = so / 2;
    int64_t N = npts(ndim, n);
    double *vp1 = (double *)malloc(sizeof(double) * N); /* v^{n+1} */
    double *v0 = (double *)malloc(sizeof(double) * N);  /* v^n     */
    double *vm1 = (double *)malloc(sizeof(double) * N); /* v^{n-1} */
    memcpy(vp1, v_state, sizeof(double) * N);
    memcpy(v0, v_state + N, sizeof(double) * N);
    double *rv = (double *)malloc(sizeof(double) * (nrec > 0 ? nrec : 1));
    if (nsrc > 0) {
        e = or_interpolate(ndim, n, h, nsrc, src_coords, v0, srca + (size_t)(nt - 1) * nsrc);
        if (e) goto done;
    }
    for (int t = nt - 1; t >= 1; --t) {
        leapfrog(ndim, n, h, w, r, dt, m, damp, v0, vp1, vm1);
        if (nrec > 0) {
            for (int q = 0; q < nrec; ++q) rv[q] = res[(size_t)t * nrec + q];
            e = or_inject(ndim, n, h, nrec, rec_coords, rv, m, dt, vm1);
            if (e) goto done;
        }
        if (nsrc > 0) {
            e = or_interpolate(ndim, n, h, nsrc, src_coords, vm1, srca + (size_t)(t - 1) * nsrc);
            if (e) goto done;
        }
        if (grad && t % save_every == 0) {
            const double *u = snaps + (size_t)(t / save_every) * N;
            double k = (double)save_every;
#pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < N; ++i)
                grad[i] -= k * u[i] * (vp1[i] - 2.0 * v0[i] + vm1[i]) / (dt * dt);
        }
        double *tmp = vp1;
        vp1 = v0;
        v0 = vm1;
        vm1 = tmp;
    }
    memcpy(v_state, vp1, sizeof(double) * N);
    memcpy(v_state + N, v0, sizeof(double) * N);
done:
    free(vp1); free(v0); free(vm1); free(rv);
    return e;
}

/* ---------------------------------------------------------------------------------
 * Linear convection (Eq. 2; reading C21).  u: [n0][n1] in/out (fp64).
 * ------------------------------------------------------------------------------- */
int or_convection2d(const int64_t *n, double c, double dt, double dx, double dy, int nt, double *u)
{
    if (!n || !u || n[0] < 2 || n[1] < 2 || nt < 0 || !(dx > 0.0) || !(dy > 0.0)) return 1;
    const int64_t n0 = n[0], n1 = n[1];
    double *un = (double *)malloc(sizeof(double) * (size_t)(n0 * n1));
    if (!un) return 1;
    const double ax = c * dt / dx, ay = c * dt / dy;
    for (int t = 0; t < nt; ++t) {
        memcpy(un, u, sizeof(double) * (size_t)(n0 * n1));
        for (int64_t i = 1; i < n0 - 1; ++i)
            for (int64_t j = 1; j < n1 - 1; ++j) {
                const double uij = un[i * n1 + j];
                u[i * n1 + j] = uij - ax * (uij - un[(i - 1) * n1 + j]) - ay * (uij - un[i * n1 + j - 1]);
            }
    }
    free(un);
    return 0;
}

/* ---------------------------------------------------------------------------------
 * Laplace / Jacobi (Eq. 4; boundary listing P:411-414; loop P:433-447;
 * reading C22).  p: [n0][n1] in = the initial buffer pn, out = the last computed p;
 * bc: [n0] the prescribed boundary row.  Stops after the first sweep with l1 <= tol or
 * after max_iter sweeps; *iters = sweeps done, *l1 = the last l1.
 * ------------------------------------------------------------------------------- */
int or_laplace2d(const int64_t *n, double dx, double dy, const double *bc, double tol, int max_iter,
                 double *p, int *iters, double *l1)
{
    if (!n || !p || !bc || n[0] < 3 || n[1] < 3 || max_iter < 0 || !(dx > 0.0) || !(dy > 0.0)) return 1;
    const int64_t n0 = n[0], n1 = n[1], N = n0 * n1;
    double *pn = (double *)malloc(sizeof(double) * (size_t)N);
    if (!pn) return 1;
    const double dx2 = dx * dx, dy2 = dy * dy;
    double l1v = 1.0;
    int it = 0;
    while (it < max_iter && l1v > tol) {
        memcpy(pn, p, sizeof(double) * (size_t)N);
        for (int64_t i = 1; i < n0 - 1; ++i)
            for (int64_t j = 1; j < n1 - 1; ++j)
                p[i * n1 + j] = (dy2 * (pn[(i + 1) * n1 + j] + pn[(i - 1) * n1 + j]) +
                                 dx2 * (pn[i * n1 + j + 1] + pn[i * n1 + j - 1])) / (2.0 * (dx2 + dy2));
        for (int64_t i = 0; i < n0; ++i) p[i * n1 + 0] = 0.0;
        for (int64_t i = 0; i < n0; ++i) p[i * n1 + n1 - 1] = bc[i];
        for (int64_t j = 0; j < n1; ++j) p[0 * n1 + j] = p[1 * n1 + j];
        for (int64_t j = 0; j < n1; ++j) p[(n0 - 1) * n1 + j] = p[(n0 - 2) * n1 + j];
        double num = 0.0, den = 0.0;
        for (int64_t k = 0; k < N; ++k) {
            num += fabs(p[k]) - fabs(pn[k]);
            den += fabs(pn[k]);
        }
        l1v = num / den;
        ++it;
    }
    free(pn);
    if (iters) *iters = it;
    if (l1) *l1 = l1v;
    return 0;
}

int or_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
