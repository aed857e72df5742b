/*
 * gsr_oracle.c -- TEST INFRASTRUCTURE ONLY (never on the product path).
 *
 * A plain, slow, obviously-correct float64 CPU implementation of GSASR's
 * scale-aware 2D Gaussian rasterization (arXiv 2501.06838), written from the
 * paper. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library. It shares no code, header,
 * constant or helper with the CUDA path (paper_2501_06838_b200/csrc).
 *
 * What it follows (PAPER.md line numbers, "P:<line>"):
 *   Eq. 1  G(x,y) = alpha * c * f(x,y)
 *   Eq. 2  f(x,y) = (2 pi sx sy sqrt(1-rho^2))^-1 *
 *                   exp[-1/(2(1-rho^2)) (dx^2/sx^2 - 2 rho dx dy/(sx sy) + dy^2/sy^2)]
 *                                                                     P:1349-1357
 *   Eq. 4  I_SR(x,y;s) = sum_i G_i(x/s, y/s), x in [0,sW-1], y in [0,sH-1]
 *                                                                     P:1395-1401
 *   Alg. 1 zero-init (sH, sW, 3); for each Gaussian, for each pixel, if
 *          |x - mu_x| < r s H and |y - mu_y| < r s W accumulate G_i(x/s,y/s)
 *                                                                     P:1368-1392
 *   r = 0.1 default
 *
 * Readings of silent/garbled points:
 *   R1  window axis pairing: x <-> W, y <-> H (Alg. 1 pairs x with H; Eq. 4
 *       pairs x with sW).
 *   R2  window test in LR units: |x/s - mu_x| < r W, |y/s - mu_y| < r H, strict.
 *       Integer form (normative for GPU and rect mode):
 *         x0 = floor(s*(mu_x - r*W)) + 1,  x1 = ceil(s*(mu_x + r*W)) - 1
 *       evaluated in IEEE fp64 in exactly this order (no FMA), bounds clamped
 *       to +-2^30 before conversion, then clipped to [0,Ws-1] (y likewise).
 *   R3  sample point (x/s, y/s), no half-pixel centring.
 *   R4  output size floor(s*H) x floor(s*W) in fp64.
 *   R7  |rho| < 1 precondition; no clamping of anything (R8).
 *   R20 invalid Gaussian (non-finite field, sigma<=0, |rho|>=1): contributes 0
 *       and gets zero gradient.
 *   R21 evaluation support (an implementation reading, not the paper's): every
 *       pair with Q >= 13.5^2 has exp(-Q/2) < 2^-131 (below the smallest fp32
 *       normal, i.e. exactly 0 in the fp32 kernels); since Q >= (dx/sx)^2 and
 *       Q >= (dy/sy)^2, such pairs include every pixel outside the box
 *       |x/s - mu_x| <= 13.5 sx, |y/s - mu_y| <= 13.5 sy. Integer box:
 *         bx0 = floor(s*(mu_x - 13.5*sx)),  bx1 = ceil(s*(mu_x + 13.5*sx))
 *       in IEEE fp64 in exactly this order, clamped to +-2^30. The support
 *       rect is window rect (R2) intersected with the box; its unclipped
 *       origin is max(window origin, box origin). Mode "support" renders over
 *       it; the difference to the window sum is pinned below 1e-30.
 *   R22 scale vector ("an upsampling scale vector"; NEXT-4): s = (sw, sh),
 *       sw along x <-> W, sh along y <-> H. Every "s" above applies per axis:
 *       output floor(sh*H) x floor(sw*W); sample (x/sw, y/sh); window and box
 *       bounds along x use sw, along y sh. sw = sh is the paper's scalar s.
 *   Summation order: per pixel, ascending Gaussian index (brute and rect modes
 *   therefore give bit-identical results).
 *
 * Pins (tests/test_oracle_*.py): Eq. 2 closed forms; Poisson-summation
 * moments (mass 1, mean mu, covariance [[sx^2, rho sx sy],[., sy^2]]);
 * window-truncation bound; coordinate-normalisation invariance; integer-scale
 * consistency; linearity/symmetry; brute == rect bit-identity; central finite
 * differences for every gradient; brute-force tile binning vs enumeration.
 *
 * Build: gcc -O2 -fno-fast-math -ffp-contract=off -fopenmp -shared -fPIC
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_PI 3.14159265358979323846

/* ------------------------------------------------------------------------- */
/* Helpers that restate the paper.                                            */
/* ------------------------------------------------------------------------- */

/* R20: a Gaussian outside the paper's parameter domain is skipped. */
static int oracle_is_valid(const double* alpha, const double* mu, const double* sigma,
                           const double* rho, const double* color, int64_t i)
{
    double v[9] = {alpha[i], mu[2 * i], mu[2 * i + 1], sigma[2 * i], sigma[2 * i + 1],
                   rho[i], color[3 * i], color[3 * i + 1], color[3 * i + 2]};
    for (int k = 0; k < 9; ++k)
        if (!isfinite(v[k])) return 0;
    if (!(sigma[2 * i] > 0.0) || !(sigma[2 * i + 1] > 0.0)) return 0;
    if (!(fabs(rho[i]) < 1.0)) return 0;
    return 1;
}

/* Eq. 2, literally: the normalised bivariate normal density
 * at offset (dx, dy) = (X - mu_x, Y - mu_y). Also returns the Mahalanobis
 * form Q (the bracket divided by 1 - rho^2) for the gradient. */
static double oracle_density(double dx, double dy, double sx, double sy, double rho,
                             double* Q_out)
{
    double D = 1.0 - rho * rho;
    double bracket = dx * dx / (sx * sx) - 2.0 * rho * dx * dy / (sx * sy) + dy * dy / (sy * sy);
    double Q = bracket / D;
    if (Q_out) *Q_out = Q;
    return exp(-0.5 * Q) / (2.0 * ORACLE_PI * sx * sy * sqrt(D));
}

/* R2: integer window rectangle, unclipped and clipped. Returns 0 if empty. */
static double oracle_clamp_bound(double v)
{
    const double lim = 1073741824.0; /* 2^30 */
    if (v < -lim) return -lim;
    if (v > lim) return lim;
    return v;
}

static int oracle_rect(double mx, double my, int H, int W, double sw, double sh, double r, int Hs, int Ws,
                       int64_t* x0u, int64_t* y0u, int64_t* x0, int64_t* x1, int64_t* y0,
                       int64_t* y1)
{
    double hx = r * (double)W;   /* half-extent along x, LR px (R1) */
    double hy = r * (double)H;   /* half-extent along y, LR px (R1) */
    double lx = sw * (mx - hx);
    double ux = sw * (mx + hx);
    double ly = sh * (my - hy);
    double uy = sh * (my + hy);
    if (isnan(lx) || isnan(ux) || isnan(ly) || isnan(uy)) return 0;
    int64_t ax0 = (int64_t)floor(oracle_clamp_bound(lx)) + 1;
    int64_t ax1 = (int64_t)ceil(oracle_clamp_bound(ux)) - 1;
    int64_t ay0 = (int64_t)floor(oracle_clamp_bound(ly)) + 1;
    int64_t ay1 = (int64_t)ceil(oracle_clamp_bound(uy)) - 1;
    if (x0u) *x0u = ax0;
    if (y0u) *y0u = ay0;
    if (ax0 < 0) ax0 = 0;
    if (ay0 < 0) ay0 = 0;
    if (ax1 > Ws - 1) ax1 = Ws - 1;
    if (ay1 > Hs - 1) ay1 = Hs - 1;
    *x0 = ax0; *x1 = ax1; *y0 = ay0; *y1 = ay1;
    return (ax0 <= ax1) && (ay0 <= ay1);
}

/* R21: window rect intersected with the +-13.5 sigma box (see header). */
#define ORACLE_SUPPORT_SIGMAS 13.5
static int oracle_support_rect(double mx, double my, double sx, double sy, int H, int W,
                               double sw, double sh, double r, int Hs, int Ws, int64_t* x0u, int64_t* y0u,
                               int64_t* x0, int64_t* x1, int64_t* y0, int64_t* y1)
{
    int64_t wx0u, wy0u;
    if (!oracle_rect(mx, my, H, W, sw, sh, r, Hs, Ws, &wx0u, &wy0u, x0, x1, y0, y1)) return 0;
    double tx = ORACLE_SUPPORT_SIGMAS * sx, ty = ORACLE_SUPPORT_SIGMAS * sy;
    double lx = sw * (mx - tx), ux = sw * (mx + tx);
    double ly = sh * (my - ty), uy = sh * (my + ty);
    if (isnan(lx) || isnan(ux) || isnan(ly) || isnan(uy)) return 0;
    int64_t bx0 = (int64_t)floor(oracle_clamp_bound(lx));
    int64_t bx1 = (int64_t)ceil(oracle_clamp_bound(ux));
    int64_t by0 = (int64_t)floor(oracle_clamp_bound(ly));
    int64_t by1 = (int64_t)ceil(oracle_clamp_bound(uy));
    if (x0u) *x0u = wx0u > bx0 ? wx0u : bx0;
    if (y0u) *y0u = wy0u > by0 ? wy0u : by0;
    if (*x0 < bx0) *x0 = bx0;
    if (*x1 > bx1) *x1 = bx1;
    if (*y0 < by0) *y0 = by0;
    if (*y1 > by1) *y1 = by1;
    return (*x0 <= *x1) && (*y0 <= *y1);
}

/* rect of Gaussian i in the given mode: 0 = window (R2), 1 = support (R21) */
static int oracle_rect_mode(int support, const double* mu, const double* sigma, int64_t i, int H,
                            int W, double sw, double sh, double r, int Hs, int Ws, int64_t* x0u,
                            int64_t* y0u, int64_t* x0, int64_t* x1, int64_t* y0, int64_t* y1)
{
    if (support)
        return oracle_support_rect(mu[2 * i], mu[2 * i + 1], sigma[2 * i], sigma[2 * i + 1], H,
                                   W, sw, sh, r, Hs, Ws, x0u, y0u, x0, x1, y0, y1);
    return oracle_rect(mu[2 * i], mu[2 * i + 1], H, W, sw, sh, r, Hs, Ws, x0u, y0u, x0, x1, y0, y1);
}

/* R4 */
void gsr_oracle_out_dims(int H, int W, double sw, double sh, int* Hs, int* Ws)
{
    *Hs = (int)floor(sh * (double)H);
    *Ws = (int)floor(sw * (double)W);
}

void gsr_oracle_set_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int gsr_oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Per-Gaussian rects for tests: out[i*6 + {x0u,y0u,x0,x1,y0,y1}], empty -> x0>x1. */
void gsr_oracle_rects(int64_t n, const double* alpha, const double* mu, const double* sigma,
                      const double* rho, const double* color, int H, int W, double sw, double sh, double r,
                      int support, int64_t* out)
{
    int Hs, Ws;
    gsr_oracle_out_dims(H, W, sw, sh, &Hs, &Ws);
    for (int64_t i = 0; i < n; ++i) {
        int64_t x0u = 0, y0u = 0, x0 = 1, x1 = 0, y0 = 1, y1 = 0;
        if (oracle_is_valid(alpha, mu, sigma, rho, color, i))
            if (!oracle_rect_mode(support, mu, sigma, i, H, W, sw, sh, r, Hs, Ws, &x0u, &y0u, &x0, &x1,
                                  &y0, &y1)) {
                x0 = 1; x1 = 0; y0 = 1; y1 = 0;
            }
        int64_t* o = out + 6 * i;
        o[0] = x0u; o[1] = y0u; o[2] = x0; o[3] = x1; o[4] = y0; o[5] = y1;
    }
}

/* Number of (Gaussian, pixel) pairs that pass the window predicate, restricted
 * to HR rows [row_begin, row_end). */
int64_t gsr_oracle_pair_count(int64_t n, const double* alpha, const double* mu,
                              const double* sigma, const double* rho, const double* color, int H,
                              int W, double sw, double sh, double r, int row_begin, int row_end, int support)
{
    int Hs, Ws;
    gsr_oracle_out_dims(H, W, sw, sh, &Hs, &Ws);
    int64_t total = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (!oracle_is_valid(alpha, mu, sigma, rho, color, i)) continue;
        int64_t x0u, y0u, x0, x1, y0, y1;
        if (!oracle_rect_mode(support, mu, sigma, i, H, W, sw, sh, r, Hs, Ws, &x0u, &y0u, &x0, &x1,
                              &y0, &y1))
            continue;
        if (y0 < row_begin) y0 = row_begin;
        if (y1 > row_end - 1) y1 = row_end - 1;
        if (y0 > y1) continue;
        total += (x1 - x0 + 1) * (y1 - y0 + 1);
    }
    return total;
}

/* ------------------------------------------------------------------------- */
/* Forward (Alg. 1 / Eq. 4).                                                  */
/* mode 0 = brute: every Gaussian at every pixel, literal fp64 predicate.     */
/* mode 1 = rect : every Gaussian over its integer rect (R2).                 */
/* mode 2 = none : untruncated sum (r ignored), for the truncation bound.     */
/* mode 3 = support: over the support rect (R21), as the CUDA path does.      */
/* Output rows [row_begin, row_end) only: out[(y-row_begin)*Ws*3 + x*3 + k].  */
/* ------------------------------------------------------------------------- */
int gsr_oracle_render_fwd(int64_t n, const double* alpha, const double* mu, const double* sigma,
                          const double* rho, const double* color, int H, int W, double sw, double sh,
                          double r, int mode, int row_begin, int row_end, double* out)
{
    int Hs, Ws;
    gsr_oracle_out_dims(H, W, sw, sh, &Hs, &Ws);
    if (row_begin < 0) row_begin = 0;
    if (row_end > Hs) row_end = Hs;
    int rows = row_end - row_begin;
    if (rows <= 0) return 0;
    memset(out, 0, sizeof(double) * (size_t)rows * (size_t)Ws * 3);
    double hx = r * (double)W, hy = r * (double)H;

    if (mode == 0 || mode == 2) {
#pragma omp parallel for schedule(dynamic, 1)
        for (int y = row_begin; y < row_end; ++y) {
            double Y = (double)y / sh;                           /* Eq. 4 sample, R3 */
            for (int x = 0; x < Ws; ++x) {
                double X = (double)x / sw;
                double* px = out + ((size_t)(y - row_begin) * Ws + x) * 3;
                for (int64_t i = 0; i < n; ++i) {               /* ascending i */
                    if (!oracle_is_valid(alpha, mu, sigma, rho, color, i)) continue;
                    double mx = mu[2 * i], my = mu[2 * i + 1];
                    if (mode == 0 && !(fabs(X - mx) < hx && fabs(Y - my) < hy)) continue; /* Alg.1 l.6, R1/R2 */
                    double f = oracle_density(X - mx, Y - my, sigma[2 * i], sigma[2 * i + 1],
                                              rho[i], NULL);
                    for (int k = 0; k < 3; ++k) px[k] += alpha[i] * color[3 * i + k] * f; /* Eq. 1 */
                }
            }
        }
        return 0;
    }
    /* rect mode: rows are distributed over threads; every thread walks the
     * Gaussians in ascending order, so each pixel's sum order is ascending i. */
#pragma omp parallel
    {
        int nt = 1, t = 0;
#ifdef _OPENMP
        nt = omp_get_num_threads();
        t = omp_get_thread_num();
#endif
        for (int64_t i = 0; i < n; ++i) {
            if (!oracle_is_valid(alpha, mu, sigma, rho, color, i)) continue;
            double mx = mu[2 * i], my = mu[2 * i + 1];
            int64_t x0u, y0u, x0, x1, y0, y1;
            if (!oracle_rect_mode(mode == 3, mu, sigma, i, H, W, sw, sh, r, Hs, Ws, &x0u, &y0u, &x0,
                                  &x1, &y0, &y1))
                continue;
            (void)mx; (void)my;
            if (y0 < row_begin) y0 = row_begin;
            if (y1 > row_end - 1) y1 = row_end - 1;
            for (int64_t y = y0; y <= y1; ++y) {
                if ((y % nt) != t) continue;
                double Y = (double)y / sh;
                for (int64_t x = x0; x <= x1; ++x) {
                    double X = (double)x / sw;
                    double f = oracle_density(X - mx, Y - my, sigma[2 * i], sigma[2 * i + 1],
                                              rho[i], NULL);
                    double* px = out + ((size_t)(y - row_begin) * Ws + x) * 3;
                    for (int k = 0; k < 3; ++k) px[k] += alpha[i] * color[3 * i + k] * f;
                }
            }
        }
    }
    return 0;
}

/* Forward at an explicit pixel list (brute, literal predicate): for sampled
 * parity at full sizes. out[p*3+k]. */
int gsr_oracle_render_pixels(int64_t n, const double* alpha, const double* mu,
                             const double* sigma, const double* rho, const double* color, int H,
                             int W, double sw, double sh, double r, int64_t npix, const int32_t* px_x,
                             const int32_t* px_y, double* out)
{
    double hx = r * (double)W, hy = r * (double)H;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t p = 0; p < npix; ++p) {
        double X = (double)px_x[p] / sw, Y = (double)px_y[p] / sh;
        double acc[3] = {0.0, 0.0, 0.0};
        for (int64_t i = 0; i < n; ++i) {
            if (!oracle_is_valid(alpha, mu, sigma, rho, color, i)) continue;
            double mx = mu[2 * i], my = mu[2 * i + 1];
            if (!(fabs(X - mx) < hx && fabs(Y - my) < hy)) continue;
            double f = oracle_density(X - mx, Y - my, sigma[2 * i], sigma[2 * i + 1], rho[i], NULL);
            for (int k = 0; k < 3; ++k) acc[k] += alpha[i] * color[3 * i + k] * f;
        }
        for (int k = 0; k < 3; ++k) out[3 * p + k] = acc[k];
    }
    return 0;
}

/* Continuous truncated field at arbitrary sample points with explicit window
 * half-extents (hx, hy) in the same units as mu (used for the coordinate-
 * normalisation pin: lengths scaled by (lx, ly) must give I / (lx*ly)).
 * pts[p*2+{0,1}] = (X, Y). Strict predicate |X-mx|<hx, |Y-my|<hy. */
int gsr_oracle_field(int64_t n, const double* alpha, const double* mu, const double* sigma,
                     const double* rho, const double* color, double hx, double hy, int64_t npts,
                     const double* pts, double* out)
{
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < npts; ++p) {
        double X = pts[2 * p], Y = pts[2 * p + 1];
        double acc[3] = {0.0, 0.0, 0.0};
        for (int64_t i = 0; i < n; ++i) {
            if (!oracle_is_valid(alpha, mu, sigma, rho, color, i)) continue;
            double mx = mu[2 * i], my = mu[2 * i + 1];
            if (!(fabs(X - mx) < hx && fabs(Y - my) < hy)) continue;
            double f = oracle_density(X - mx, Y - my, sigma[2 * i], sigma[2 * i + 1], rho[i], NULL);
            for (int k = 0; k < 3; ++k) acc[k] += alpha[i] * color[3 * i + k] * f;
        }
        for (int k = 0; k < 3; ++k) out[3 * p + k] = acc[k];
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Backward: direct per-pair derivatives of Eq. 1-2 (no moment formulas).     */
/* grad_out holds rows [row_begin,row_end) of dL/dI.  Gradients are written   */
/* (overwritten) for the Gaussians listed in idx (or all if idx == NULL).     */
/* absmass (optional, [n,9]) = sum over pairs of the monomial magnitudes of   */
/* each term (its fp32 rounding scale, R18), per output:            */
/*   alpha, mu_x, mu_y, sigma_x, sigma_y, rho, c_r, c_g, c_b                  */
/* termabs (optional, [n,9]) = sum over pairs of |term| (SURVEY 8(c).18's S). */
/* mode 0 brute (literal predicate over all pixels), mode 1 rect.             */
/* Per-pair derivatives (u = dx/sx, v = dy/sy, D = 1-rho^2, w = alpha f g.c): */
/*   d alpha = f g.c ;  d c_k = alpha f g_k                                   */
/*   d mu_x = w (u - rho v)/(sx D) ;  d mu_y = w (v - rho u)/(sy D)           */
/*   d sx = w (u (u - rho v)/D - 1)/sx ;  d sy = w (v (v - rho u)/D - 1)/sy   */
/*   d rho = w (rho + u v - rho Q)/D                                          */
/* (dx = X - mu_x, so d/d mu_x = -d/d dx; d ln K/d rho = rho/D.)              */
/* ------------------------------------------------------------------------- */
int gsr_oracle_render_bwd(int64_t n, const double* alpha, const double* mu, const double* sigma,
                          const double* rho, const double* color, int H, int W, double sw, double sh,
                          double r, int mode, int row_begin, int row_end, const double* grad_out,
                          int64_t nidx, const int64_t* idx, double* d_alpha, double* d_mu,
                          double* d_sigma, double* d_rho, double* d_color, double* absmass,
                          double* termabs)
{
    int Hs, Ws;
    gsr_oracle_out_dims(H, W, sw, sh, &Hs, &Ws);
    if (row_begin < 0) row_begin = 0;
    if (row_end > Hs) row_end = Hs;
    double hx = r * (double)W, hy = r * (double)H;
    int64_t cnt = idx ? nidx : n;

#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t t = 0; t < cnt; ++t) {
        int64_t i = idx ? idx[t] : t;
        double g9[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
        double a9[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
        double t9[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
        if (oracle_is_valid(alpha, mu, sigma, rho, color, i) && row_begin < row_end) {
            double mx = mu[2 * i], my = mu[2 * i + 1];
            double sx = sigma[2 * i], sy = sigma[2 * i + 1], rh = rho[i], al = alpha[i];
            const double* c = color + 3 * i;
            double D = 1.0 - rh * rh;
            int64_t xa = 0, xb = Ws - 1, ya = row_begin, yb = row_end - 1;
            int have = 1;
            if (mode == 1 || mode == 3) {
                int64_t x0u, y0u, x0, x1, y0, y1;
                have = oracle_rect_mode(mode == 3, mu, sigma, i, H, W, sw, sh, r, Hs, Ws, &x0u, &y0u,
                                        &x0, &x1, &y0, &y1);
                xa = x0; xb = x1;
                ya = y0 > row_begin ? y0 : row_begin;
                yb = y1 < row_end - 1 ? y1 : row_end - 1;
            }
            if (have) {
                for (int64_t y = ya; y <= yb; ++y) {
                    double Y = (double)y / sh;
                    for (int64_t x = xa; x <= xb; ++x) {
                        double X = (double)x / sw;
                        if (mode == 0 && !(fabs(X - mx) < hx && fabs(Y - my) < hy)) continue;
                        const double* g = grad_out + ((size_t)(y - row_begin) * Ws + x) * 3;
                        double dx = X - mx, dy = Y - my, Q;
                        double f = oracle_density(dx, dy, sx, sy, rh, &Q);
                        double u = dx / sx, v = dy / sy;
                        double gc = g[0] * c[0] + g[1] * c[1] + g[2] * c[2];
                        double w = al * f * gc;
                        double term[9], mono[9];
                        term[0] = f * gc;
                        term[1] = w * (u - rh * v) / (sx * D);
                        term[2] = w * (v - rh * u) / (sy * D);
                        term[3] = w * (u * (u - rh * v) / D - 1.0) / sx;
                        term[4] = w * (v * (v - rh * u) / D - 1.0) / sy;
                        term[5] = w * (rh + u * v - rh * Q) / D;
                        term[6] = al * f * g[0];
                        term[7] = al * f * g[1];
                        term[8] = al * f * g[2];
                        /* rounding scale of each term (R18): the sum of the absolute
                         * values of its monomials, with |g.c| -> sum_k |g_k c_k| */
                        double gca = fabs(g[0] * c[0]) + fabs(g[1] * c[1]) + fabs(g[2] * c[2]);
                        double wa = al * f * gca;
                        mono[0] = f * gca;
                        mono[1] = wa * (fabs(u) + fabs(rh * v)) / (sx * D);
                        mono[2] = wa * (fabs(v) + fabs(rh * u)) / (sy * D);
                        mono[3] = wa * ((u * u + fabs(rh * u * v)) / D + 1.0) / sx;
                        mono[4] = wa * ((v * v + fabs(rh * u * v)) / D + 1.0) / sy;
                        mono[5] = wa * (fabs(rh) + fabs(u * v) + fabs(rh) * Q) / D;
                        mono[6] = fabs(term[6]);
                        mono[7] = fabs(term[7]);
                        mono[8] = fabs(term[8]);
                        for (int k = 0; k < 9; ++k) {
                            g9[k] += term[k];
                            a9[k] += mono[k];
                            t9[k] += fabs(term[k]);
                        }
                    }
                }
            }
        }
        d_alpha[t] = g9[0];
        d_mu[2 * t] = g9[1];
        d_mu[2 * t + 1] = g9[2];
        d_sigma[2 * t] = g9[3];
        d_sigma[2 * t + 1] = g9[4];
        d_rho[t] = g9[5];
        d_color[3 * t] = g9[6];
        d_color[3 * t + 1] = g9[7];
        d_color[3 * t + 2] = g9[8];
        if (absmass)
            for (int k = 0; k < 9; ++k) absmass[9 * t + k] = a9[k];
        if (termabs)
            for (int k = 0; k < 9; ++k) termabs[9 * t + k] = t9[k];
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Brute-force tile binning (north_star: "tile binning bit-exact against a    */
/* CPU brute-force binning"). For tiles of tw x th HR px covering             */
/* [0,Ws) x [row_begin,row_end) in row-major tile order, list every valid     */
/* Gaussian whose clipped rect intersects the tile, ascending i, by          */
/* O(N * tiles) intersection tests. CSR output: counts[ntiles] then ids.     */
/* Call with ids == NULL to get counts only; returns total.                   */
/* ------------------------------------------------------------------------- */
int64_t gsr_oracle_tile_lists(int64_t n, const double* alpha, const double* mu,
                              const double* sigma, const double* rho, const double* color, int H,
                              int W, double sw, double sh, double r, int tw, int th, int row_begin,
                              int row_end, int support, int64_t* counts, int64_t* ids)
{
    int Hs, Ws;
    gsr_oracle_out_dims(H, W, sw, sh, &Hs, &Ws);
    if (row_end > Hs) row_end = Hs;
    int ntx = (Ws + tw - 1) / tw;
    int nty = (row_end - row_begin + th - 1) / th;
    int64_t total = 0;
    for (int ty = 0; ty < nty; ++ty)
        for (int tx = 0; tx < ntx; ++tx) {
            int64_t tx0 = (int64_t)tx * tw, tx1 = tx0 + tw - 1;
            int64_t ty0 = row_begin + (int64_t)ty * th, ty1 = ty0 + th - 1;
            if (tx1 > Ws - 1) tx1 = Ws - 1;
            if (ty1 > row_end - 1) ty1 = row_end - 1;
            int64_t c = 0;
            for (int64_t i = 0; i < n; ++i) {
                if (!oracle_is_valid(alpha, mu, sigma, rho, color, i)) continue;
                int64_t x0u, y0u, x0, x1, y0, y1;
                if (!oracle_rect_mode(support, mu, sigma, i, H, W, sw, sh, r, Hs, Ws, &x0u, &y0u, &x0,
                                      &x1, &y0, &y1))
                    continue;
                if (x1 < tx0 || x0 > tx1 || y1 < ty0 || y0 > ty1) continue;
                if (ids) ids[total] = i;
                ++total;
                ++c;
            }
            counts[(int64_t)ty * ntx + tx] = c;
        }
    return total;
}
