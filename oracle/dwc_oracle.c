/*
 * dwc_oracle.c -- the plain, slow, obviously-correct fp64 CPU ORACLE for
 * DAMAS on the wavelet-compressed computational grid (Ma & Liu, arXiv
 * 1608.05179; /root/reference/PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.
 * The product path (paper_1608_05179_b200/) never links, imports or calls it,
 * and this file shares no code, header, table or constant generator with it.
 *
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared -pthread (no FMA contraction,
 * no intrinsics, no -ffast-math): every expression below is evaluated exactly
 * as written, left to right, in IEEE binary64.
 *
 * Readings of the paper that this file implements are the ones listed in
 * DESIGN.md "Readings" (R1..R18, = SURVEY.md §8(c) A1..A18).  Each function
 * cites the passage it follows.  Pins (tests/test_oracle_*.py) tie every
 * function to values the paper or mathematics fixes.  Parity status: all
 * functions pinned; the end-to-end sigma/eta against the paper's Table 1 is
 * "parity unpinned" (unpublished 60-mic array).
 *
 * Return codes mirror include/dwc.h: 0 ok, -1 invalid, -2 singular,
 * -3 numeric (non-finite value / non-positive A_ii).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_EINVAL (-1)
#define OR_ESINGULAR (-2)
#define OR_ENUMERIC (-3)
#define OR_ENOMEM (-4)

/* ------------------------------------------------------------------------ */
/* Geometry (§2, :83-86; reading R17 dx = L/(N-1)).  */
/* Scan-grid node s = r*N + c sits at x = cx - L/2 + c*dx, y = cy - L/2 + r*dx,
 * z = z0.                                                                    */
void or_grid_point(int n, double L, double z0, double cx, double cy, int s,
                   double *xyz) {
    double dx = L / (double)(n - 1);
    int r = s / n, c = s % n;
    xyz[0] = cx - L / 2.0 + (double)c * dx;
    xyz[1] = cy - L / 2.0 + (double)r * dx;
    xyz[2] = z0;
}

/* Rayleigh beamwidth, Eq. 24: B = 1.22 z0 c0/(cos^3(phi) D f).
 * Grid-fineness rule dx/B <= 0.2 is a WARNING:
 * with D = 2 max_m |(x_m, y_m)|, phi = alpha/2 = atan(L / (2 z0)) (PAPER.md:85,
 * :288), dx = L/(N-1).  Returns 1 when dx/B > 0.2.                            */
double or_rayleigh_beamwidth(double z0, double c0, double phi, double D, double f) {
    double cp = cos(phi);
    return 1.22 * z0 * c0 / (cp * cp * cp * D * f);
}

int or_spacing_warning(int m, const double *mic, double c0, int n, double L, double z0,
                       double freq) {
    double rmax = 0.0;
    for (int i = 0; i < m; i++) {
        double r = sqrt(mic[3 * i] * mic[3 * i] + mic[3 * i + 1] * mic[3 * i + 1]);
        if (r > rmax) rmax = r;
    }
    double phi = atan(L / (2.0 * z0));
    double B = or_rayleigh_beamwidth(z0, c0, phi, 2.0 * rmax, freq);
    double dx = L / (double)(n - 1);
    return dx / B > 0.2;
}

/* ------------------------------------------------------------------------ */
/* S1 steering vector of one scan point (Eq. 3-4; Eq. 7,
 * PAPER.md:128-131; reading R1 = SURVEY A1): the per-column-normalised
 * propagation vector
 *     d_m = |r_s - r_m|,   g_m = exp(-j k d_m) / d_m,   k = 2 pi f / c0,
 *     e_m = sqrt(M) * g_m / ||g||_2 .
 * e is written as M interleaved (re, im) pairs.                              */
int or_steer_point(int m, const double *mic, double c0, int n, double L,
                   double z0, double cx, double cy, double freq, int s,
                   double *e) {
    double p[3];
    double k = 2.0 * M_PI * freq / c0;
    double norm2 = 0.0;
    or_grid_point(n, L, z0, cx, cy, s, p);
    for (int i = 0; i < m; i++) {
        double dx = p[0] - mic[3 * i + 0];
        double dy = p[1] - mic[3 * i + 1];
        double dz = p[2] - mic[3 * i + 2];
        double d = sqrt(dx * dx + dy * dy + dz * dz);
        if (!(d > 0.0)) return OR_ESINGULAR;       /* grid point on a mic */
        double gre = cos(k * d) / d;
        double gim = -sin(k * d) / d;
        e[2 * i + 0] = gre;
        e[2 * i + 1] = gim;
        norm2 += gre * gre + gim * gim;
    }
    double scale = sqrt((double)m) / sqrt(norm2);
    for (int i = 0; i < 2 * m; i++) e[i] = e[i] * scale;
    return OR_OK;
}

int or_steering(int m, const double *mic, double c0, int n, double L, double z0,
                double cx, double cy, double freq, int npts, const int *idx,
                double *E /* npts x m x 2 */) {
    for (int i = 0; i < npts; i++) {
        int rc = or_steer_point(m, mic, c0, n, L, z0, cx, cy, freq, idx[i], E + (size_t)2 * m * i);
        if (rc) return rc;
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* S2 DAS map, Eq. 2: b(r) = v^H C v / M^2 with v = e (R1).
 * Real part of the Hermitian form (reading R3); m outer, n inner, complex
 * fp64 accumulation.  csm is M x M complex128 row-major (C[m][n]).           */
/* dr != 0: diagonal removal ("Diagonal removal is usually applied to CSM";
 * reading R20): the m == j terms are left out, the quadratic form is
 * normalised by M^2 - M instead of M^2 and negative map values are clamped to 0.           */
int or_das(int m, const double *mic, double c0, int n, double L, double z0,
           double cx, double cy, double freq, const double *csm, double *b, int dr) {
    if (dr && m < 2) return OR_EINVAL;
    int S = n * n;
    double *e = (double *)malloc(sizeof(double) * 2 * (size_t)m);
    if (!e) return OR_ENOMEM;
    for (int s = 0; s < S; s++) {
        int rc = or_steer_point(m, mic, c0, n, L, z0, cx, cy, freq, s, e);
        if (rc) { free(e); return rc; }
        double acc_re = 0.0, acc_im = 0.0;
        for (int i = 0; i < m; i++) {
            double ar = e[2 * i], ai = -e[2 * i + 1];          /* conj(e_i) */
            for (int j = 0; j < m; j++) {
                if (dr && j == i) continue;                     /* C with its diagonal removed */
                double cr = csm[2 * ((size_t)i * m + j)];
                double ci = csm[2 * ((size_t)i * m + j) + 1];
                double er = e[2 * j], ei = e[2 * j + 1];
                double tr = cr * er - ci * ei;                  /* C_ij e_j */
                double ti = cr * ei + ci * er;
                acc_re += ar * tr - ai * ti;                    /* conj(e_i) * (...) */
                acc_im += ar * ti + ai * tr;
            }
        }
        (void)acc_im;                                           /* rounding residue (R3) */
        if (dr) {
            b[s] = acc_re / ((double)m * (double)m - (double)m);
            if (b[s] < 0.0) b[s] = 0.0;
        } else {
            b[s] = acc_re / ((double)m * (double)m);
        }
        if (!isfinite(b[s])) { free(e); return OR_ENUMERIC; }
    }
    free(e);
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* S3/S4 wavelet compression, Algorithm 1, Eq. 15
 * (PAPER.md:189-194), Eq. 20-22.  Readings R5-R10.
 *
 * J = floor(log2 N) (Alg. 1 line 1).  Level j grid G^j = nodes whose row and
 * column are multiples of 2^(J-j) (x_k^j = x_2k^(j+1), Eq. 15).
 * Loop j = J-1 .. 0 (Alg. 1 line 3): interpolate b on G^j to the points of
 * G^(j+1) \ G^j (line 5) with the linear interpolating stencil of R7, keep a
 * point if |interp - b| >= eps (line 7).  G^0 is always kept (line 12,
 * PAPER.md:227).  The union over levels (lines 13-16) is returned in
 * ascending node order (R9).                                                  */
int or_max_level(int n) {
    int J = 0;
    while (((long)2 << J) <= (long)n) J++;  /* largest J with 2^J <= N */
    return J;
}

/* 1-D interpolation taps for index i at fine stride h (R7).  Returns count. */
static int taps_1d(int i, int h, int n, int *pos, double *w) {
    int H = 2 * h;
    if (i % H == 0) {              /* on the coarse lattice */
        pos[0] = i; w[0] = 1.0; return 1;
    }
    if (i + h <= n - 1) {          /* interior: midpoint of two coarse neighbours */
        pos[0] = i - h; w[0] = 0.5; pos[1] = i + h; w[1] = 0.5; return 2;
    }
    if (i - 3 * h >= 0) {          /* right edge: linear extrapolation */
        pos[0] = i - h; w[0] = 1.5; pos[1] = i - 3 * h; w[1] = -0.5; return 2;
    }
    pos[0] = i - h; w[0] = 1.0;    /* only one coarse neighbour: constant */
    return 1;
}

/* 1-D taps of the 4-point (cubic) interpolating wavelet, SURVEY §8(f) NEXT-1 (PAPER.md:228
 * cites the Deslauriers-Dubuc interpolating family; reading R19 in DESIGN.md): Lagrange
 * interpolation at i through the 4 nearest coarse points i + k h, k odd.  Interior
 * {-3,-1,1,3}: (-1, 9, 9, -1)/16; left edge {-1,1,3,5}: (5, 15, -5, 1)/16; right edge
 * {-5,-3,-1,1}: (1, -5, 15, 5)/16; past the last coarse point {-7,-5,-3,-1}:
 * (-5, 21, -35, 35)/16; taps in ascending position.  Fewer than 4 coarse points in reach:
 * the linear rule (R7).                                                       */
static int taps_1d_cubic(int i, int h, int n, int *pos, double *w) {
    int H = 2 * h;
    if (i % H == 0) { pos[0] = i; w[0] = 1.0; return 1; }
    static const int off[4][4] = {{-3, -1, 1, 3}, {-1, 1, 3, 5}, {-5, -3, -1, 1}, {-7, -5, -3, -1}};
    static const double wt[4][4] = {{-1.0, 9.0, 9.0, -1.0}, {5.0, 15.0, -5.0, 1.0},
                                    {1.0, -5.0, 15.0, 5.0}, {-5.0, 21.0, -35.0, 35.0}};
    int set = -1;
    if (i - 3 * h >= 0 && i + 3 * h <= n - 1) set = 0;
    else if (i - 3 * h < 0 && i + 5 * h <= n - 1) set = 1;
    else if (i + h <= n - 1 && i + 3 * h > n - 1 && i - 5 * h >= 0) set = 2;
    else if (i + h > n - 1 && i - 7 * h >= 0) set = 3;
    if (set < 0) return taps_1d(i, h, n, pos, w);
    for (int k = 0; k < 4; k++) {
        pos[k] = i + off[set][k] * h;
        w[k] = wt[set][k] / 16.0;   /* exact */
    }
    return 4;
}

/* Interpolated value at (r,c) from level-j values of b (fine stride h).
 * Tensor product "interpolate rows then column" (R7):
 * t_a = sum_b w_b * b[r_a][c_b] (along x), pred = sum_a w_a * t_a, sums left to right. */
static double interp_2d(const double *b, int n, int r, int c, int h, int order) {
    int rp[4], cp[4];
    double rw[4], cw[4];
    int nr = order == 3 ? taps_1d_cubic(r, h, n, rp, rw) : taps_1d(r, h, n, rp, rw);
    int nc = order == 3 ? taps_1d_cubic(c, h, n, cp, cw) : taps_1d(c, h, n, cp, cw);
    double pred = 0.0;
    for (int a = 0; a < nr; a++) {
        double t = 0.0;
        for (int q = 0; q < nc; q++) {
            double v = cw[q] * b[(size_t)rp[a] * n + cp[q]];
            t = (q == 0) ? v : t + v;
        }
        double v = rw[a] * t;
        pred = (a == 0) ? v : pred + v;
    }
    return pred;
}

/* Detail coefficients d = b - interp (Eq. 22) for every point of every level
 * > 0, and the level of every node.  d[s] = 0 on G^0.  order: 1 linear (R7), 3 cubic (R19). */
int or_wavelet_details(int n, const double *b, double *d, uint8_t *level, int order) {
    if (n < 2 || (order != 1 && order != 3)) return OR_EINVAL;
    int J = or_max_level(n);
    int S = n * n;
    for (int s = 0; s < S; s++) { d[s] = 0.0; if (level) level[s] = 0; }
    for (int j = J - 1; j >= 0; j--) {                 /* Alg. 1 line 3 */
        int H = 1 << (J - j);                          /* stride of G^j     */
        int h = H >> 1;                                /* stride of G^(j+1) */
        for (int r = 0; r < n; r += h)
            for (int c = 0; c < n; c += h) {
                if (r % H == 0 && c % H == 0) continue;   /* in G^j already */
                double pred = interp_2d(b, n, r, c, h, order);   /* Alg. 1 line 5 */
                d[(size_t)r * n + c] = b[(size_t)r * n + c] - pred;
                if (level) level[(size_t)r * n + c] = (uint8_t)(j + 1);
            }
    }
    return OR_OK;
}

/* eps_mode 0: eps_eff = eps * max|b| (R6, relative);
 * eps_mode 1: eps_eff = eps (absolute).  full_grid != 0: keep everything.
 * Returns n_keep (> 0) or a negative error.                                   */
int or_compress(int n, const double *b, double eps, int eps_mode, int full_grid,
                int *keep, uint8_t *level, double *d_out, double *eps_eff_out, int order) {
    if (n < 2 || !(eps > 0.0)) return OR_EINVAL;
    int S = n * n;
    double *d = d_out ? d_out : (double *)malloc(sizeof(double) * (size_t)S);
    uint8_t *lv = level ? level : (uint8_t *)malloc((size_t)S);
    if (!d || !lv) return OR_ENOMEM;
    int rc = or_wavelet_details(n, b, d, lv, order);
    double maxabs = 0.0;
    for (int s = 0; s < S; s++) {
        double a = fabs(b[s]);
        if (!isfinite(a)) rc = OR_ENUMERIC;
        if (a > maxabs) maxabs = a;
    }
    double eps_eff = (eps_mode == 0) ? eps * maxabs : eps;
    int degenerate = (eps_mode == 0 && maxabs == 0.0);   /* R6: keep G^0 only */
    if (eps_eff_out) *eps_eff_out = eps_eff;
    int nk = 0;
    for (int s = 0; s < S && rc == OR_OK; s++) {
        int kp;
        if (full_grid) kp = 1;
        else if (lv[s] == 0) kp = 1;                      /* G^0 always kept */
        else if (degenerate) kp = 0;
        else kp = fabs(d[s]) >= eps_eff;                  /* Alg. 1 line 7, ties kept (R5) */
        if (kp) keep[nk++] = s;
    }
    if (!d_out) free(d);
    if (!level) free(lv);
    return rc == OR_OK ? nk : rc;
}

/* ------------------------------------------------------------------------ */
/* S5 PSF on the kept points, Eq. 9-12 with v = g = e (R1):
 *   A_ij = |e_i^H e_j|^2 / M^2     (Eq. 23 restriction).  */
/* dr != 0 (reading R20): the PSF consistent with the diagonal-removed DAS, i.e. b = A x for
 * C = sum_s x_s e_s e_s^H with its diagonal removed:
 *   A_ij = (|e_i^H e_j|^2 - sum_q |e_qi|^2 |e_qj|^2) / (M^2 - M),  negative entries clamped to 0. */
int or_psf(int m, const double *mic, double c0, int n, double L, double z0,
           double cx, double cy, double freq, int nk, const int *keep,
           double *A /* nk x nk row-major */, int dr) {
    if (dr && m < 2) return OR_EINVAL;
    double *E = (double *)malloc(sizeof(double) * 2 * (size_t)m * (size_t)nk);
    if (!E) return OR_ENOMEM;
    int rc = or_steering(m, mic, c0, n, L, z0, cx, cy, freq, nk, keep, E);
    if (rc) { free(E); return rc; }
    double m2 = (double)m * (double)m;
    for (int i = 0; i < nk; i++)
        for (int j = 0; j < nk; j++) {
            double gr = 0.0, gi = 0.0;
            const double *ei = E + (size_t)2 * m * i, *ej = E + (size_t)2 * m * j;
            for (int q = 0; q < m; q++) {
                double ar = ei[2 * q], ai = -ei[2 * q + 1];   /* conj(e_qi) */
                double br = ej[2 * q], bi = ej[2 * q + 1];
                gr += ar * br - ai * bi;
                gi += ar * bi + ai * br;
            }
            if (dr) {
                double q4 = 0.0;
                for (int q = 0; q < m; q++) {
                    double pi2 = ei[2 * q] * ei[2 * q] + ei[2 * q + 1] * ei[2 * q + 1];
                    double pj2 = ej[2 * q] * ej[2 * q] + ej[2 * q + 1] * ej[2 * q + 1];
                    q4 += pi2 * pj2;
                }
                double v = (gr * gr + gi * gi - q4) / (m2 - (double)m);
                A[(size_t)i * nk + j] = v > 0.0 ? v : 0.0;
            } else {
                A[(size_t)i * nk + j] = (gr * gr + gi * gi) / m2;
            }
        }
    free(E);
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* The paper-literal beamformer and PSF (SURVEY §8(c) "paper-literal variant", NEXT-4; for the
 * fidelity discussion of reading R1 only): Eq. 4 v_m(r) = (d_m/|r|) e^{-jk d_m}
 * for the focus, Eq. 7 g_m(r_s) = (|r_s|/d_m) e^{-jk d_m} (exponent per R2) for
 * the source, |r| = distance to the array centre (the coordinate origin of the array plane):
 *   b_P(r) = Re(v(r)^H C v(r)) / M^2 (Eq. 2),   A_P[r][s] = |v(r)^H g(r_s)|^2 / M^2 (Eq. 10).
 * A_P[r][r] = 1 exactly in exact arithmetic (conj(v_m) g_m = 1), A_P is not symmetric.       */
static int paper_vectors(int m, const double *mic, double c0, int n, double L, double z0, double cx,
                         double cy, double freq, int s, double *v, double *g) {
    double p[3];
    double k = 2.0 * M_PI * freq / c0;
    or_grid_point(n, L, z0, cx, cy, s, p);
    double rn = sqrt(p[0] * p[0] + p[1] * p[1] + p[2] * p[2]);
    for (int i = 0; i < m; i++) {
        double dx = p[0] - mic[3 * i + 0], dy = p[1] - mic[3 * i + 1], dz = p[2] - mic[3 * i + 2];
        double d = sqrt(dx * dx + dy * dy + dz * dz);
        if (!(d > 0.0)) return OR_ESINGULAR;
        double c = cos(k * d), sn = sin(k * d);
        v[2 * i] = (d / rn) * c;  v[2 * i + 1] = -(d / rn) * sn;
        g[2 * i] = (rn / d) * c;  g[2 * i + 1] = -(rn / d) * sn;
    }
    return OR_OK;
}

int or_das_paper(int m, const double *mic, double c0, int n, double L, double z0,
                 double cx, double cy, double freq, const double *csm, double *b) {
    int S = n * n;
    double *v = (double *)malloc(sizeof(double) * 4 * (size_t)m);
    if (!v) return OR_ENOMEM;
    for (int s = 0; s < S; s++) {
        int rc = paper_vectors(m, mic, c0, n, L, z0, cx, cy, freq, s, v, v + 2 * m);
        if (rc) { free(v); return rc; }
        double acc = 0.0;
        for (int i = 0; i < m; i++) {
            double ar = v[2 * i], ai = -v[2 * i + 1];
            for (int j = 0; j < m; j++) {
                double cr = csm[2 * ((size_t)i * m + j)], ci = csm[2 * ((size_t)i * m + j) + 1];
                double tr = cr * v[2 * j] - ci * v[2 * j + 1], ti = cr * v[2 * j + 1] + ci * v[2 * j];
                acc += ar * tr - ai * ti;
            }
        }
        b[s] = acc / ((double)m * (double)m);
    }
    free(v);
    return OR_OK;
}

int or_psf_paper(int m, const double *mic, double c0, int n, double L, double z0,
                 double cx, double cy, double freq, int nk, const int *keep, double *A) {
    double *V = (double *)malloc(sizeof(double) * 4 * (size_t)m * (size_t)nk);
    if (!V) return OR_ENOMEM;
    double *G = V + (size_t)2 * m * nk;
    for (int i = 0; i < nk; i++) {
        int rc = paper_vectors(m, mic, c0, n, L, z0, cx, cy, freq, keep[i], V + (size_t)2 * m * i,
                               G + (size_t)2 * m * i);
        if (rc) { free(V); return rc; }
    }
    double m2 = (double)m * (double)m;
    for (int i = 0; i < nk; i++)
        for (int j = 0; j < nk; j++) {
            const double *vi = V + (size_t)2 * m * i, *gj = G + (size_t)2 * m * j;
            double gr = 0.0, gi = 0.0;
            for (int q = 0; q < m; q++) {
                double ar = vi[2 * q], ai = -vi[2 * q + 1];
                gr += ar * gj[2 * q] - ai * gj[2 * q + 1];
                gi += ar * gj[2 * q + 1] + ai * gj[2 * q];
            }
            A[(size_t)i * nk + j] = (gr * gr + gi * gi) / m2;
        }
    free(V);
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Eq. 1, the step before the path:
 *   C = (1/I) sum_i p_i p_i^H,   p_i = snap[:, i],
 * snap complex128 [m][I] interleaved (row = microphone), C complex128 [m][m];
 * sums over i ascending in fp64, then divided by I.                            */
int or_csm(int m, int I, const double *snap, double *C) {
    if (m < 1 || I < 1) return OR_EINVAL;
    for (int a = 0; a < m; a++)
        for (int b = 0; b < m; b++) {
            double re = 0.0, im = 0.0;
            for (int i = 0; i < I; i++) {
                double pr = snap[2 * ((size_t)a * I + i)], pi = snap[2 * ((size_t)a * I + i) + 1];
                double qr = snap[2 * ((size_t)b * I + i)], qi = snap[2 * ((size_t)b * I + i) + 1];
                re += pr * qr + pi * qi;            /* p_a conj(p_b) */
                im += pi * qr - pr * qi;
            }
            C[2 * ((size_t)a * m + b)] = re / (double)I;
            C[2 * ((size_t)a * m + b) + 1] = im / (double)I;
        }
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* S7 DAMAS Gauss-Seidel with positivity, Eq. 13-14:
 *   r_i = sum_{j<i} A_ij x_j^(n+1) + sum_{j>=i} A_ij x_j^(n) - b_i
 *   x_i^(n+1) = max(x_i^(n) - r_i / A_ii, 0),   x^0 = 0.
 * In-place forward sweep, i ascending; "l" of Eq. 13 = n (R4); fixed sweep
 * count (R18).  The sum runs left to right in fp64.                          */
/* alt != 0 (reading R21): the original DAMAS practice of alternating
 * sweep directions: odd-numbered sweeps run i descending, same update.         */
int or_gs(int nk, const double *A, const double *b, int sweeps, double *x, int alt) {
    if (nk < 1 || sweeps < 1) return OR_EINVAL;
    for (int i = 0; i < nk; i++) {
        double aii = A[(size_t)i * nk + i];
        if (!(aii > 0.0) || !isfinite(aii)) return OR_ENUMERIC;
        x[i] = 0.0;
    }
    for (int it = 0; it < sweeps; it++) {
        const int back = alt && (it & 1);
        for (int ii = 0; ii < nk; ii++) {
            const int i = back ? nk - 1 - ii : ii;
            const double *row = A + (size_t)i * nk;
            double r = 0.0;
            for (int j = 0; j < nk; j++) r += row[j] * x[j];
            r = r - b[i];
            double v = x[i] - r / row[i];
            x[i] = v > 0.0 ? v : 0.0;
            if (!isfinite(x[i])) return OR_ENUMERIC;
        }
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* One bin, S1..S8.  keep (S ints) ascending, first n_keep valid.  x_map (S)
 * is the source power on the full grid, zero off the kept set (S8).
 * flags: bit 0 full grid (keep every node), bit 1 cubic predictor (R19),
 * bit 2 diagonal removal (R20), bit 3 alternating sweep directions (R21),
 * bit 4 paper-literal beamformer and PSF (Eq. 4 v for the focus, Eq. 7 g for the source,
 * PAPER.md:108, :130; asymmetric A, fidelity variant of R1; not with bit 2).        */
int or_solve_bin(int m, const double *mic, double c0, int n, double L, double z0,
                 double cx, double cy, double freq, const double *csm,
                 double eps, int eps_mode, int sweeps, int flags,
                 int *n_keep, int *keep, double *x_map, double *b_map) {
    int S = n * n;
    double *b = b_map ? b_map : (double *)malloc(sizeof(double) * (size_t)S);
    if (!b) return OR_ENOMEM;
    if ((flags & 16) && (flags & 4)) {
        if (!b_map) free(b);
        return OR_EINVAL;
    }
    int rc = (flags & 16) ? or_das_paper(m, mic, c0, n, L, z0, cx, cy, freq, csm, b)
                          : or_das(m, mic, c0, n, L, z0, cx, cy, freq, csm, b, flags & 4);
    int nk = 0;
    double *A = NULL, *bt = NULL, *xt = NULL;
    if (rc == OR_OK) {
        nk = or_compress(n, b, eps, eps_mode, flags & 1, keep, NULL, NULL, NULL, (flags & 2) ? 3 : 1);
        if (nk < 0) rc = nk;
    }
    if (rc == OR_OK) {
        A = (double *)malloc(sizeof(double) * (size_t)nk * (size_t)nk);
        bt = (double *)malloc(sizeof(double) * (size_t)nk);
        xt = (double *)malloc(sizeof(double) * (size_t)nk);
        if (!A || !bt || !xt) rc = OR_ENOMEM;
    }
    if (rc == OR_OK)
        rc = (flags & 16) ? or_psf_paper(m, mic, c0, n, L, z0, cx, cy, freq, nk, keep, A)
                          : or_psf(m, mic, c0, n, L, z0, cx, cy, freq, nk, keep, A, flags & 4);
    if (rc == OR_OK) {
        for (int i = 0; i < nk; i++) bt[i] = b[keep[i]];   /* S6: b~ = b[keep] */
        rc = or_gs(nk, A, bt, sweeps, xt, flags & 8);
    }
    if (rc == OR_OK) {
        for (int s = 0; s < S; s++) x_map[s] = 0.0;         /* S8 embed */
        for (int i = 0; i < nk; i++) x_map[keep[i]] = xt[i];
        for (int i = nk; i < S; i++) keep[i] = -1;
        *n_keep = nk;
    }
    free(A); free(bt); free(xt);
    if (!b_map) free(b);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* S0 batch over frequency bins: bins are independent;
 * a plain pthread pool runs one bin per thread at a time.                    */
typedef struct {
    int m; const double *mic; double c0; int n; double L, z0, cx, cy;
    int K; const double *freq; const double *csm;
    double eps; int eps_mode, sweeps, flags;
    int *n_keep, *keep; double *x_map, *b_map;
    int next; int rc; pthread_mutex_t mu;
} band_job;

static void *band_worker(void *arg) {
    band_job *jb = (band_job *)arg;
    int S = jb->n * jb->n;
    for (;;) {
        pthread_mutex_lock(&jb->mu);
        int k = jb->next++;
        pthread_mutex_unlock(&jb->mu);
        if (k >= jb->K) break;
        int rc = or_solve_bin(jb->m, jb->mic, jb->c0, jb->n, jb->L, jb->z0, jb->cx, jb->cy,
                              jb->freq[k], jb->csm + (size_t)2 * jb->m * jb->m * k,
                              jb->eps, jb->eps_mode, jb->sweeps, jb->flags,
                              jb->n_keep + k, jb->keep + (size_t)S * k,
                              jb->x_map + (size_t)S * k,
                              jb->b_map ? jb->b_map + (size_t)S * k : NULL);
        if (rc) {
            pthread_mutex_lock(&jb->mu);
            if (jb->rc == OR_OK) jb->rc = rc;
            pthread_mutex_unlock(&jb->mu);
        }
    }
    return NULL;
}

int or_solve_band(int m, const double *mic, double c0, int n, double L, double z0,
                  double cx, double cy, int K, const double *freq, const double *csm,
                  double eps, int eps_mode, int sweeps, int flags,
                  int *n_keep, int *keep, double *x_map, double *b_map, int n_threads) {
    if (K < 1) return OR_OK;
    if (n_threads < 1) n_threads = 1;
    if (n_threads > K) n_threads = K;
    band_job jb = {m, mic, c0, n, L, z0, cx, cy, K, freq, csm, eps, eps_mode, sweeps,
                   flags, n_keep, keep, x_map, b_map, 0, OR_OK, PTHREAD_MUTEX_INITIALIZER};
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)n_threads);
    if (!th) return OR_ENOMEM;
    for (int t = 0; t < n_threads; t++) pthread_create(&th[t], NULL, band_worker, &jb);
    for (int t = 0; t < n_threads; t++) pthread_join(th[t], NULL);
    free(th);
    return jb.rc;
}
