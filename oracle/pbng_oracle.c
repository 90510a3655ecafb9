/*
 * oracle/pbng_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, serial, fp64 CPU reference ("oracle") for the hot path of
 *   Chen, Han, Chen, Teran, "Position-Based Nonlinear Gauss-Seidel for Quasistatic Hyperelasticity",
 *   arXiv 2306.09021 (the paper text is PAPER.md; line numbers below are PAPER.md lines).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load
 * this file.  It shares no code, header, table or constant generator with the CUDA path
 * (paper_2306_09021_b200/csrc) and neither side includes or links the other.
 *
 * Every function follows the paper's definitions in the paper's order and notation; nothing is fused,
 * blocked or reordered.  Readings of silent / garbled passages:
 *   Z1  Neo-Hookean energy shifted by a constant so that Psi(I) = 0 (forces unchanged).
 *   Z2  the modified Hessian density uses the Lame lambda (not lambda-hat) for every model.
 *   Z3  "J F^{-1}" in eq:mod_hess_dens is the cofactor matrix cof(F) = det(F) F^{-T}.
 *   Z4  R(F) is the closest ROTATION (sign-corrected SVD, det R = +1), also for inverted F.
 *   Z5  Chebyshev omega_1 = omega_2 = 1, omega_3 = 2/(2-rho^2), omega_{l+1} = 4/(4-rho^2 omega_l).
 *   Z7  SOR blends against x^{l-1} exactly as printed.
 *   Z8  x^{-1} := x^0.    Z9  Dirichlet rows keep their targets under blending.
 *   Z13 the external-work term sums over all vertices.  Z14 residual = 2-norm over free vertices.
 *   Weak constraint with an empty side 1 uses a fixed anchor point instead (rigid-plane contact).
 *   Backward Euler (eq:fem_be) keeps f^ext in the residual and uses xtilde = 2 x^n - x^{n-1}; the
 *   energy then is the incremental potential with the inertia of the free nodes.
 *
 * Matrices are row-major double[9]: M[3*a+b] = M_{ab}.  Fourth-order tensors are double[81] with
 * T[(3*alpha+gamma)*9 + 3*beta+delta] = T_{alpha gamma beta delta}.
 * Pinned by tests/test_oracle_*.py (materials, colouring, solver); no function is "parity unpinned".
 */
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { ORC_OK = 0, ORC_E_ARG = 1, ORC_E_DEGENERATE = 2, ORC_E_ISOLATED = 3, ORC_E_NOMEM = 4 };
enum { ORC_NH = 0, ORC_FCR = 1, ORC_SNH = 2 };
enum { ORC_ACCEL_NONE = 0, ORC_ACCEL_SOR = 1, ORC_ACCEL_CHEBYSHEV = 2 };

/* ------------------------------------------------------------------------------------------------ */
/* 3x3 helpers                                                                                      */
/* ------------------------------------------------------------------------------------------------ */

static double det3(const double *M) {
    return M[0] * (M[4] * M[8] - M[5] * M[7]) - M[1] * (M[3] * M[8] - M[5] * M[6]) +
           M[2] * (M[3] * M[7] - M[4] * M[6]);
}

/* cof(F)_{ab} = d det(F) / d F_{ab}  ("J F^{-T} ... the cofactor matrix", defined for all F) */
void orc_cofactor(const double *F, double *C) {
    C[0] = F[4] * F[8] - F[5] * F[7];
    C[1] = F[5] * F[6] - F[3] * F[8];
    C[2] = F[3] * F[7] - F[4] * F[6];
    C[3] = F[2] * F[7] - F[1] * F[8];
    C[4] = F[0] * F[8] - F[2] * F[6];
    C[5] = F[1] * F[6] - F[0] * F[7];
    C[6] = F[1] * F[5] - F[2] * F[4];
    C[7] = F[2] * F[3] - F[0] * F[5];
    C[8] = F[0] * F[4] - F[1] * F[3];
}

double orc_det(const double *F) { return det3(F); }

/* eq:lame: mu = E / (2 (1 + nu)),  lambda = E nu / ((1 + nu)(1 - 2 nu)) */
int orc_lame(double E, double nu, double *mu, double *lambda) {
    if (!(E > 0.0) || !(nu >= 0.0) || !(nu < 0.5)) return ORC_E_ARG;
    *mu = E / (2.0 * (1.0 + nu));
    *lambda = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    return ORC_OK;
}

/* ------------------------------------------------------------------------------------------------ */
/* Polar rotation R(F) of F = R S, reading Z4: closest rotation.                 */
/* Cyclic Jacobi eigen-decomposition of S = F^T F (textbook), then U from F V by Gram-Schmidt,        */
/* u3 = u1 x u2 (so det U = det V = +1 and the smallest singular value carries the sign of det F).   */
/* ------------------------------------------------------------------------------------------------ */

static void jacobi_eig_sym3(double *S, double *V) {
    int p, q, k, sweep;
    static const int P[3] = {0, 0, 1}, Q[3] = {1, 2, 2};
    for (k = 0; k < 9; ++k) V[k] = (k % 4 == 0) ? 1.0 : 0.0;
    for (sweep = 0; sweep < 64; ++sweep) {
        double off = S[1] * S[1] + S[2] * S[2] + S[5] * S[5];
        double diag = S[0] * S[0] + S[4] * S[4] + S[8] * S[8];
        if (off == 0.0 || off <= 1e-40 * diag) break;
        for (k = 0; k < 3; ++k) {
            double apq, app, aqq, theta, t, c, s;
            int r;
            p = P[k];
            q = Q[k];
            apq = S[3 * p + q];
            if (apq == 0.0) continue;
            app = S[3 * p + p];
            aqq = S[3 * q + q];
            theta = (aqq - app) / (2.0 * apq);
            t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
            c = 1.0 / sqrt(t * t + 1.0);
            s = t * c;
            /* S <- J^T S J with J the (p,q) Givens rotation [c s; -s c] */
            for (r = 0; r < 3; ++r) { /* columns p,q */
                double srp = S[3 * r + p], srq = S[3 * r + q];
                S[3 * r + p] = c * srp - s * srq;
                S[3 * r + q] = s * srp + c * srq;
            }
            for (r = 0; r < 3; ++r) { /* rows p,q */
                double spr = S[3 * p + r], sqr = S[3 * q + r];
                S[3 * p + r] = c * spr - s * sqr;
                S[3 * q + r] = s * spr + c * sqr;
            }
            for (r = 0; r < 3; ++r) {
                double vrp = V[3 * r + p], vrq = V[3 * r + q];
                V[3 * r + p] = c * vrp - s * vrq;
                V[3 * r + q] = s * vrp + c * vrq;
            }
        }
    }
}

static void cross3(const double *a, const double *b, double *c) {
    c[0] = a[1] * b[2] - a[2] * b[1];
    c[1] = a[2] * b[0] - a[0] * b[2];
    c[2] = a[0] * b[1] - a[1] * b[0];
}

static double norm3(const double *a) { return sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]); }

/* a unit vector perpendicular to unit u, chosen deterministically */
static void perp_unit(const double *u, double *out) {
    double e[3] = {0, 0, 0}, c[3], n;
    int k = 0;
    if (fabs(u[1]) < fabs(u[k])) k = 1;
    if (fabs(u[2]) < fabs(u[k])) k = 2;
    e[k] = 1.0;
    cross3(u, e, c);
    n = norm3(c);
    out[0] = c[0] / n;
    out[1] = c[1] / n;
    out[2] = c[2] / n;
}

void orc_polar(const double *F, double *R) {
    double S[9], V[9], ev[3], u[3][3], fv[3][3], n1, n2, d;
    int a, b, k, order[3] = {0, 1, 2};
    for (a = 0; a < 3; ++a)
        for (b = 0; b < 3; ++b) {
            S[3 * a + b] = 0.0;
            for (k = 0; k < 3; ++k) S[3 * a + b] += F[3 * k + a] * F[3 * k + b];
        }
    jacobi_eig_sym3(S, V);
    for (k = 0; k < 3; ++k) ev[k] = S[4 * k];
    /* sort eigenpairs by decreasing eigenvalue (insertion sort of the index list) */
    for (a = 1; a < 3; ++a)
        for (b = a; b > 0 && ev[order[b]] > ev[order[b - 1]]; --b) {
            int t = order[b];
            order[b] = order[b - 1];
            order[b - 1] = t;
        }
    {
        double Vs[9];
        for (a = 0; a < 3; ++a)
            for (k = 0; k < 3; ++k) Vs[3 * a + k] = V[3 * a + order[k]];
        memcpy(V, Vs, sizeof(Vs));
    }
    if (det3(V) < 0.0)
        for (a = 0; a < 3; ++a) V[3 * a + 2] = -V[3 * a + 2];
    /* F v_k */
    for (k = 0; k < 3; ++k)
        for (a = 0; a < 3; ++a) {
            fv[k][a] = 0.0;
            for (b = 0; b < 3; ++b) fv[k][a] += F[3 * a + b] * V[3 * b + k];
        }
    n1 = norm3(fv[0]);
    if (n1 == 0.0) { /* F == 0: every rotation is closest; take R = I */
        for (k = 0; k < 9; ++k) R[k] = (k % 4 == 0) ? 1.0 : 0.0;
        return;
    }
    for (a = 0; a < 3; ++a) u[0][a] = fv[0][a] / n1;
    d = u[0][0] * fv[1][0] + u[0][1] * fv[1][1] + u[0][2] * fv[1][2];
    for (a = 0; a < 3; ++a) u[1][a] = fv[1][a] - d * u[0][a];
    n2 = norm3(u[1]);
    if (n2 <= 1e-13 * n1) {
        perp_unit(u[0], u[1]);
    } else {
        for (a = 0; a < 3; ++a) u[1][a] /= n2;
    }
    cross3(u[0], u[1], u[2]);
    /* R = U V^T */
    for (a = 0; a < 3; ++a)
        for (b = 0; b < 3; ++b) {
            R[3 * a + b] = 0.0;
            for (k = 0; k < 3; ++k) R[3 * a + b] += u[k][a] * V[3 * b + k];
        }
}

/* ------------------------------------------------------------------------------------------------ */
/* Constitutive models                                                           */
/* ------------------------------------------------------------------------------------------------ */

/* Stable Neo-Hookean (eq:snh), reading Z18: the printed volume coefficient 1/2 is taken
 * as lambda_s/2 and the Lame parameters are re-parameterised as in the cited model, mu_s = 4 mu / 3,
 * lambda_s = lambda + 5 mu / 6, alpha = 1 + 3 mu_s / (4 lambda_s), which makes the Hessian at F = I equal
 * linear elasticity's (the requirement of PAPER.md:645; pinned by the tests):
 *   Psi = mu_s/2 (|F|^2 - 3) + lambda_s/2 (J - alpha)^2 - mu_s/2 log(1 + |F|^2)  [- Psi(I) unless raw] */
static void snh_params(double mu, double lambda, double *ms, double *ls, double *alpha) {
    *ms = 4.0 * mu / 3.0;
    *ls = lambda + 5.0 * mu / 6.0;
    *alpha = 1.0 + 3.0 * (*ms) / (4.0 * (*ls));
}

/* Psi(F).  FCR eq:cor: mu |F - R(F)|_F^2 + lambda/2 (det F - 1)^2.
 * NH eq:nh: 1/2 mu |F|_F^2 + lambdahat/2 (det F - 1 - mu/lambdahat)^2, lambdahat = mu +
 * lambda; with raw == 0 the constant 3/2 mu + mu^2/(2 lambdahat) is subtracted (reading Z1). */
double orc_psi(int model, double mu, double lambda, const double *F, int raw) {
    double J = det3(F);
    int k;
    if (model == ORC_FCR) {
        double R[9], s = 0.0;
        orc_polar(F, R);
        for (k = 0; k < 9; ++k) s += (F[k] - R[k]) * (F[k] - R[k]);
        return mu * s + 0.5 * lambda * (J - 1.0) * (J - 1.0);
    } else if (model == ORC_SNH) {
        double ms, ls, al, ic = 0.0, psi;
        snh_params(mu, lambda, &ms, &ls, &al);
        for (k = 0; k < 9; ++k) ic += F[k] * F[k];
        psi = 0.5 * ms * (ic - 3.0) + 0.5 * ls * (J - al) * (J - al) - 0.5 * ms * log(1.0 + ic);
        if (!raw) psi -= 0.5 * ls * (1.0 - al) * (1.0 - al) - 0.5 * ms * log(4.0);
        return psi;
    } else {
        double lh = mu + lambda, fro = 0.0, t, psi;
        for (k = 0; k < 9; ++k) fro += F[k] * F[k];
        t = J - 1.0 - mu / lh;
        psi = 0.5 * mu * fro + 0.5 * lh * t * t;
        if (!raw) psi -= 1.5 * mu + mu * mu / (2.0 * lh);
        return psi;
    }
}

/* P = dPsi/dF.  NH: mu F + lambdahat (J - 1 - mu/lambdahat) cof F.
 * FCR: 2 mu (F - R) + lambda (J - 1) cof F. */
void orc_piola(int model, double mu, double lambda, const double *F, double *P) {
    double C[9], J = det3(F);
    int k;
    orc_cofactor(F, C);
    if (model == ORC_FCR) {
        double R[9];
        orc_polar(F, R);
        for (k = 0; k < 9; ++k) P[k] = 2.0 * mu * (F[k] - R[k]) + lambda * (J - 1.0) * C[k];
    } else if (model == ORC_SNH) {
        /* P = mu_s F + lambda_s (J - alpha) cof F - mu_s F / (1 + |F|^2) */
        double ms, ls, al, ic = 0.0;
        snh_params(mu, lambda, &ms, &ls, &al);
        for (k = 0; k < 9; ++k) ic += F[k] * F[k];
        for (k = 0; k < 9; ++k) P[k] = ms * F[k] + ls * (J - al) * C[k] - ms * F[k] / (1.0 + ic);
    } else {
        double lh = mu + lambda;
        for (k = 0; k < 9; ++k) P[k] = mu * F[k] + lh * (J - 1.0 - mu / lh) * C[k];
    }
}

/* eq:mod_hess_dens: Ctilde_{alpha gamma beta delta} = 2 mu delta_{alpha beta}
 * delta_{gamma delta} + lambda cof(F)_{alpha gamma} cof(F)_{beta delta}   (readings Z2, Z3) */
void orc_mod_hess_density(double mu, double lambda, const double *F, double *T) {
    double C[9];
    int al, ga, be, de;
    orc_cofactor(F, C);
    for (al = 0; al < 3; ++al)
        for (ga = 0; ga < 3; ++ga)
            for (be = 0; be < 3; ++be)
                for (de = 0; de < 3; ++de)
                    T[(3 * al + ga) * 9 + 3 * be + de] =
                        2.0 * mu * (al == be ? 1.0 : 0.0) * (ga == de ? 1.0 : 0.0) +
                        lambda * C[3 * al + ga] * C[3 * be + de];
}

/* ------------------------------------------------------------------------------------------------ */
/* Scene and its plain precompute                                                */
/* ------------------------------------------------------------------------------------------------ */

typedef struct {
    int64_t nv;
    const double *X;
    int64_t nt;
    const int32_t *tets;
    int32_t model;
    const double *E;
    int64_t nE;
    double nu, density;
    double gravity[3];
    int64_t npin;
    const int32_t *pinned;
    int64_t nwc;
    const int32_t *wc_n0, *wc_n1, *wc_idx0, *wc_idx1;
    const double *wc_w0, *wc_w1, *wc_anchor, *wc_K;
} orc_scene;

typedef struct {
    int64_t nv, nt, nwc;
    int32_t model;
    double nu, density, gravity[3];
    double *X;
    int32_t *tets;
    double *B;      /* nt*9 : Dm^{-1}; row k-1 is dN_k/dX for local node k = 1..3 */
    double *V;      /* nt   : rest measure V^0_e */
    double *mu, *lambda;
    double *fext;   /* nv*3 : consistent body force  f^ext_i = sum_e R^0 g V_e / 4 */
    char *pinned;
    int32_t *wc_n0, *wc_n1, *wc_idx0, *wc_idx1;
    double *wc_w0, *wc_w1, *wc_anchor, *wc_K;
    int64_t *vt_off; /* vertex -> incident tets, ascending tet index */
    int32_t *vt;
    int64_t *vc_off; /* vertex -> incident weak constraints, input order */
    int32_t *vc;
    int32_t *colour;
    int32_t ncolours;
    /* backward Euler (eq:fem_be): lumped masses m_i = sum_e R^0 V_e / 4, 1/dt^2 (0 =
     * quasistatic) and the inertial target xtilde_i = 2 x^n_i - x^{n-1}_i */
    double *mass;
    double inv_dt2;
    double *xtilde;
} orc_prep;

void orc_free(orc_prep *p) {
    if (!p) return;
    free(p->X); free(p->tets); free(p->B); free(p->V); free(p->mu); free(p->lambda); free(p->fext);
    free(p->pinned); free(p->wc_n0); free(p->wc_n1); free(p->wc_idx0); free(p->wc_idx1);
    free(p->wc_w0); free(p->wc_w1); free(p->wc_anchor); free(p->wc_K); free(p->vt_off); free(p->vt);
    free(p->vc_off); free(p->vc); free(p->colour); free(p->mass); free(p->xtilde);
    free(p);
}

static void *xdup(const void *src, size_t bytes) {
    void *d = malloc(bytes ? bytes : 1);
    if (d && bytes) memcpy(d, src, bytes);
    return d;
}

/* gradient of the linear shape function of local node k in tet e: k >= 1 -> row k-1 of B,
 * k = 0 -> minus the sum of the rows (the shape functions sum to one) */
static void shape_grad(const orc_prep *p, int64_t e, int k, double *g) {
    const double *B = p->B + 9 * e;
    int b;
    if (k > 0) {
        for (b = 0; b < 3; ++b) g[b] = B[3 * (k - 1) + b];
    } else {
        for (b = 0; b < 3; ++b) g[b] = -(B[b] + B[3 + b] + B[6 + b]);
    }
}

/* PBNG node colouring: visiting vertices in ascending index, colour(v) = least colour
 * not in the union of S_c over the elements / weak constraints c incident to v; then register the
 * colour in S_c for each of them.  S_c holds at most (#nodes of c) colours, so it is a short list. */
static int colour_nodes(orc_prep *p) {
    int64_t nt = p->nt, nwc = p->nwc, v, k;
    int32_t *ts_n = calloc((size_t)(nt + nwc) + 1, sizeof(int32_t));
    int32_t *ts = malloc(((size_t)(nt + nwc) * 8 + 1) * sizeof(int32_t)); /* <= 8 nodes per stencil */
    char *used = NULL;
    int32_t maxc = 0;
    if (!ts_n || !ts) { free(ts_n); free(ts); return ORC_E_NOMEM; }
    for (v = 0; v < p->nv; ++v) {
        int32_t cap = 0, c;
        /* count an upper bound for the forbidden set */
        for (k = p->vt_off[v]; k < p->vt_off[v + 1]; ++k) cap += ts_n[p->vt[k]];
        for (k = p->vc_off[v]; k < p->vc_off[v + 1]; ++k) cap += ts_n[nt + p->vc[k]];
        used = realloc(used, (size_t)cap + 2);
        memset(used, 0, (size_t)cap + 2);
        for (k = p->vt_off[v]; k < p->vt_off[v + 1]; ++k) {
            int64_t s = p->vt[k];
            int32_t q;
            for (q = 0; q < ts_n[s]; ++q)
                if (ts[8 * s + q] <= cap) used[ts[8 * s + q]] = 1;
        }
        for (k = p->vc_off[v]; k < p->vc_off[v + 1]; ++k) {
            int64_t s = nt + p->vc[k];
            int32_t q;
            for (q = 0; q < ts_n[s]; ++q)
                if (ts[8 * s + q] <= cap) used[ts[8 * s + q]] = 1;
        }
        c = 0;
        while (used[c]) ++c;
        p->colour[v] = c;
        if (c + 1 > maxc) maxc = c + 1;
        for (k = p->vt_off[v]; k < p->vt_off[v + 1]; ++k) {
            int64_t s = p->vt[k];
            ts[8 * s + ts_n[s]++] = c;
        }
        for (k = p->vc_off[v]; k < p->vc_off[v + 1]; ++k) {
            int64_t s = nt + p->vc[k];
            if (ts_n[s] < 8) ts[8 * s + ts_n[s]++] = c;
        }
    }
    p->ncolours = maxc;
    free(used); free(ts_n); free(ts);
    return ORC_OK;
}

/* builds vertex -> stencil lists; a weak constraint is listed once per distinct node */
static int build_incidence(orc_prep *p) {
    int64_t e, c, v, q;
    int64_t *cnt;
    p->vt_off = calloc((size_t)p->nv + 1, sizeof(int64_t));
    p->vc_off = calloc((size_t)p->nv + 1, sizeof(int64_t));
    cnt = calloc((size_t)p->nv + 1, sizeof(int64_t));
    if (!p->vt_off || !p->vc_off || !cnt) { free(cnt); return ORC_E_NOMEM; }
    for (e = 0; e < p->nt; ++e)
        for (q = 0; q < 4; ++q) p->vt_off[p->tets[4 * e + q] + 1]++;
    for (v = 0; v < p->nv; ++v) p->vt_off[v + 1] += p->vt_off[v];
    p->vt = malloc((size_t)(4 * p->nt + 1) * sizeof(int32_t));
    if (!p->vt) { free(cnt); return ORC_E_NOMEM; }
    for (e = 0; e < p->nt; ++e) /* ascending e -> each list ascending */
        for (q = 0; q < 4; ++q) {
            v = p->tets[4 * e + q];
            p->vt[p->vt_off[v] + cnt[v]++] = (int32_t)e;
        }
    memset(cnt, 0, (size_t)(p->nv + 1) * sizeof(int64_t));
    /* weak constraints: node list = side-0 nodes then side-1 nodes, deduplicated per constraint */
    for (c = 0; c < p->nwc; ++c) {
        int32_t nodes[8], nn = 0, a, b;
        for (a = 0; a < p->wc_n0[c]; ++a) nodes[nn++] = p->wc_idx0[4 * c + a];
        for (a = 0; a < p->wc_n1[c]; ++a) nodes[nn++] = p->wc_idx1[4 * c + a];
        for (a = 0; a < nn; ++a) {
            int dup = 0;
            for (b = 0; b < a; ++b) dup |= nodes[b] == nodes[a];
            if (!dup) p->vc_off[nodes[a] + 1]++;
        }
    }
    for (v = 0; v < p->nv; ++v) p->vc_off[v + 1] += p->vc_off[v];
    p->vc = malloc((size_t)(p->vc_off[p->nv] + 1) * sizeof(int32_t));
    if (!p->vc) { free(cnt); return ORC_E_NOMEM; }
    for (c = 0; c < p->nwc; ++c) {
        int32_t nodes[8], nn = 0, a, b;
        for (a = 0; a < p->wc_n0[c]; ++a) nodes[nn++] = p->wc_idx0[4 * c + a];
        for (a = 0; a < p->wc_n1[c]; ++a) nodes[nn++] = p->wc_idx1[4 * c + a];
        for (a = 0; a < nn; ++a) {
            int dup = 0;
            for (b = 0; b < a; ++b) dup |= nodes[b] == nodes[a];
            if (!dup) {
                v = nodes[a];
                p->vc[p->vc_off[v] + cnt[v]++] = (int32_t)c;
            }
        }
    }
    free(cnt);
    return ORC_OK;
}

/* Set-up: copy the scene, rest precompute (Dm, Dm^{-1}, V^0_e), Lame per tet
 * (eq:lame), body force, incidence and colouring.  *bad receives the offending index. */
int orc_prepare(const orc_scene *s, orc_prep **out, int64_t *bad) {
    orc_prep *p;
    int64_t e, v, k, c;
    int st;
    *out = NULL;
    if (bad) *bad = -1;
    if (s->nv <= 0 || s->nt < 0 || (s->model != ORC_NH && s->model != ORC_FCR && s->model != ORC_SNH)) return ORC_E_ARG;
    if (s->nE != 1 && s->nE != s->nt) return ORC_E_ARG;
    if (!(s->nu >= 0.0 && s->nu < 0.5)) return ORC_E_ARG;
    for (e = 0; e < s->nt * 4; ++e)
        if (s->tets[e] < 0 || s->tets[e] >= s->nv) { if (bad) *bad = e / 4; return ORC_E_ARG; }
    for (k = 0; k < s->npin; ++k)
        if (s->pinned[k] < 0 || s->pinned[k] >= s->nv) { if (bad) *bad = k; return ORC_E_ARG; }
    for (c = 0; c < s->nwc; ++c) {
        int a;
        if (s->wc_n0[c] < 1 || s->wc_n0[c] > 4 || s->wc_n1[c] < 0 || s->wc_n1[c] > 4) { if (bad) *bad = c; return ORC_E_ARG; }
        for (a = 0; a < s->wc_n0[c]; ++a)
            if (s->wc_idx0[4 * c + a] < 0 || s->wc_idx0[4 * c + a] >= s->nv) { if (bad) *bad = c; return ORC_E_ARG; }
        for (a = 0; a < s->wc_n1[c]; ++a)
            if (s->wc_idx1[4 * c + a] < 0 || s->wc_idx1[4 * c + a] >= s->nv) { if (bad) *bad = c; return ORC_E_ARG; }
    }
    p = calloc(1, sizeof(orc_prep));
    if (!p) return ORC_E_NOMEM;
    p->nv = s->nv; p->nt = s->nt; p->nwc = s->nwc; p->model = s->model; p->nu = s->nu;
    p->density = s->density;
    for (k = 0; k < 3; ++k) p->gravity[k] = s->gravity[k];
    p->X = xdup(s->X, (size_t)s->nv * 3 * sizeof(double));
    p->tets = xdup(s->tets, (size_t)s->nt * 4 * sizeof(int32_t));
    p->wc_n0 = xdup(s->wc_n0, (size_t)s->nwc * sizeof(int32_t));
    p->wc_n1 = xdup(s->wc_n1, (size_t)s->nwc * sizeof(int32_t));
    p->wc_idx0 = xdup(s->wc_idx0, (size_t)s->nwc * 4 * sizeof(int32_t));
    p->wc_idx1 = xdup(s->wc_idx1, (size_t)s->nwc * 4 * sizeof(int32_t));
    p->wc_w0 = xdup(s->wc_w0, (size_t)s->nwc * 4 * sizeof(double));
    p->wc_w1 = xdup(s->wc_w1, (size_t)s->nwc * 4 * sizeof(double));
    p->wc_anchor = xdup(s->wc_anchor, (size_t)s->nwc * 3 * sizeof(double));
    p->wc_K = xdup(s->wc_K, (size_t)s->nwc * 6 * sizeof(double));
    p->B = malloc((size_t)(s->nt * 9 + 1) * sizeof(double));
    p->V = malloc((size_t)(s->nt + 1) * sizeof(double));
    p->mu = malloc((size_t)(s->nt + 1) * sizeof(double));
    p->lambda = malloc((size_t)(s->nt + 1) * sizeof(double));
    p->fext = calloc((size_t)s->nv * 3, sizeof(double));
    p->pinned = calloc((size_t)s->nv, 1);
    p->colour = malloc((size_t)s->nv * sizeof(int32_t));
    p->mass = calloc((size_t)s->nv, sizeof(double));
    p->xtilde = calloc((size_t)s->nv * 3, sizeof(double));
    p->inv_dt2 = 0.0;
    if (!p->X || !p->tets || !p->B || !p->V || !p->mu || !p->lambda || !p->fext || !p->pinned || !p->colour ||
        !p->mass || !p->xtilde) {
        orc_free(p);
        return ORC_E_NOMEM;
    }
    for (k = 0; k < s->npin; ++k) p->pinned[s->pinned[k]] = 1;
    for (e = 0; e < s->nt; ++e) {
        const int32_t *t = p->tets + 4 * e;
        double Dm[9], adj[9], det, ell = 0.0;
        int a, b;
        int pa[6] = {0, 0, 0, 1, 1, 2}, pb[6] = {1, 2, 3, 2, 3, 3};
        /* Dm = [X1 - X0, X2 - X0, X3 - X0] (columns) */
        for (a = 0; a < 3; ++a)
            for (b = 0; b < 3; ++b) Dm[3 * a + b] = p->X[3 * t[b + 1] + a] - p->X[3 * t[0] + a];
        det = det3(Dm);
        for (a = 0; a < 6; ++a) {
            double d[3];
            for (b = 0; b < 3; ++b) d[b] = p->X[3 * t[pa[a]] + b] - p->X[3 * t[pb[a]] + b];
            ell += norm3(d) / 6.0;
        }
        if (!(fabs(det) > 1e-12 * ell * ell * ell)) {
            if (bad) *bad = e;
            orc_free(p);
            return ORC_E_DEGENERATE;
        }
        /* B = Dm^{-1} = adj(Dm) / det = cof(Dm)^T / det */
        orc_cofactor(Dm, adj);
        for (a = 0; a < 3; ++a)
            for (b = 0; b < 3; ++b) p->B[9 * e + 3 * a + b] = adj[3 * b + a] / det;
        p->V[e] = fabs(det) / 6.0;
        if (orc_lame(s->E[s->nE == 1 ? 0 : e], s->nu, &p->mu[e], &p->lambda[e]) != ORC_OK) {
            if (bad) *bad = e;
            orc_free(p);
            return ORC_E_ARG;
        }
        for (a = 0; a < 4; ++a) {
            for (b = 0; b < 3; ++b) p->fext[3 * t[a] + b] += p->density * p->gravity[b] * p->V[e] / 4.0;
            p->mass[t[a]] += p->density * p->V[e] / 4.0; /* m_ii = int R^0 N_i dX */
        }
    }
    st = build_incidence(p);
    if (st != ORC_OK) { orc_free(p); return st; }
    for (v = 0; v < p->nv; ++v)
        if (!p->pinned[v] && p->vt_off[v + 1] == p->vt_off[v] && p->vc_off[v + 1] == p->vc_off[v]) {
            if (bad) *bad = v;
            orc_free(p);
            return ORC_E_ISOLATED;
        }
    st = colour_nodes(p);
    if (st != ORC_OK) { orc_free(p); return st; }
    *out = p;
    return ORC_OK;
}

int32_t orc_num_colours(const orc_prep *p) { return p->ncolours; }
void orc_get_colour(const orc_prep *p, int32_t *out) { memcpy(out, p->colour, (size_t)p->nv * sizeof(int32_t)); }
void orc_get_rest(const orc_prep *p, double *B, double *V) {
    memcpy(B, p->B, (size_t)p->nt * 9 * sizeof(double));
    memcpy(V, p->V, (size_t)p->nt * sizeof(double));
}
void orc_get_fext(const orc_prep *p, double *out) { memcpy(out, p->fext, (size_t)p->nv * 3 * sizeof(double)); }

/* deformation gradient of tet e (eq:disc_pe): F = sum_j y_j (dN_j/dX)^T */
static void deformation_gradient(const orc_prep *p, const double *y, int64_t e, double *F) {
    int j, a, b;
    double g[3];
    for (a = 0; a < 9; ++a) F[a] = 0.0;
    for (j = 0; j < 4; ++j) {
        const double *yj = y + 3 * (int64_t)p->tets[4 * e + j];
        shape_grad(p, e, j, g);
        for (a = 0; a < 3; ++a)
            for (b = 0; b < 3; ++b) F[3 * a + b] += yj[a] * g[b];
    }
}

void orc_deformation_gradient(const orc_prep *p, const double *y, int64_t e, double *F) {
    deformation_gradient(p, y, e, F);
}

/* C_c(y) = sum_j w0_j y_j - sum_j w1_j y_j; side 1 empty -> fixed anchor point */
static void constraint_value(const orc_prep *p, const double *y, int64_t c, double *C) {
    int a, b;
    for (b = 0; b < 3; ++b) C[b] = 0.0;
    for (a = 0; a < p->wc_n0[c]; ++a)
        for (b = 0; b < 3; ++b) C[b] += p->wc_w0[4 * c + a] * y[3 * (int64_t)p->wc_idx0[4 * c + a] + b];
    if (p->wc_n1[c] == 0) {
        for (b = 0; b < 3; ++b) C[b] -= p->wc_anchor[3 * c + b];
    } else {
        for (a = 0; a < p->wc_n1[c]; ++a)
            for (b = 0; b < 3; ++b) C[b] -= p->wc_w1[4 * c + a] * y[3 * (int64_t)p->wc_idx1[4 * c + a] + b];
    }
}

static void constraint_K(const orc_prep *p, int64_t c, double *K) {
    const double *k = p->wc_K + 6 * c; /* xx yy zz xy yz xz */
    K[0] = k[0]; K[1] = k[3]; K[2] = k[5];
    K[3] = k[3]; K[4] = k[1]; K[5] = k[4];
    K[6] = k[5]; K[7] = k[4]; K[8] = k[2];
}

/* w^c_{0i} - w^c_{1i} */
static double constraint_weight_diff(const orc_prep *p, int64_t c, int64_t i) {
    double d = 0.0;
    int a;
    for (a = 0; a < p->wc_n0[c]; ++a)
        if (p->wc_idx0[4 * c + a] == i) d += p->wc_w0[4 * c + a];
    for (a = 0; a < p->wc_n1[c]; ++a)
        if (p->wc_idx1[4 * c + a] == i) d -= p->wc_w1[4 * c + a];
    return d;
}

/* The right-hand side f_i(y) + f^ext_i of eq:pbgn_dx and the modified nodal Hessian A of eq:mod_hess,
 * for node i at positions y:
 *   f_i = - sum_e P_e(y) dN_i/dX V_e - sum_c (w0_ci - w1_ci) K_c C_c(y)
 *   A_ab = sum_e sum_{gamma,delta} Ctilde_{a gamma b delta} (dN_i/dX)_gamma (dN_i/dX)_delta V_e
 *          + sum_c (w0_ci - w1_ci)^2 K_c,ab                                                        */
void orc_nodal(const orc_prep *p, const double *y, int64_t i, double *f, double *A) {
    int64_t k;
    int a, b, ga, de;
    for (a = 0; a < 3; ++a) f[a] = p->fext[3 * i + a];
    for (a = 0; a < 9; ++a) A[a] = 0.0;
    for (k = p->vt_off[i]; k < p->vt_off[i + 1]; ++k) {
        int64_t e = p->vt[k];
        int slot = 0;
        double F[9], P[9], T[81], g[3], Ve = p->V[e];
        while (p->tets[4 * e + slot] != i) ++slot;
        shape_grad(p, e, slot, g);
        deformation_gradient(p, y, e, F);
        orc_piola(p->model, p->mu[e], p->lambda[e], F, P);
        for (a = 0; a < 3; ++a)
            for (b = 0; b < 3; ++b) f[a] -= P[3 * a + b] * g[b] * Ve;
        orc_mod_hess_density(p->mu[e], p->lambda[e], F, T);
        for (a = 0; a < 3; ++a)
            for (b = 0; b < 3; ++b) {
                double s = 0.0;
                for (ga = 0; ga < 3; ++ga)
                    for (de = 0; de < 3; ++de) s += T[(3 * a + ga) * 9 + 3 * b + de] * g[ga] * g[de];
                A[3 * a + b] += s * Ve;
            }
    }
    for (k = p->vc_off[i]; k < p->vc_off[i + 1]; ++k) {
        int64_t c = p->vc[k];
        double C[3], K[9], d = constraint_weight_diff(p, c, i);
        constraint_value(p, y, c, C);
        constraint_K(p, c, K);
        for (a = 0; a < 3; ++a)
            for (b = 0; b < 3; ++b) {
                f[a] -= d * K[3 * a + b] * C[b];
                A[3 * a + b] += d * d * K[3 * a + b];
            }
    }
    /* backward Euler: the node's share of the incremental potential m_i / (2 dt^2) |y_i - xtilde_i|^2 adds
     * -m_i (y_i - xtilde_i) / dt^2 to the right-hand side and m_i / dt^2 I to A (eq:fem_be) */
    if (p->inv_dt2 > 0.0) {
        const double m = p->mass[i] * p->inv_dt2;
        for (a = 0; a < 3; ++a) {
            f[a] -= m * (y[3 * i + a] - p->xtilde[3 * i + a]);
            A[4 * a] += m;
        }
    }
}

/* backward-Euler mode: dt > 0 with xtilde (nv*3) = 2 x^n - x^{n-1}; dt == 0 returns to quasistatics */
int orc_set_inertia(orc_prep *p, double dt, const double *xtilde) {
    if (!(dt >= 0.0)) return ORC_E_ARG;
    if (dt == 0.0) {
        p->inv_dt2 = 0.0;
        return ORC_OK;
    }
    if (!xtilde) return ORC_E_ARG;
    p->inv_dt2 = 1.0 / (dt * dt);
    memcpy(p->xtilde, xtilde, (size_t)p->nv * 3 * sizeof(double));
    return ORC_OK;
}

void orc_get_mass(const orc_prep *p, double *out) { memcpy(out, p->mass, (size_t)p->nv * sizeof(double)); }

/* solve the 3x3 SPD system A dx = r by Cholesky (plain, fp64) */
static int spd_solve3(const double *A, const double *r, double *x) {
    double L[9] = {0}, z[3];
    int i, j, k;
    for (j = 0; j < 3; ++j) {
        double s = A[3 * j + j];
        for (k = 0; k < j; ++k) s -= L[3 * j + k] * L[3 * j + k];
        if (!(s > 0.0)) return 1;
        L[3 * j + j] = sqrt(s);
        for (i = j + 1; i < 3; ++i) {
            double t = A[3 * i + j];
            for (k = 0; k < j; ++k) t -= L[3 * i + k] * L[3 * j + k];
            L[3 * i + j] = t / L[3 * j + j];
        }
    }
    for (i = 0; i < 3; ++i) {
        double s = r[i];
        for (k = 0; k < i; ++k) s -= L[3 * i + k] * z[k];
        z[i] = s / L[3 * i + i];
    }
    for (i = 2; i >= 0; --i) {
        double s = z[i];
        for (k = i + 1; k < 3; ++k) s -= L[3 * k + i] * x[k];
        x[i] = s / L[3 * i + i];
    }
    return 0;
}

/* One PBNG iteration in place: colours in ascending order; within a
 * colour, free nodes in ascending index; each node takes ONE modified-Newton step from a zero initial
 * guess, x_i += A^{-1} (f_i + f^ext_i), with no line search.  Returns the number of failed solves. */
int64_t orc_sweep_colour(const orc_prep *p, double *w, int32_t c) {
    int64_t i, fails = 0;
    /* The paper's own implementation runs this loop in parallel with OpenMP.  Node i reads
     * only nodes of other colours, which this pass does not write, so every node's
     * update is independent of the order and of the thread count: the OpenMP build (liborc_omp.so) is
     * bitwise identical to the serial one (pinned by tests/test_oracle_openmp.py). */
#pragma omp parallel for schedule(dynamic, 512) reduction(+ : fails)
    for (i = 0; i < p->nv; ++i) {
        double f[3], A[9], dx[3];
        if (p->colour[i] != c || p->pinned[i]) continue;
        orc_nodal(p, w, i, f, A);
        if (spd_solve3(A, f, dx)) { ++fails; continue; }
        w[3 * i + 0] += dx[0];
        w[3 * i + 1] += dx[1];
        w[3 * i + 2] += dx[2];
    }
    return fails;
}

int64_t orc_sweep(const orc_prep *p, double *w) {
    int32_t c;
    int64_t fails = 0;
    for (c = 0; c < p->ncolours; ++c) fails += orc_sweep_colour(p, w, c);
    return fails;
}

/* Chebyshev weight omega_m (reading Z5): omega_m = 1 for m <= 2, omega_3 = 2/(2-rho^2),
 * omega_m = 4/(4 - rho^2 omega_{m-1}) for m > 3. */
double orc_chebyshev_omega(int64_t m, double rho) {
    double om;
    int64_t k;
    if (m <= 2) return 1.0;
    om = 2.0 / (2.0 - rho * rho);
    for (k = 4; k <= m; ++k) om = 4.0 / (4.0 - rho * rho * om);
    return om;
}

/* n accelerated iterations starting at iteration index l0.
 *   x   : x^{l}   (in), x^{l0+n}   (out)
 *   xm1 : x^{l-1} (in), x^{l0+n-1} (out)   (caller sets xm1 = x^0 when l0 == 0, reading Z8)
 * none      : x^{l+1} = x_PBNG
 * SOR       : x^{l+1} = omega (x_PBNG - x^{l-1}) + x^{l-1}
 * Chebyshev : x^{l+1} = omega_{l+1} (gamma (x_PBNG - x^l) + x^l - x^{l-1}) + x^{l-1}
 * Dirichlet rows are never updated (reading Z9).  Returns the number of failed nodal solves. */
int64_t orc_iterate(const orc_prep *p, double *x, double *xm1, int64_t l0, int32_t n, int32_t accel,
                    double omega, double rho, double gamma) {
    int64_t N = p->nv * 3, l, k, fails = 0;
    double *w = malloc((size_t)N * sizeof(double));
    if (!w) return -1;
    for (l = l0; l < l0 + n; ++l) {
        double om = orc_chebyshev_omega(l + 1, rho);
        memcpy(w, x, (size_t)N * sizeof(double));
        fails += orc_sweep(p, w);
#pragma omp parallel for schedule(static)
        for (k = 0; k < N; ++k) {
            double xl = x[k], xl1 = xm1[k], xn;
            if (p->pinned[k / 3]) continue;
            if (accel == ORC_ACCEL_SOR) {
                xn = omega * (w[k] - xl1) + xl1;
            } else if (accel == ORC_ACCEL_CHEBYSHEV) {
                xn = om * (gamma * (w[k] - xl) + xl - xl1) + xl1;
            } else {
                xn = w[k];
            }
            xm1[k] = xl;
            x[k] = xn;
        }
    }
    free(w);
    return fails;
}

/* r_i = f_i(y) + f^ext_i for every node (pinned included; the residual norm skips them) */
void orc_forces(const orc_prep *p, const double *y, double *r) {
    int64_t i;
#pragma omp parallel for schedule(dynamic, 512)
    for (i = 0; i < p->nv; ++i) {
        double A[9];
        orc_nodal(p, y, i, r + 3 * i, A);
    }
}

/* Newton residual 2-norm over free nodes (Fig. 10 caption; reading Z14) */
double orc_residual(const orc_prep *p, const double *y) {
    int64_t i;
    double s = 0.0;
    double *r = malloc((size_t)p->nv * 3 * sizeof(double));
    if (!r) return NAN;
    orc_forces(p, y, r); /* per node, then summed in ascending node order (thread-count independent) */
    for (i = 0; i < p->nv; ++i) {
        const double *f = r + 3 * i;
        if (p->pinned[i]) continue;
        s += f[0] * f[0] + f[1] * f[1] + f[2] * f[2];
    }
    free(r);
    return sqrt(s);
}

/* total energy PE^Psi(y) + PE^wc(y) - y . f^ext (reading Z13);
 * parts (optional): [elastic, weak-constraint, external-work] */
double orc_energy(const orc_prep *p, const double *y, double *parts) {
    int64_t e, c, i;
    double el = 0.0, wc = 0.0, ext = 0.0;
    double *psi = malloc((size_t)(p->nt > 0 ? p->nt : 1) * sizeof(double));
    if (!psi) return NAN;
    /* per-element V_e Psi(F_e), then summed in ascending element order (thread-count independent) */
#pragma omp parallel for schedule(static)
    for (e = 0; e < p->nt; ++e) {
        double F[9];
        deformation_gradient(p, y, e, F);
        psi[e] = p->V[e] * orc_psi(p->model, p->mu[e], p->lambda[e], F, 0);
    }
    for (e = 0; e < p->nt; ++e) el += psi[e];
    free(psi);
    for (c = 0; c < p->nwc; ++c) {
        double C[3], K[9];
        int a, b;
        constraint_value(p, y, c, C);
        constraint_K(p, c, K);
        for (a = 0; a < 3; ++a)
            for (b = 0; b < 3; ++b) wc += 0.5 * C[a] * K[3 * a + b] * C[b];
    }
    for (i = 0; i < p->nv * 3; ++i) ext -= y[i] * p->fext[i];
    if (p->inv_dt2 > 0.0) /* incremental potential: inertia of the free nodes (pinned nodes are constant) */
        for (i = 0; i < p->nv; ++i) {
            int a;
            if (p->pinned[i]) continue;
            for (a = 0; a < 3; ++a) {
                const double dx = y[3 * i + a] - p->xtilde[3 * i + a];
                ext += 0.5 * p->inv_dt2 * p->mass[i] * dx * dx;
            }
        }
    if (parts) { parts[0] = el; parts[1] = wc; parts[2] = ext; }
    return el + wc + ext;
}

/* ------------------------------------------------------------------------------------------------ */
/* Dynamic weak constraints                                                      */
/* ------------------------------------------------------------------------------------------------ */

/* Incremental node recolouring, PAPER.md:748-754 ("Collision Coloring"): only the nodes incident to the
 * newly added weak constraints are recoloured; for each such node x the used colour set is the union
 * of the colours of the stencils containing x; x keeps its previous colour as the initial guess unless
 * that colour is used, in which case it takes the minimal unused colour.  Reading Z20 (the paper is
 * silent on the order): the nodes are visited in ascending index and a node's used set sees the NEW
 * colours of the nodes visited before it; a stencil's colours exclude x itself.
 * Stencils: the nt tets (4 nodes each) and the nc constraints of the NEW constraint set (node lists in
 * CSR c_off / c_nodes, duplicates allowed); is_new[c] != 0 marks the newly added ones.
 * Returns the number of nodes whose colour changed in *n_changed (optional). */
int orc_recolor_incremental(int64_t nv, int64_t nt, const int32_t *tets, int64_t nc, const int64_t *c_off,
                            const int32_t *c_nodes, const uint8_t *is_new, const int32_t *colour_prev,
                            int32_t *colour_out, int64_t *n_changed) {
    int64_t v, e, c, k, changed = 0;
    int64_t *vs_off = calloc((size_t)nv + 1, sizeof(int64_t));
    int64_t *vs, *fill;
    uint8_t *extra = calloc((size_t)nv + 1, 1);
    int32_t maxc = 0;
    char *used;
    if (!vs_off || !extra) { free(vs_off); free(extra); return ORC_E_NOMEM; }
    for (v = 0; v < nv; ++v) {
        colour_out[v] = colour_prev[v];
        if (colour_prev[v] + 1 > maxc) maxc = colour_prev[v] + 1;
    }
    /* vertex -> stencil incidence (stencil id: tets 0..nt-1, constraint c -> nt + c) */
    for (e = 0; e < nt; ++e)
        for (k = 0; k < 4; ++k) vs_off[tets[4 * e + k] + 1]++;
    for (c = 0; c < nc; ++c)
        for (k = c_off[c]; k < c_off[c + 1]; ++k) vs_off[c_nodes[k] + 1]++;
    for (v = 0; v < nv; ++v) vs_off[v + 1] += vs_off[v];
    vs = malloc(((size_t)vs_off[nv] + 1) * sizeof(int64_t));
    fill = malloc(((size_t)nv + 1) * sizeof(int64_t));
    used = malloc((size_t)maxc + 8 * (size_t)(nc + 1) + 64);
    if (!vs || !fill || !used) { free(vs_off); free(extra); free(vs); free(fill); free(used); return ORC_E_NOMEM; }
    memcpy(fill, vs_off, (size_t)nv * sizeof(int64_t));
    for (e = 0; e < nt; ++e)
        for (k = 0; k < 4; ++k) vs[fill[tets[4 * e + k]]++] = e;
    for (c = 0; c < nc; ++c)
        for (k = c_off[c]; k < c_off[c + 1]; ++k) vs[fill[c_nodes[k]]++] = nt + c;
    /* the nodes incident to newly added constraints */
    for (c = 0; c < nc; ++c)
        if (is_new[c])
            for (k = c_off[c]; k < c_off[c + 1]; ++k) extra[c_nodes[k]] = 1;
    for (v = 0; v < nv; ++v) {
        int64_t q;
        int32_t col, cap;
        if (!extra[v]) continue;
        cap = maxc + 1;
        memset(used, 0, (size_t)cap + 1);
        for (q = vs_off[v]; q < vs_off[v + 1]; ++q) {
            const int64_t s = vs[q];
            if (s < nt) {
                for (k = 0; k < 4; ++k)
                    if (tets[4 * s + k] != v) used[colour_out[tets[4 * s + k]]] = 1;
            } else {
                for (k = c_off[s - nt]; k < c_off[s - nt + 1]; ++k)
                    if (c_nodes[k] != v) used[colour_out[c_nodes[k]]] = 1;
            }
        }
        if (used[colour_prev[v]]) {
            col = 0;
            while (used[col]) ++col;
            colour_out[v] = col;
            if (col + 1 > maxc) maxc = col + 1;
            ++changed;
        }
    }
    if (n_changed) *n_changed = changed;
    free(vs_off); free(extra); free(vs); free(fill); free(used);
    return ORC_OK;
}

/* Closest point of triangle (a, b, c) to p, as barycentric weights (u, v, w): q = u a + v b + w c.
 * Textbook Voronoi-region classification: vertex regions, then edge regions, then the interior. */
void orc_closest_point_triangle(const double *p, const double *a, const double *b, const double *c, double *bary) {
    double ab[3], ac[3], ap[3], bp[3], cp[3];
    double d1, d2, d3, d4, d5, d6, va, vb, vc, t, den;
    int k;
    for (k = 0; k < 3; ++k) {
        ab[k] = b[k] - a[k];
        ac[k] = c[k] - a[k];
        ap[k] = p[k] - a[k];
        bp[k] = p[k] - b[k];
        cp[k] = p[k] - c[k];
    }
    d1 = ab[0] * ap[0] + ab[1] * ap[1] + ab[2] * ap[2];
    d2 = ac[0] * ap[0] + ac[1] * ap[1] + ac[2] * ap[2];
    if (d1 <= 0.0 && d2 <= 0.0) { bary[0] = 1.0; bary[1] = 0.0; bary[2] = 0.0; return; }
    d3 = ab[0] * bp[0] + ab[1] * bp[1] + ab[2] * bp[2];
    d4 = ac[0] * bp[0] + ac[1] * bp[1] + ac[2] * bp[2];
    if (d3 >= 0.0 && d4 <= d3) { bary[0] = 0.0; bary[1] = 1.0; bary[2] = 0.0; return; }
    vc = d1 * d4 - d3 * d2;
    if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
        t = d1 / (d1 - d3);
        bary[0] = 1.0 - t; bary[1] = t; bary[2] = 0.0;
        return;
    }
    d5 = ab[0] * cp[0] + ab[1] * cp[1] + ab[2] * cp[2];
    d6 = ac[0] * cp[0] + ac[1] * cp[1] + ac[2] * cp[2];
    if (d6 >= 0.0 && d5 <= d6) { bary[0] = 0.0; bary[1] = 0.0; bary[2] = 1.0; return; }
    vb = d5 * d2 - d1 * d6;
    if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
        t = d2 / (d2 - d6);
        bary[0] = 1.0 - t; bary[1] = 0.0; bary[2] = t;
        return;
    }
    va = d3 * d6 - d5 * d4;
    if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) {
        t = (d4 - d3) / ((d4 - d3) + (d5 - d6));
        bary[0] = 0.0; bary[1] = 1.0 - t; bary[2] = t;
        return;
    }
    den = 1.0 / (va + vb + vc);
    bary[1] = vb * den;
    bary[2] = vc * den;
    bary[0] = 1.0 - bary[1] - bary[2];
}

/* Boundary triangles of a tet mesh: the faces that belong to exactly one tet, in order of (tet index,
 * local face k), face k = the three vertices other than local vertex k, oriented so that the normal
 * (v1 - v0) x (v2 - v0) points away from the tet's vertex k at the REST positions X.  tri (capacity
 * 3 * 4 nt) receives the vertex triples, tri_tet the owning tet; returns the count. */
int64_t orc_surface(int64_t nt, const int32_t *tets, const double *X, int32_t *tri, int32_t *tri_tet) {
    int64_t e, f, n = 0;
    /* a face is interior iff another tet has the same vertex set: brute-force key compare over all faces
     * (sorted triples, quadratic in the face count is too slow, so sort the keys) */
    int64_t nf = 4 * nt, i, j;
    int64_t *key = malloc((size_t)(nf + 1) * 3 * sizeof(int64_t));
    int64_t *idx = malloc((size_t)(nf + 1) * sizeof(int64_t));
    uint8_t *interior = calloc((size_t)nf + 1, 1);
    if (!key || !idx || !interior) { free(key); free(idx); free(interior); return -1; }
    for (e = 0; e < nt; ++e)
        for (f = 0; f < 4; ++f) {
            int32_t v[3], m = 0, k, t;
            for (k = 0; k < 4; ++k)
                if (k != f) v[m++] = tets[4 * e + k];
            /* sort the triple */
            if (v[0] > v[1]) { t = v[0]; v[0] = v[1]; v[1] = t; }
            if (v[1] > v[2]) { t = v[1]; v[1] = v[2]; v[2] = t; }
            if (v[0] > v[1]) { t = v[0]; v[0] = v[1]; v[1] = t; }
            key[3 * (4 * e + f)] = v[0]; key[3 * (4 * e + f) + 1] = v[1]; key[3 * (4 * e + f) + 2] = v[2];
            idx[4 * e + f] = 4 * e + f;
        }
    /* insertion-free sort: simple bottom-up merge sort of idx by key */
    {
        int64_t *tmp = malloc((size_t)(nf + 1) * sizeof(int64_t)), w;
        if (!tmp) { free(key); free(idx); free(interior); return -1; }
        for (w = 1; w < nf; w *= 2) {
            for (i = 0; i < nf; i += 2 * w) {
                int64_t lo = i, mid = i + w < nf ? i + w : nf, hi = i + 2 * w < nf ? i + 2 * w : nf;
                int64_t a = lo, b = mid, o = lo;
                while (a < mid && b < hi) {
                    const int64_t *ka = key + 3 * idx[a], *kb = key + 3 * idx[b];
                    int less = ka[0] < kb[0] || (ka[0] == kb[0] && (ka[1] < kb[1] || (ka[1] == kb[1] && ka[2] <= kb[2])));
                    tmp[o++] = less ? idx[a++] : idx[b++];
                }
                while (a < mid) tmp[o++] = idx[a++];
                while (b < hi) tmp[o++] = idx[b++];
            }
            memcpy(idx, tmp, (size_t)nf * sizeof(int64_t));
        }
        free(tmp);
    }
    for (i = 0; i + 1 < nf; ++i) {
        const int64_t *ka = key + 3 * idx[i];
        for (j = i + 1; j < nf; ++j) {
            const int64_t *kb = key + 3 * idx[j];
            if (ka[0] != kb[0] || ka[1] != kb[1] || ka[2] != kb[2]) break;
            interior[idx[i]] = 1;
            interior[idx[j]] = 1;
        }
    }
    for (e = 0; e < nt; ++e)
        for (f = 0; f < 4; ++f) {
            int32_t v[3], m = 0, k;
            double u[3], w[3], nrm[3], d[3], s;
            if (interior[4 * e + f]) continue;
            for (k = 0; k < 4; ++k)
                if (k != f) v[m++] = tets[4 * e + k];
            for (k = 0; k < 3; ++k) {
                u[k] = X[3 * v[1] + k] - X[3 * v[0] + k];
                w[k] = X[3 * v[2] + k] - X[3 * v[0] + k];
                d[k] = X[3 * tets[4 * e + f] + k] - X[3 * v[0] + k];
            }
            cross3(u, w, nrm);
            s = nrm[0] * d[0] + nrm[1] * d[1] + nrm[2] * d[2];
            if (s > 0.0) { int32_t t = v[1]; v[1] = v[2]; v[2] = t; } /* vertex k must lie behind */
            tri[3 * n] = v[0]; tri[3 * n + 1] = v[1]; tri[3 * n + 2] = v[2];
            tri_tet[n] = (int32_t)e;
            ++n;
        }
    free(key); free(idx); free(interior);
    return n;
}

/* Bodies: connected components of the tets (two tets are connected when they share a vertex); body[v]
 * = smallest vertex index of v's component (vertices in no tet are their own body). */
void orc_bodies(int64_t nv, int64_t nt, const int32_t *tets, int32_t *body) {
    int64_t v, e, k;
    int changed = 1;
    for (v = 0; v < nv; ++v) body[v] = (int32_t)v;
    while (changed) { /* label propagation to the component minimum (plain fixed-point iteration) */
        changed = 0;
        for (e = 0; e < nt; ++e) {
            int32_t m = body[tets[4 * e]];
            for (k = 1; k < 4; ++k)
                if (body[tets[4 * e + k]] < m) m = body[tets[4 * e + k]];
            for (k = 0; k < 4; ++k)
                if (body[tets[4 * e + k]] != m) { body[tets[4 * e + k]] = m; changed = 1; }
        }
        for (v = 0; v < nv; ++v) /* path compression: follow labels to their fixed point */
            while (body[body[v]] != body[v]) body[v] = body[body[v]];
    }
}

/* Contact weak constraints at positions y (the paper builds collision weak constraints
 * dynamically but specifies no detection scheme, PAPER.md:843-846 -- reading Z21): for every free vertex
 * of a boundary triangle, the closest boundary triangle of ANOTHER body (orc_bodies) whose closest point
 * is within `thickness` (|p - q|^2 <= thickness^2); among the triangles whose squared distance is within
 * 1e-10 thickness^2 of the least one (shared edges / vertices), the lowest triangle index.  The constraint has side
 * 0 = the vertex (weight 1), side 1 = the triangle's vertices with the closest point's barycentric
 * weights, and K = k_n n n^T with n the triangle's unit normal at y (k_tau = 0).
 * Outputs per vertex (dense, nv entries): tri_out (3 ids, -1 if none), bary (3), normal (3).
 * Brute force over all triangle pairs (test sizes only).  Returns the number of contacts. */
int64_t orc_detect_contacts(int64_t nv, const double *X, const double *y, int64_t nt, const int32_t *tets,
                            const uint8_t *is_free, double thickness, int32_t *tri_out, double *bary_out,
                            double *normal_out) {
    int32_t *tri = malloc((size_t)(12 * nt + 3) * sizeof(int32_t));
    int32_t *tri_tet = malloc((size_t)(4 * nt + 1) * sizeof(int32_t));
    int32_t *body = malloc((size_t)(nv + 1) * sizeof(int32_t));
    uint8_t *on_surf = calloc((size_t)nv + 1, 1);
    int64_t ntri, v, t, found = 0;
    int pass;
    if (!tri || !tri_tet || !body || !on_surf) { free(tri); free(tri_tet); free(body); free(on_surf); return -1; }
    ntri = orc_surface(nt, tets, X, tri, tri_tet);
    orc_bodies(nv, nt, tets, body);
    for (t = 0; t < 3 * ntri; ++t) on_surf[tri[t]] = 1;
    for (v = 0; v < nv; ++v) {
        double best = 0.0, bb[3] = {0, 0, 0};
        int64_t bt = -1;
        tri_out[3 * v] = tri_out[3 * v + 1] = tri_out[3 * v + 2] = -1;
        bary_out[3 * v] = bary_out[3 * v + 1] = bary_out[3 * v + 2] = 0.0;
        normal_out[3 * v] = normal_out[3 * v + 1] = normal_out[3 * v + 2] = 0.0;
        if (!on_surf[v] || !is_free[v]) continue;
        /* pass 1: the least squared distance; pass 2: the lowest-index triangle within 1e-10 thickness^2 of
         * it (a closest point on an edge or vertex shared by several triangles is a tie, reading Z21) */
        for (pass = 0; pass < 2; ++pass)
            for (t = 0; t < ntri; ++t) {
                const int32_t *tv = tri + 3 * t;
                double br[3], q[3], d2 = 0.0;
                int k;
                if (body[tv[0]] == body[v]) continue;
                orc_closest_point_triangle(y + 3 * v, y + 3 * tv[0], y + 3 * tv[1], y + 3 * tv[2], br);
                for (k = 0; k < 3; ++k) {
                    q[k] = br[0] * y[3 * tv[0] + k] + br[1] * y[3 * tv[1] + k] + br[2] * y[3 * tv[2] + k];
                    d2 += (y[3 * v + k] - q[k]) * (y[3 * v + k] - q[k]);
                }
                if (d2 > thickness * thickness) continue;
                if (pass == 0) {
                    if (bt < 0 || d2 < best) { best = d2; bt = t; }
                } else if (d2 <= best + 1e-10 * thickness * thickness) {
                    bt = t;
                    bb[0] = br[0]; bb[1] = br[1]; bb[2] = br[2];
                    break;
                }
            }
        if (bt >= 0) {
            const int32_t *tv = tri + 3 * bt;
            double u[3], w[3], nrm[3], s;
            int k;
            for (k = 0; k < 3; ++k) {
                u[k] = y[3 * tv[1] + k] - y[3 * tv[0] + k];
                w[k] = y[3 * tv[2] + k] - y[3 * tv[0] + k];
            }
            cross3(u, w, nrm);
            s = norm3(nrm);
            for (k = 0; k < 3; ++k) {
                tri_out[3 * v + k] = tv[k];
                bary_out[3 * v + k] = bb[k];
                normal_out[3 * v + k] = s > 0.0 ? nrm[k] / s : 0.0;
            }
            ++found;
        }
    }
    free(tri); free(tri_tet); free(body); free(on_surf);
    return found;
}

/* K = k_n n n^T + k_tau (I - n n^T) of a contact weak constraint (k_tau = 0 for collisions),
 * as the six entries xx, yy, zz, xy, yz, xz */
void orc_contact_stiffness(const double *n, double kn, double kt, double *K6) {
    K6[0] = kn * n[0] * n[0] + kt * (1.0 - n[0] * n[0]);
    K6[1] = kn * n[1] * n[1] + kt * (1.0 - n[1] * n[1]);
    K6[2] = kn * n[2] * n[2] + kt * (1.0 - n[2] * n[2]);
    K6[3] = (kn - kt) * n[0] * n[1];
    K6[4] = (kn - kt) * n[1] * n[2];
    K6[5] = (kn - kt) * n[0] * n[2];
}

/* Replace the colouring (e.g. by orc_recolor_incremental's); sweeps then visit these colours in ascending
 * order.  Returns ORC_E_ARG for a negative colour. */
/* threads used by the OpenMP build (n > 0 sets the count); the serial build always reports 1 */
int orc_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
    return omp_get_max_threads();
#else
    (void)n;
    return 1;
#endif
}

int orc_set_colours(orc_prep *p, const int32_t *colour) {
    int64_t v;
    int32_t m = 0;
    for (v = 0; v < p->nv; ++v) {
        if (colour[v] < 0) return ORC_E_ARG;
        if (colour[v] + 1 > m) m = colour[v] + 1;
    }
    memcpy(p->colour, colour, (size_t)p->nv * sizeof(int32_t));
    p->ncolours = m;
    return ORC_OK;
}
