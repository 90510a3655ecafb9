// pbng_kernels.cu -- sm_100a kernels of the PBNG hot path (arXiv 2306.09021).
//
//  sweep_kernel        one colour of one PBNG iteration: every free vertex of
//                      the colour accumulates f_i + f^ext_i and the SPD modified Hessian A (eq:mod_hess)
//                      over its incident tets and weak constraints, solves the 3x3 system in registers
//                      and takes one Newton step; the SOR / Chebyshev blend is fused
//                      into the same store.  One thread per vertex, one warp per 32-vertex SELL chunk:
//                      record k of the 32 lanes is one contiguous 512 B (f32) line per field.
//  energy_kernel       per-tet energy sum V_e Psi(F_e) - x.f^ext and weak-constraint energy, fp64 math,
//                      fixed-order block partials (deterministic).
//  residual_kernel     ||f_i + f^ext_i|| over free vertices from the same pair records, fp64 math.
//  reduce_kernel       per-sample final reduction of the partials.
//  set/get_positions   original <-> internal (colour-major) vertex order.
// No tensor cores: the path is a gather + 3x3 register math, not a dense contraction.
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>
#include <atomic>
#include <tuple>

#include "pbng_internal.h"

// PBNG_DEBUG=1 builds (tools/build_variants.py dbg=PBNG_DEBUG=1) check every record slot and gathered
// vertex index against the context's bounds with device asserts (the pool refuses compute-sanitizer)
#ifndef PBNG_DEBUG
#define PBNG_DEBUG 0
#endif
#if PBNG_DEBUG
#include <cassert>
#define PBNG_CHECK(c) assert(c)
#else
#define PBNG_CHECK(c) ((void)0)
#endif

namespace pbng {
namespace {

template <class R> struct RT;
template <> struct RT<float> { using R4 = float4; using RC = float; };
template <> struct RT<double> { using R4 = double4; using RC = double2; };

__device__ __forceinline__ float ld(const float *p) { return __ldg(p); }
__device__ __forceinline__ double ld(const double *p) { return __ldg(p); }
__device__ __forceinline__ int ld(const int *p) { return __ldg(p); }
__device__ __forceinline__ int64_t ld(const int64_t *p) {
    return (int64_t)__ldg(reinterpret_cast<const long long *>(p));
}
__device__ __forceinline__ int4 ld(const int4 *p) { return __ldg(p); }
__device__ __forceinline__ int2 ld(const int2 *p) { return __ldg(p); }
__device__ __forceinline__ float4 ld(const float4 *p) { return __ldg(p); }
__device__ __forceinline__ float2 ld(const float2 *p) { return __ldg(p); }
__device__ __forceinline__ double2 ld(const double2 *p) { return __ldg(p); }
__device__ __forceinline__ double4 ld(const double4 *p) {
    const double2 *q = reinterpret_cast<const double2 *>(p);
    const double2 a = __ldg(q), b = __ldg(q + 1);
    return make_double4(a.x, a.y, b.x, b.y);
}

// neighbour-position gathers: read-only path inside one colour launch (the neighbours belong to other
// colours), coherent loads in the pipelined kernel (positions written by other CTAs of the same launch)
enum { GATHER_NC = 0, GATHER_COHERENT = 1 };
template <int G, class R4> __device__ __forceinline__ R4 gather(const R4 *p) {
    if (G == GATHER_NC) return ld(p);
    return *p;
}

__device__ __forceinline__ float rsq(float x) { return rsqrtf(x); }
// the fp32 Jacobi rotation does not need IEEE-rounded sqrt / division (the angle only has to zero the
// off-diagonal to working accuracy): MUFU-based approximations; fp64 keeps the exact operations
__device__ __forceinline__ float sqrt_fast(float x) { return x > 0.f ? x * rsqrtf(x) : 0.f; }
__device__ __forceinline__ double sqrt_fast(double x) { return sqrt(x); }
__device__ __forceinline__ float div_fast(float a, float b) { return __fdividef(a, b); }
__device__ __forceinline__ double div_fast(double a, double b) { return a / b; }
__device__ __forceinline__ double rsq(double x) { return rsqrt(x); }

template <class R> __device__ __forceinline__ typename RT<R>::R4 mk4(R x, R y, R z);
template <> __device__ __forceinline__ float4 mk4<float>(float x, float y, float z) { return make_float4(x, y, z, 0.f); }
template <> __device__ __forceinline__ double4 mk4<double>(double x, double y, double z) { return make_double4(x, y, z, 0.0); }

// element index of (sample b, vertex v): samples grouped by 2^sh lanes, sample-minor inside a group
// (sh = 0: [n_batch][x_stride]; sh = 5: [n_batch/32][x_stride][32])
__device__ __forceinline__ int64_t pos_index(int64_t b, int64_t v, int64_t xs, int sh) {
    return (((b >> sh) * xs + v) << sh) + (b & ((1 << sh) - 1));
}
// sh = 6 (fp32 Neo-Hookean batches, sweep_batched2_kernel): [n_batch/64][x_stride][32 lanes][8 floats];
// lane l of group pair gp holds samples 64 gp + l (q = 0) and 64 gp + 32 + l (q = 1) component-
// interleaved as {x0 x1 y0 y1 z0 z1 0 0}, so that one 16 B + one 8 B load give the packed FP32x2
// operands of both samples.  Float index of sample b's x at vertex v (y at +2, z at +4):
__device__ __forceinline__ int64_t pos6_elem(int64_t b, int64_t v, int64_t xs) {
    return (((((b >> 6) * xs + v) << 5) + (b & 31)) << 3) + ((b >> 5) & 1);
}
// position of (sample b, vertex v) in a position-layout buffer, any layout (the w slot reads as 0)
template <class R>
__device__ __forceinline__ typename RT<R>::R4 pos_load(const void *buf, int64_t b, int64_t v, int64_t xs, int sh) {
    if (sh == 6) {
        const R *q = reinterpret_cast<const R *>(buf) + pos6_elem(b, v, xs);
        return mk4<R>(q[0], q[2], q[4]);
    }
    return reinterpret_cast<const typename RT<R>::R4 *>(buf)[pos_index(b, v, xs, sh)];
}
template <class R>
__device__ __forceinline__ void pos_store(void *buf, int64_t b, int64_t v, int64_t xs, int sh,
                                          const typename RT<R>::R4 &x) {
    if (sh == 6) {
        R *q = reinterpret_cast<R *>(buf) + pos6_elem(b, v, xs);
        q[0] = x.x; q[2] = x.y; q[4] = x.z;
        return;
    }
    reinterpret_cast<typename RT<R>::R4 *>(buf)[pos_index(b, v, xs, sh)] = x;
}


// packed FP32x2 arithmetic (sm_100 FFMA2 / FADD2 / FMUL2: two fp32 operations per lane per instruction,
// each rounded as the scalar operation)
__device__ __forceinline__ float2 bc(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 ng(float2 a) { return make_float2(-a.x, -a.y); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __fadd2_rn(a, ng(b)); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }

// ------------------------------------------------------------------------------------------------
// Polar rotation R(F) (eq:cor): closest rotation, det R = +1 also for inverted F.
// Cyclic Jacobi on S = F^T F (fixed sweep count) -> V; B = F V with columns sorted by decreasing norm
// (each swap negates one column so det V stays +1); Givens QR of B -> Q (a rotation, the sign of
// det F lands in the last diagonal entry); R = Q V^T.
// ------------------------------------------------------------------------------------------------
#ifndef PBNG_POLAR_SWEEPS_F32
#define PBNG_POLAR_SWEEPS_F32 4
#endif
template <class R> struct PolarSweeps { static constexpr int n = PBNG_POLAR_SWEEPS_F32; };
template <> struct PolarSweeps<double> { static constexpr int n = 7; };

template <int p, int q, class R>
__device__ __forceinline__ void jacobi_rot(R (&S)[3][3], R (&V)[3][3]) {
    constexpr int r = 3 - p - q;
    const R apq = S[p][q];
    const R d = S[q][q] - S[p][p];
    // t = tan(phi) = sign(d) 2 apq / (|d| + sqrt(d^2 + 4 apq^2)), the smaller root (stable)
    const R den = fabs(d) + sqrt_fast(d * d + R(4) * apq * apq);
    R t = den > R(0) ? div_fast(R(2) * apq, den) : R(0);
    t = d < R(0) ? -t : t;
    const R c = rsq(R(1) + t * t);
    const R s = t * c;
    S[p][p] -= t * apq;
    S[q][q] += t * apq;
    S[p][q] = S[q][p] = R(0);
    const R srp = S[r][p], srq = S[r][q];
    S[r][p] = S[p][r] = c * srp - s * srq;
    S[r][q] = S[q][r] = s * srp + c * srq;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const R vkp = V[k][p], vkq = V[k][q];
        V[k][p] = c * vkp - s * vkq;
        V[k][q] = s * vkp + c * vkq;
    }
}

template <int i, int j, class R>
__device__ __forceinline__ void sort_swap(R (&B)[3][3], R (&V)[3][3], R (&n)[3]) {
    const bool sw = n[i] < n[j];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const R bi = B[k][i], bj = B[k][j], vi = V[k][i], vj = V[k][j];
        B[k][i] = sw ? bj : bi;
        B[k][j] = sw ? -bi : bj;
        V[k][i] = sw ? vj : vi;
        V[k][j] = sw ? -vi : vj;
    }
    const R ni = n[i], nj = n[j];
    n[i] = sw ? nj : ni;
    n[j] = sw ? ni : nj;
}

template <class R>
__device__ __forceinline__ void givens(R a, R b, R &c, R &s) {
    const R n2 = a * a + b * b;
    const bool ok = n2 > R(0);
    const R inv = ok ? rsq(n2) : R(0);
    c = ok ? a * inv : R(1);
    s = b * inv;
}

template <int r0, int r1, int c0, class R>
__device__ __forceinline__ void rot_rows(R (&M)[3][3], R c, R s) {
#pragma unroll
    for (int k = c0; k < 3; ++k) {
        const R a = M[r0][k], b = M[r1][k];
        M[r0][k] = c * a + s * b;
        M[r1][k] = -s * a + c * b;
    }
}

template <class R>
__device__ __forceinline__ void polar_rotation(const R (&F)[3][3], R (&Rm)[3][3]) {
    R S[3][3], V[3][3], B[3][3], Qt[3][3], n[3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = a; b < 3; ++b) {
            S[a][b] = F[0][a] * F[0][b] + F[1][a] * F[1][b] + F[2][a] * F[2][b];
            S[b][a] = S[a][b];
        }
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) V[a][b] = Qt[a][b] = (a == b) ? R(1) : R(0);
#pragma unroll
    for (int it = 0; it < PolarSweeps<R>::n; ++it) {
        jacobi_rot<0, 1>(S, V);
        jacobi_rot<0, 2>(S, V);
        jacobi_rot<1, 2>(S, V);
    }
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k) B[i][k] = F[i][0] * V[0][k] + F[i][1] * V[1][k] + F[i][2] * V[2][k];
#pragma unroll
    for (int k = 0; k < 3; ++k) n[k] = B[0][k] * B[0][k] + B[1][k] * B[1][k] + B[2][k] * B[2][k];
    sort_swap<0, 1>(B, V, n);
    sort_swap<0, 2>(B, V, n);
    sort_swap<1, 2>(B, V, n);
    R c, s;
    givens(B[0][0], B[1][0], c, s);
    rot_rows<0, 1, 0>(B, c, s);
    rot_rows<0, 1, 0>(Qt, c, s);
    givens(B[0][0], B[2][0], c, s);
    rot_rows<0, 2, 0>(B, c, s);
    rot_rows<0, 2, 0>(Qt, c, s);
    givens(B[1][1], B[2][1], c, s);
    rot_rows<1, 2, 0>(Qt, c, s);
    // R = Q V^T, Q = Qt^T
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) Rm[i][j] = Qt[0][i] * V[j][0] + Qt[1][i] * V[j][1] + Qt[2][i] * V[j][2];
}

// Scaled Newton iteration for the polar factor (fp32 fast path of the fixed-corotated sweep):
// X_{k+1} = (g X_k + X_k^{-T} / g) / 2 with g = |det X_k|^{-1/3} and X^{-T} = cof(X) / det X, from
// X_0 = F (cofactor C and J = det F already computed by the caller).  For det F > 0 it converges to the
// orthogonal polar factor, which then is the closest rotation (det +1) of reading Z4; 6 iterations reach
// fp32 accuracy for condition numbers up to ~1e3.  The caller routes inverted and nearly
// singular F (det F <= 1e-4 |F|^3) to the Jacobi routine.
#ifndef PBNG_NEWTON_ITERS
#define PBNG_NEWTON_ITERS 6
#endif
template <class R>
__device__ __forceinline__ void polar_newton(const R (&F)[3][3], const R (&C0)[3][3], R J0, R (&X)[3][3]) {
    R C[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            X[a][b] = F[a][b];
            C[a][b] = C0[a][b];
        }
    R d = J0;
#pragma unroll
    for (int it = 0; it < PBNG_NEWTON_ITERS; ++it) {
        // g = |det X|^{-1/3} (det X > 0 along the iteration); MUFU approximations suffice for a scaling
        float lg, g;
        asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg) : "f"(float(d)));
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(g) : "f"(-0.33333334f * lg));
        const R hx = R(0.5) * R(g), hc = div_fast(R(0.5), R(g) * d);
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) X[a][b] = hx * X[a][b] + hc * C[a][b];
        if (it + 1 < PBNG_NEWTON_ITERS) {
            C[0][0] = X[1][1] * X[2][2] - X[1][2] * X[2][1];
            C[0][1] = X[1][2] * X[2][0] - X[1][0] * X[2][2];
            C[0][2] = X[1][0] * X[2][1] - X[1][1] * X[2][0];
            C[1][0] = X[0][2] * X[2][1] - X[0][1] * X[2][2];
            C[1][1] = X[0][0] * X[2][2] - X[0][2] * X[2][0];
            C[1][2] = X[0][1] * X[2][0] - X[0][0] * X[2][1];
            C[2][0] = X[0][1] * X[1][2] - X[0][2] * X[1][1];
            C[2][1] = X[0][2] * X[1][0] - X[0][0] * X[1][2];
            C[2][2] = X[0][0] * X[1][1] - X[0][1] * X[1][0];
            d = X[0][0] * C[0][0] + X[0][1] * C[0][1] + X[0][2] * C[0][2];
        }
    }
}

#ifndef PBNG_FCR_PACKED
#define PBNG_FCR_PACKED 1
#endif
// fp32 overload: the X update runs in packed FP32x2 on X and cof(X) held as register pairs (element
// 3a + b in pair (3a + b) / 2); the cofactor itself stays scalar.  Same iteration as the template.
__device__ __forceinline__ void polar_newton(const float (&F)[3][3], const float (&C0)[3][3], float J0,
                                             float (&Xo)[3][3]) {
    if (!PBNG_FCR_PACKED) {
        polar_newton<float>(F, C0, J0, Xo);
        return;
    }
    float2 X[5], C[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int e0 = 2 * k, e1 = 2 * k + 1;
        X[k] = make_float2(F[e0 / 3][e0 % 3], e1 < 9 ? F[e1 / 3][e1 % 3] : 0.f);
        C[k] = make_float2(C0[e0 / 3][e0 % 3], e1 < 9 ? C0[e1 / 3][e1 % 3] : 0.f);
    }
#define PX(e) (((e) & 1) ? X[(e) >> 1].y : X[(e) >> 1].x)
    float d = J0;
#pragma unroll
    for (int it = 0; it < PBNG_NEWTON_ITERS; ++it) {
        float lg, g;
        asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg) : "f"(d));
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(g) : "f"(-0.33333334f * lg));
        const float2 hx = bc(0.5f * g), hc = bc(__fdividef(0.5f, g * d));
#pragma unroll
        for (int k = 0; k < 5; ++k) X[k] = fma2(hc, C[k], mul2(hx, X[k]));
        if (it + 1 < PBNG_NEWTON_ITERS) {
            const float c00 = PX(4) * PX(8) - PX(5) * PX(7), c01 = PX(5) * PX(6) - PX(3) * PX(8),
                        c02 = PX(3) * PX(7) - PX(4) * PX(6), c10 = PX(2) * PX(7) - PX(1) * PX(8),
                        c11 = PX(0) * PX(8) - PX(2) * PX(6), c12 = PX(1) * PX(6) - PX(0) * PX(7),
                        c20 = PX(1) * PX(5) - PX(2) * PX(4), c21 = PX(2) * PX(3) - PX(0) * PX(5),
                        c22 = PX(0) * PX(4) - PX(1) * PX(3);
            C[0] = make_float2(c00, c01);
            C[1] = make_float2(c02, c10);
            C[2] = make_float2(c11, c12);
            C[3] = make_float2(c20, c21);
            C[4] = make_float2(c22, 0.f);
            d = PX(0) * c00 + PX(1) * c01 + PX(2) * c02;
        }
    }
#pragma unroll
    for (int e = 0; e < 9; ++e) Xo[e / 3][e % 3] = PX(e);
#undef PX
}

// R(F) as the fixed-corotated sweep computes it: fp32 -> scaled Newton when det F > 1e-4 |F|_F^3, else the
// Jacobi routine; fp64 -> Jacobi (7 sweeps).  C = cof F and J = det F are passed in.
template <class R>
__device__ __forceinline__ void polar_fcr(const R (&F)[3][3], const R (&C)[3][3], R J, R (&Rm)[3][3]) {
#ifdef PBNG_POLAR_F64  // experiment: the fp32 path with an fp64 polar factor (isolates the polar's share of fp32 drift)
    if (sizeof(R) == 4) {
        double Fd[3][3], Rd[3][3];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) Fd[a][b] = double(F[a][b]);
        polar_rotation(Fd, Rd);
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) Rm[a][b] = R(Rd[a][b]);
        return;
    }
#endif
    if (sizeof(R) == 4) {
        R fro = R(0);
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) fro += F[a][b] * F[a][b];
        if (J > R(1e-4) * fro * sqrt_fast(fro)) {
            polar_newton(F, C, J, Rm);
            return;
        }
    }
    polar_rotation(F, Rm);
}

// ------------------------------------------------------------------------------------------------
// Per (vertex, tet) contribution: F = sum_j (x_j - x_i) g_j^T, C = cof F,
//   f -= V P(F) g_i,   A += V (2 mu |g_i|^2 I + lambda (C g_i)(C g_i)^T).
// NH: V P g = Vmu F g + (Vlamhat (J - 1) - Vmu) C g (eq:nh, lamhat = mu + lambda).
// FCR: V P g = 2 Vmu (F g - R g) + Vlam (J - 1) C g (eq:cor).
// A is kept as {00, 11, 22, 01, 12, 02}.
// ------------------------------------------------------------------------------------------------
template <int MODEL, bool HESS, class T>
__device__ __forceinline__ void pair_contrib(const T (&d1)[3], const T (&d2)[3], const T (&d3)[3],
                                             const T (&g1)[3], const T (&g2)[3], const T (&g3)[3], T Vmu, T Vlam,
                                             T (&f)[3], T (&A)[6]) {
    T F[3][3];
    if constexpr (sizeof(T) == 4 && PBNG_FCR_PACKED) {  // columns 0, 1 of F in packed FP32x2
        const float2 g1p = make_float2(g1[0], g1[1]), g2p = make_float2(g2[0], g2[1]), g3p = make_float2(g3[0], g3[1]);
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            const float2 fr = fma2(bc(d3[r]), g3p, fma2(bc(d2[r]), g2p, mul2(bc(d1[r]), g1p)));
            F[r][0] = fr.x;
            F[r][1] = fr.y;
            F[r][2] = d1[r] * g1[2] + d2[r] * g2[2] + d3[r] * g3[2];
        }
    } else {
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c) F[r][c] = d1[r] * g1[c] + d2[r] * g2[c] + d3[r] * g3[c];
    }
    const T g[3] = {-(g1[0] + g2[0] + g3[0]), -(g1[1] + g2[1] + g3[1]), -(g1[2] + g2[2] + g3[2])};
    T C[3][3];
    C[0][0] = F[1][1] * F[2][2] - F[1][2] * F[2][1];
    C[0][1] = F[1][2] * F[2][0] - F[1][0] * F[2][2];
    C[0][2] = F[1][0] * F[2][1] - F[1][1] * F[2][0];
    C[1][0] = F[0][2] * F[2][1] - F[0][1] * F[2][2];
    C[1][1] = F[0][0] * F[2][2] - F[0][2] * F[2][0];
    C[1][2] = F[0][1] * F[2][0] - F[0][0] * F[2][1];
    C[2][0] = F[0][1] * F[1][2] - F[0][2] * F[1][1];
    C[2][1] = F[0][2] * F[1][0] - F[0][0] * F[1][2];
    C[2][2] = F[0][0] * F[1][1] - F[0][1] * F[1][0];
    const T J = F[0][0] * C[0][0] + F[0][1] * C[0][1] + F[0][2] * C[0][2];
    T Fg[3], w[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        Fg[r] = F[r][0] * g[0] + F[r][1] * g[1] + F[r][2] * g[2];
        w[r] = C[r][0] * g[0] + C[r][1] * g[1] + C[r][2] * g[2];
    }
    if (MODEL == MODEL_NH) {
        const T s = (Vmu + Vlam) * (J - T(1)) - Vmu;
#pragma unroll
        for (int r = 0; r < 3; ++r) f[r] -= Vmu * Fg[r] + s * w[r];
    } else if (MODEL == MODEL_SNH) {
        // eq:snh with mu_s = 4 mu/3, lambda_s = lambda + 5 mu/6, alpha = 1 + 3 mu_s/(4 lambda_s) (reading
        // Z18): V P g = V mu_s (1 - 1/(1 + |F|^2)) F g + V lambda_s (J - alpha) cof(F) g
        T ic = T(0);
#pragma unroll
        for (int r = 0; r < 3; ++r) ic += F[r][0] * F[r][0] + F[r][1] * F[r][1] + F[r][2] * F[r][2];
        const T Vms = T(4) / T(3) * Vmu, Vls = Vlam + T(5) / T(6) * Vmu;
        const T alpha = T(1) + div_fast(T(3) * Vms, T(4) * Vls);
        const T a = Vms * (T(1) - div_fast(T(1), T(1) + ic)), b = Vls * (J - alpha);
#pragma unroll
        for (int r = 0; r < 3; ++r) f[r] -= a * Fg[r] + b * w[r];
    } else {
        T Rm[3][3];
        polar_fcr(F, C, J, Rm);
        const T s = Vlam * (J - T(1));
        const T m2 = T(2) * Vmu;
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            const T Rg = Rm[r][0] * g[0] + Rm[r][1] * g[1] + Rm[r][2] * g[2];
            f[r] -= m2 * (Fg[r] - Rg) + s * w[r];
        }
    }
    if (HESS) {
        const T dg = T(2) * Vmu * (g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
        A[0] += dg + Vlam * w[0] * w[0];
        A[1] += dg + Vlam * w[1] * w[1];
        A[2] += dg + Vlam * w[2] * w[2];
        A[3] += Vlam * w[0] * w[1];
        A[4] += Vlam * w[1] * w[2];
        A[5] += Vlam * w[0] * w[2];
    }
}

// streamed (read-once) record loads: L1::no_allocate keeps L1 for the neighbour-position gathers
#ifndef PBNG_REC_HINT
#define PBNG_REC_HINT 1
#endif
__device__ __forceinline__ int4 lds(const int4 *p) {
#if PBNG_REC_HINT
    int4 r;
    asm("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
#else
    return __ldg(p);
#endif
}
__device__ __forceinline__ float4 lds(const float4 *p) {
#if PBNG_REC_HINT
    float4 r;
    asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
#else
    return __ldg(p);
#endif
}
__device__ __forceinline__ float lds(const float *p) {
#if PBNG_REC_HINT
    float r;
    asm("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(p));
    return r;
#else
    return __ldg(p);
#endif
}
__device__ __forceinline__ double2 lds(const double2 *p) {
#if PBNG_REC_HINT
    double2 r;
    asm("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
#else
    return __ldg(p);
#endif
}
__device__ __forceinline__ int2 lds(const int2 *p) {
#if PBNG_REC_HINT
    int2 r;
    asm("ld.global.nc.L1::no_allocate.v2.s32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
    return r;
#else
    return __ldg(p);
#endif
}
__device__ __forceinline__ double4 lds(const double4 *p) {
    const double2 *q = reinterpret_cast<const double2 *>(p);
    const double2 a = lds(q), b = lds(q + 1);
    return make_double4(a.x, a.y, b.x, b.y);
}

// record field decode
template <class R> struct Rec;
template <> struct Rec<float> {
    // shared by the 32 lanes of a warp (batched kernel): cached broadcast loads
    static __device__ __forceinline__ void load_shared(const Layout &L, int64_t r, int4 &id, float (&g1)[3],
                                                       float (&g2)[3], float (&g3)[3], float &VE) {
        id = ld(L.rec_id + r);
        const float4 a = ld(reinterpret_cast<const float4 *>(L.rec_a) + r);
        const float4 b = ld(reinterpret_cast<const float4 *>(L.rec_b) + r);
        const float c = ld(reinterpret_cast<const float *>(L.rec_c) + r);
        g1[0] = a.x; g1[1] = a.y; g1[2] = a.z;
        g2[0] = a.w; g2[1] = b.x; g2[2] = b.y;
        g3[0] = b.z; g3[1] = b.w; g3[2] = c;
        VE = __int_as_float(id.w);
    }
    static __device__ __forceinline__ void load(const Layout &L, int64_t r, int4 &id, float (&g1)[3], float (&g2)[3],
                                                float (&g3)[3], float &VE) {
        id = lds(L.rec_id + r);
        const float4 a = lds(reinterpret_cast<const float4 *>(L.rec_a) + r);
        const float4 b = lds(reinterpret_cast<const float4 *>(L.rec_b) + r);
        const float c = lds(reinterpret_cast<const float *>(L.rec_c) + r);
        g1[0] = a.x; g1[1] = a.y; g1[2] = a.z;
        g2[0] = a.w; g2[1] = b.x; g2[2] = b.y;
        g3[0] = b.z; g3[1] = b.w; g3[2] = c;
        VE = __int_as_float(id.w);
    }
};
template <> struct Rec<double> {
    static __device__ __forceinline__ void load_shared(const Layout &L, int64_t r, int4 &id, double (&g1)[3],
                                                       double (&g2)[3], double (&g3)[3], double &VE) {
        id = ld(L.rec_id + r);
        const double4 a = ld(reinterpret_cast<const double4 *>(L.rec_a) + r);
        const double4 b = ld(reinterpret_cast<const double4 *>(L.rec_b) + r);
        const double2 c = ld(reinterpret_cast<const double2 *>(L.rec_c) + r);
        g1[0] = a.x; g1[1] = a.y; g1[2] = a.z;
        g2[0] = a.w; g2[1] = b.x; g2[2] = b.y;
        g3[0] = b.z; g3[1] = b.w; g3[2] = c.x;
        VE = c.y;
    }
    static __device__ __forceinline__ void load(const Layout &L, int64_t r, int4 &id, double (&g1)[3], double (&g2)[3],
                                                double (&g3)[3], double &VE) {
        id = lds(L.rec_id + r);
        const double4 a = lds(reinterpret_cast<const double4 *>(L.rec_a) + r);
        const double4 b = lds(reinterpret_cast<const double4 *>(L.rec_b) + r);
        const double2 c = lds(reinterpret_cast<const double2 *>(L.rec_c) + r);
        g1[0] = a.x; g1[1] = a.y; g1[2] = a.z;
        g2[0] = a.w; g2[1] = b.x; g2[2] = b.y;
        g3[0] = b.z; g3[1] = b.w; g3[2] = c.x;
        VE = c.y;
    }
};

// ------------------------------------------------------------------------------------------------
// Pair records decoded in registers.  Fixed-corotated needs F itself (for R(F)), so its record carries
// the three shape-function gradients g_j.  Neo-Hookean only needs F g_i, cof(F) g_i and det F.  With
// F = Ds B (Ds = [d_1 d_2 d_3], d_j = x_j - x_i, B = Dm^{-1} with rows g_j, g_i = -(g_1 + g_2 + g_3)):
//   F g_i = sum_j s_j d_j  with s_j = g_j . g_i,
//   cof(F) g_i = cof(Ds) cof(B) g_i = cof(Ds) Dm^T g_i / det Dm = -det B (c_1 + c_2 + c_3)
//     (g_i . D_k = -1 because B Dm = I), where c_1 + c_2 + c_3 = d_2 x d_3 + d_3 x d_1 + d_1 x d_2
//     = (d_2 - d_1) x (d_3 - d_1) =: n, the deformed face normal opposite vertex i,
//   det F = det Ds det B = (d_1 . n) det B,   |g_i|^2 = -(s_1 + s_2 + s_3),
// so its record carries s_1, s_2, s_3 and det B (precomputed in fp64): 32 B per pair in fp32 instead of
// 52 B, and about 60 instead of 110 flops per pair.
// ------------------------------------------------------------------------------------------------
template <class R, int MODEL> struct Pair;
template <class R> struct PairG {  // gradient record (FCR, SNH)
    int4 id;
    R g1[3], g2[3], g3[3], VE;
};
template <class R> struct Pair<R, MODEL_FCR> : PairG<R> {};
template <class R> struct Pair<R, MODEL_SNH> : PairG<R> {};
template <class R> struct Pair<R, MODEL_NH> {
    int4 id;
    R s[3], detB, VE;
};

__device__ __forceinline__ void check_ids(const Layout &L, int64_t r, const int4 &id) {
    PBNG_CHECK(r >= 0 && r < L.n_slots);
    PBNG_CHECK(id.x >= 0 && id.x < L.n_vertices && id.y >= 0 && id.y < L.n_vertices && id.z >= 0 &&
               id.z < L.n_vertices);
}

// STREAM: read-once record (L1::no_allocate); otherwise cached (the batched kernel's broadcast loads)
template <bool STREAM, class R>
__device__ __forceinline__ void load_pair(const Layout &L, int64_t r, PairG<R> &p) {
    if (STREAM) Rec<R>::load(L, r, p.id, p.g1, p.g2, p.g3, p.VE);
    else Rec<R>::load_shared(L, r, p.id, p.g1, p.g2, p.g3, p.VE);
    check_ids(L, r, p.id);
}
template <bool STREAM>
__device__ __forceinline__ void load_pair(const Layout &L, int64_t r, Pair<float, MODEL_NH> &p) {
    const float4 *a = reinterpret_cast<const float4 *>(L.rec_a) + r;
    const int4 id = STREAM ? lds(L.rec_id + r) : ld(L.rec_id + r);
    const float4 x = STREAM ? lds(a) : ld(a);
    p.id = id;
    p.s[0] = x.x; p.s[1] = x.y; p.s[2] = x.z; p.detB = x.w;
    p.VE = __int_as_float(id.w);
    check_ids(L, r, p.id);
}
template <bool STREAM>
__device__ __forceinline__ void load_pair(const Layout &L, int64_t r, Pair<double, MODEL_NH> &p) {
    const double4 *a = reinterpret_cast<const double4 *>(L.rec_a) + r;
    const double *c = reinterpret_cast<const double *>(L.rec_c) + r;
    p.id = STREAM ? lds(L.rec_id + r) : ld(L.rec_id + r);
    const double4 x = STREAM ? lds(a) : ld(a);
    p.s[0] = x.x; p.s[1] = x.y; p.s[2] = x.z; p.detB = x.w;
    p.VE = ld(c);
    check_ids(L, r, p.id);
}

// L2 prefetch of a later record of the stream (no registers held while it is in flight)
__device__ __forceinline__ void pf_l2(const void *p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
__device__ __forceinline__ void pf_l1(const void *p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }
// ------------------------------------------------------------------------------------------------
// Path records (Problem::path, Neo-Hookean; host: vertex_path_records).  A vertex's records follow paths
// in the dual graph of its link, so consecutive records share two of their three neighbours.  The kernels
// keep three position slots and each record pushes ONE new neighbour:
//     drop 2: S2 <- S1;   drop >= 1: S1 <- S0;   S0 <- x_new      (drop = the slot whose content leaves)
// and (d_1, d_2, d_3) = (S0, S1, S2) - x_i with the record's s'_0..2 and det B' in that slot order.  A
// relabelling pi of the three neighbours flips n = (d_2 - d_1) x (d_3 - d_1) by sgn(pi) and leaves
// d_j . n unchanged, so det B' = sgn(pi) det B keeps J and cof(F) g_i exact.  Before record 0 the slots
// S1, S2 hold path0[v].  Load-only records (VE = 0, zero s' and det B') start further paths and add
// exactly 0.  fp32: rec_id = int2 {id | drop << 30, VE bits}, rec_a float4 {s'_0 s'_1 s'_2 det B'} = 24 B;
// fp64: int2 {id | drop << 30, 0}, double4, rec_c VE = 48 B.
// ------------------------------------------------------------------------------------------------
// TAB (table records, Problem::path_mode 3): rec_a holds the mesh's DISTINCT {s'_0..2, det B'} tuples and
// bits 22..29 of the record's code index them (ids < 2^22); the code returned has those bits cleared.
template <bool STREAM, bool TAB = false>
__device__ __forceinline__ int load_path_rec(const Layout &L, int64_t r, Pair<float, MODEL_NH> &p) {
    const int2 *ip = reinterpret_cast<const int2 *>(L.rec_id) + r;
    const int2 id = STREAM ? lds(ip) : ld(ip);
    const float4 x = TAB ? ld(reinterpret_cast<const float4 *>(L.rec_a) + (((unsigned)id.x >> 22) & 0xffu))
                         : STREAM ? lds(reinterpret_cast<const float4 *>(L.rec_a) + r)
                                  : ld(reinterpret_cast<const float4 *>(L.rec_a) + r);
    p.s[0] = x.x; p.s[1] = x.y; p.s[2] = x.z; p.detB = x.w;
    p.VE = __int_as_float(id.y);
    const int code = TAB ? (int)((unsigned)id.x & ~(0xffu << 22)) : id.x;
    PBNG_CHECK(r >= 0 && r < L.n_slots && (code & 0x3fffffff) < L.n_vertices);
    return code;
}
template <bool STREAM, bool TAB = false>
__device__ __forceinline__ int load_path_rec(const Layout &L, int64_t r, Pair<double, MODEL_NH> &p) {
    const int2 *ip = reinterpret_cast<const int2 *>(L.rec_id) + r;
    const int2 id = STREAM ? lds(ip) : ld(ip);
    const double4 x = TAB ? ld(reinterpret_cast<const double4 *>(L.rec_a) + (((unsigned)id.x >> 22) & 0xffu))
                          : STREAM ? lds(reinterpret_cast<const double4 *>(L.rec_a) + r)
                                   : ld(reinterpret_cast<const double4 *>(L.rec_a) + r);
    p.s[0] = x.x; p.s[1] = x.y; p.s[2] = x.z; p.detB = x.w;
    p.VE = ld(reinterpret_cast<const double *>(L.rec_c) + r);
    const int code = TAB ? (int)((unsigned)id.x & ~(0xffu << 22)) : id.x;
    PBNG_CHECK(r >= 0 && r < L.n_slots && (code & 0x3fffffff) < L.n_vertices);
    return code;
}
// table records in groups of kRecGroup (RG = 4) slots per lane (pbng_host.cpp group_table_records): the first
// slot of lane `lane`'s group g is chunk_off + g * 32 RG + RG lane = base + (RG - 1) lane + g * 32 RG with
// base = chunk_off + lane (chunk_off is a multiple of 32 RG).  One group = RG/2 16-byte loads of
// {code, VE bits} pairs (fp32; fp64 VE: RG/4 more 32-byte loads from rec_c).
constexpr int RG = kRecGroup;
__device__ __forceinline__ int64_t group_base(int64_t base) { return base + (RG - 1) * (base & 31); }
template <class R> struct RecGroup {
    int code[RG];
    R VE[RG];
};
__device__ __forceinline__ void load_group(const Layout &L, int64_t r, RecGroup<float> &g) {
    const int4 *p = reinterpret_cast<const int4 *>(reinterpret_cast<const int2 *>(L.rec_id) + r);
#pragma unroll
    for (int h = 0; h < RG / 2; ++h) {
        const int4 a = lds(p + h);
        g.code[2 * h] = a.x; g.code[2 * h + 1] = a.z;
        g.VE[2 * h] = __int_as_float(a.y); g.VE[2 * h + 1] = __int_as_float(a.w);
    }
    PBNG_CHECK(r >= 0 && r + RG - 1 < L.n_slots && (r % RG) == 0);
}
__device__ __forceinline__ void load_group(const Layout &L, int64_t r, RecGroup<double> &g) {
    const int4 *p = reinterpret_cast<const int4 *>(reinterpret_cast<const int2 *>(L.rec_id) + r);
#pragma unroll
    for (int h = 0; h < RG / 2; ++h) {
        const int4 a = lds(p + h);
        g.code[2 * h] = a.x; g.code[2 * h + 1] = a.z;
    }
#pragma unroll
    for (int h = 0; h < RG / 4; ++h) {
        const double4 v = lds(reinterpret_cast<const double4 *>(L.rec_c) + (r >> 2) + h);
        g.VE[4 * h] = v.x; g.VE[4 * h + 1] = v.y; g.VE[4 * h + 2] = v.z; g.VE[4 * h + 3] = v.w;
    }
    PBNG_CHECK(r >= 0 && r + RG - 1 < L.n_slots && (r % RG) == 0);
}
// the table entry {s'_0..2, det B'} of a table-record code; returns the code without the entry bits
template <class R>
__device__ __forceinline__ int table_pair(const Layout &L, const int code, const R VE, Pair<R, MODEL_NH> &p) {
    const typename RT<R>::R4 x = ld(reinterpret_cast<const typename RT<R>::R4 *>(L.rec_a) + (((unsigned)code >> 22) & 0xffu));
    p.s[0] = x.x; p.s[1] = x.y; p.s[2] = x.z; p.detB = x.w;
    p.VE = VE;
    return (int)((unsigned)code & ~(0xffu << 22));
}
template <class R>
__device__ __forceinline__ int table_pair_smem(const typename RT<R>::R4 *stab, const int code, const R VE,
                                               Pair<R, MODEL_NH> &p) {
    const typename RT<R>::R4 x = stab[((unsigned)code >> 22) & 0xffu];
    p.s[0] = x.x; p.s[1] = x.y; p.s[2] = x.z; p.detB = x.w;
    p.VE = VE;
    return (int)((unsigned)code & ~(0xffu << 22));
}

template <class T>
__device__ __forceinline__ void path_push(T &S0, T &S1, T &S2, const T &nw, const int code) {
    const int drop = (int)((unsigned)code >> 30);
    S2 = drop == 2 ? S1 : S2;
    S1 = drop >= 1 ? S0 : S1;
    S0 = nw;
}
template <class R>
__device__ __forceinline__ void prefetch_path(const Layout &L, int64_t r) {
    pf_l2(reinterpret_cast<const int2 *>(L.rec_id) + r);
    pf_l2(reinterpret_cast<const typename RT<R>::R4 *>(L.rec_a) + r);
}

// ------------------------------------------------------------------------------------------------
// Rest-recompute path records (Problem::rest, pbng_set_records; SURVEY.md §8(d) lower-byte variant (i)).
// A record keeps only the new neighbour {id | drop << 30} and E_e/6 (fp32: rec_id.y bits, 8 B; fp64: rec_c,
// 16 B); the rest data is rebuilt from three REST slots T_0..2 pushed exactly like the position slots,
// from the rest positions X, in slot order:
//   a_k = X_{T_k} - X_i,  Dm' = [a_0 a_1 a_2],  c_0 = a_1 x a_2, c_1 = a_2 x a_0, c_2 = a_0 x a_1,
//   det Dm' = a_0 . c_0;  the rows of B' = Dm'^{-1} are g_k = c_k / det Dm', and g_i = -(g_0 + g_1 + g_2)
//   = -N / det Dm' with N = c_0 + c_1 + c_2, so
//   s'_k = g_k . g_i = -(c_k . N) / det^2,   det B' = 1 / det Dm',   V_e E_e = |det Dm'| E_e / 6.
// These are the stored record's quantities by definition (the slot relabelling is built in), computed in
// the compute dtype instead of fp64.  Load-only records (E_e/6 = 0) take 1/det := 0 and so contribute
// exactly 0 whatever their slots hold.
// ------------------------------------------------------------------------------------------------
template <bool STREAM>
__device__ __forceinline__ int load_rest_rec(const Layout &L, int64_t r, float &E6) {
    const int2 *ip = reinterpret_cast<const int2 *>(L.rec_id) + r;
    const int2 id = STREAM ? lds(ip) : ld(ip);
    E6 = __int_as_float(id.y);
    PBNG_CHECK(r >= 0 && r < L.n_slots && (id.x & 0x3fffffff) < L.n_vertices);
    return id.x;
}
template <bool STREAM>
__device__ __forceinline__ int load_rest_rec(const Layout &L, int64_t r, double &E6) {
    const int2 *ip = reinterpret_cast<const int2 *>(L.rec_id) + r;
    const int2 id = STREAM ? lds(ip) : ld(ip);
    E6 = ld(reinterpret_cast<const double *>(L.rec_c) + r);
    PBNG_CHECK(r >= 0 && r < L.n_slots && (id.x & 0x3fffffff) < L.n_vertices);
    return id.x;
}
template <class R>
__device__ __forceinline__ typename RT<R>::R4 rest_at(const Layout &L, int i) {
    return ld(reinterpret_cast<const typename RT<R>::R4 *>(L.rest) + i);
}
template <class R, class R4>
__device__ __forceinline__ void rest_pair(const R4 &T0, const R4 &T1, const R4 &T2, const R (&Xi)[3], const R E6,
                                          Pair<R, MODEL_NH> &p) {
    const R a0[3] = {T0.x - Xi[0], T0.y - Xi[1], T0.z - Xi[2]};
    const R a1[3] = {T1.x - Xi[0], T1.y - Xi[1], T1.z - Xi[2]};
    const R a2[3] = {T2.x - Xi[0], T2.y - Xi[1], T2.z - Xi[2]};
    const R c0[3] = {a1[1] * a2[2] - a1[2] * a2[1], a1[2] * a2[0] - a1[0] * a2[2], a1[0] * a2[1] - a1[1] * a2[0]};
    const R c1[3] = {a2[1] * a0[2] - a2[2] * a0[1], a2[2] * a0[0] - a2[0] * a0[2], a2[0] * a0[1] - a2[1] * a0[0]};
    const R c2[3] = {a0[1] * a1[2] - a0[2] * a1[1], a0[2] * a1[0] - a0[0] * a1[2], a0[0] * a1[1] - a0[1] * a1[0]};
    const R det = a0[0] * c0[0] + a0[1] * c0[1] + a0[2] * c0[2];
    const R N[3] = {c0[0] + c1[0] + c2[0], c0[1] + c1[1] + c2[1], c0[2] + c1[2] + c2[2]};
    const R inv = E6 != R(0) ? R(1) / det : R(0);
    const R q = -inv * inv;
    p.s[0] = q * (c0[0] * N[0] + c0[1] * N[1] + c0[2] * N[2]);
    p.s[1] = q * (c1[0] * N[0] + c1[1] * N[1] + c1[2] * N[2]);
    p.s[2] = q * (c2[0] * N[0] + c2[1] * N[1] + c2[2] * N[2]);
    p.detB = inv;
    p.VE = E6 * fabs(det);
}

template <class R, int MODEL>
__device__ __forceinline__ void prefetch_pair(const Layout &L, int64_t r) {
    pf_l2(L.rec_id + r);
    pf_l2(reinterpret_cast<const typename RT<R>::R4 *>(L.rec_a) + r);
    if (MODEL != MODEL_NH) pf_l2(reinterpret_cast<const typename RT<R>::R4 *>(L.rec_b) + r);
}

// byte sizes of the record fields per slot (field 0 = rec_id, 1 = rec_a, 2 = rec_b, 3 = rec_c) and their
// offsets inside a shared-memory stage holding one record step of 32 lanes
template <class R, int MODEL> struct RecFmt {
    static constexpr bool nh = MODEL == MODEL_NH;
    static constexpr int s0 = 16, s1 = 4 * (int)sizeof(R), s2 = nh ? 0 : 4 * (int)sizeof(R),
                         s3 = nh ? (sizeof(R) == 8 ? 8 : 0) : (sizeof(R) == 8 ? 16 : 4);
    static __host__ __device__ constexpr int size(int k) { return k == 0 ? s0 : k == 1 ? s1 : k == 2 ? s2 : s3; }
    static __host__ __device__ constexpr int off(int k) {
        return k == 0 ? 0 : k == 1 ? 32 * s0 : k == 2 ? 32 * (s0 + s1) : 32 * (s0 + s1 + s2);
    }
    static constexpr int stage_bytes = 32 * (s0 + s1 + s2 + s3);
};
template <class R, int MODEL> __device__ __forceinline__ const void *rec_field(const Layout &L, int k) {
    return k == 0 ? static_cast<const void *>(L.rec_id) : k == 1 ? L.rec_a : k == 2 ? L.rec_b : L.rec_c;
}
// a record from a shared-memory group of kg record steps: step j, lane `lane` (plain loads)
__device__ __forceinline__ void decode_stage(const unsigned char *g, int kg, int j, int lane, Pair<float, MODEL_NH> &p) {
    using F = RecFmt<float, MODEL_NH>;
    const int e = j * 32 + lane;
    p.id = reinterpret_cast<const int4 *>(g)[e];
    const float4 x = reinterpret_cast<const float4 *>(g + kg * F::off(1))[e];
    p.s[0] = x.x; p.s[1] = x.y; p.s[2] = x.z; p.detB = x.w;
    p.VE = __int_as_float(p.id.w);
}
__device__ __forceinline__ void decode_stage(const unsigned char *g, int kg, int j, int lane, Pair<double, MODEL_NH> &p) {
    using F = RecFmt<double, MODEL_NH>;
    const int e = j * 32 + lane;
    p.id = reinterpret_cast<const int4 *>(g)[e];
    const double4 x = reinterpret_cast<const double4 *>(g + kg * F::off(1))[e];
    p.s[0] = x.x; p.s[1] = x.y; p.s[2] = x.z; p.detB = x.w;
    p.VE = reinterpret_cast<const double *>(g + kg * F::off(3))[e];
}
__device__ __forceinline__ void decode_stage(const unsigned char *g, int kg, int j, int lane, PairG<float> &p) {
    using F = RecFmt<float, MODEL_FCR>;
    const int e = j * 32 + lane;
    p.id = reinterpret_cast<const int4 *>(g)[e];
    const float4 a = reinterpret_cast<const float4 *>(g + kg * F::off(1))[e];
    const float4 b = reinterpret_cast<const float4 *>(g + kg * F::off(2))[e];
    const float c = reinterpret_cast<const float *>(g + kg * F::off(3))[e];
    p.g1[0] = a.x; p.g1[1] = a.y; p.g1[2] = a.z;
    p.g2[0] = a.w; p.g2[1] = b.x; p.g2[2] = b.y;
    p.g3[0] = b.z; p.g3[1] = b.w; p.g3[2] = c;
    p.VE = __int_as_float(p.id.w);
}
__device__ __forceinline__ void decode_stage(const unsigned char *g, int kg, int j, int lane, PairG<double> &p) {
    using F = RecFmt<double, MODEL_FCR>;
    const int e = j * 32 + lane;
    p.id = reinterpret_cast<const int4 *>(g)[e];
    const double4 a = reinterpret_cast<const double4 *>(g + kg * F::off(1))[e];
    const double4 b = reinterpret_cast<const double4 *>(g + kg * F::off(2))[e];
    const double2 c = reinterpret_cast<const double2 *>(g + kg * F::off(3))[e];
    p.g1[0] = a.x; p.g1[1] = a.y; p.g1[2] = a.z;
    p.g2[0] = a.w; p.g2[1] = b.x; p.g2[2] = b.y;
    p.g3[0] = b.z; p.g3[1] = b.w; p.g3[2] = c.x;
    p.VE = c.y;
}

// TMA (bulk copy) + mbarrier primitives for the record ring of sweep_kernel
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
    uint32_t ok;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(bar), "r"(phase)
            : "memory");
    } while (!ok);
}
__device__ __forceinline__ uint64_t l2_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// global -> shared bulk copy completing on `bar`; the record stream is read once: evict-first in L2
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(pol)
        : "memory");
}

template <bool HESS, class T, class R>
__device__ __forceinline__ void contrib(const T (&d1)[3], const T (&d2)[3], const T (&d3)[3],
                                        const Pair<R, MODEL_FCR> &p, T cmu, T clam, T (&f)[3], T (&A)[6]) {
    const T g1[3] = {T(p.g1[0]), T(p.g1[1]), T(p.g1[2])}, g2[3] = {T(p.g2[0]), T(p.g2[1]), T(p.g2[2])},
            g3[3] = {T(p.g3[0]), T(p.g3[1]), T(p.g3[2])};
    pair_contrib<MODEL_FCR, HESS>(d1, d2, d3, g1, g2, g3, T(p.VE) * cmu, T(p.VE) * clam, f, A);
}

template <bool HESS, class T, class R>
__device__ __forceinline__ void contrib(const T (&d1)[3], const T (&d2)[3], const T (&d3)[3],
                                        const Pair<R, MODEL_SNH> &p, T cmu, T clam, T (&f)[3], T (&A)[6]) {
    const T g1[3] = {T(p.g1[0]), T(p.g1[1]), T(p.g1[2])}, g2[3] = {T(p.g2[0]), T(p.g2[1]), T(p.g2[2])},
            g3[3] = {T(p.g3[0]), T(p.g3[1]), T(p.g3[2])};
    pair_contrib<MODEL_SNH, HESS>(d1, d2, d3, g1, g2, g3, T(p.VE) * cmu, T(p.VE) * clam, f, A);
}

template <bool HESS, class T, class R>
__device__ __forceinline__ void contrib(const T (&d1)[3], const T (&d2)[3], const T (&d3)[3],
                                        const Pair<R, MODEL_NH> &p, T cmu, T clam, T (&f)[3], T (&A)[6]) {
    // n = (d_2 - d_1) x (d_3 - d_1) = sum of the columns of cof(Ds)
    const T e1[3] = {d2[0] - d1[0], d2[1] - d1[1], d2[2] - d1[2]};
    const T e2[3] = {d3[0] - d1[0], d3[1] - d1[1], d3[2] - d1[2]};
    const T n[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]};
    const T detB = T(p.detB);
    const T J = (d1[0] * n[0] + d1[1] * n[1] + d1[2] * n[2]) * detB;
    const T s0 = T(p.s[0]), s1 = T(p.s[1]), s2 = T(p.s[2]);
    const T Vmu = T(p.VE) * cmu, Vlam = T(p.VE) * clam;
    const T sc = (Vmu + Vlam) * (J - T(1)) - Vmu;  // lamhat (J - 1) - mu, times V (eq:nh)
    T w[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        w[r] = -detB * n[r];                                           // cof(F) g_i
        const T Fg = s0 * d1[r] + s1 * d2[r] + s2 * d3[r];             // F g_i
        f[r] -= Vmu * Fg + sc * w[r];
    }
    if (HESS) {
        const T dg = T(-2) * Vmu * (s0 + s1 + s2);                     // 2 mu V |g_i|^2
        A[0] += dg + Vlam * w[0] * w[0];
        A[1] += dg + Vlam * w[1] * w[1];
        A[2] += dg + Vlam * w[2] * w[2];
        A[3] += Vlam * w[0] * w[1];
        A[4] += Vlam * w[1] * w[2];
        A[5] += Vlam * w[0] * w[2];
    }
}

// backward Euler (eq:fem_be): the node's inertia m_i/(2 dt^2)|y_i - xtilde_i|^2 adds
// -m_i/dt^2 (y_i - xtilde_i) to f and m_i/dt^2 I to A.  `xt` = xtilde at this vertex's element index.
template <class R, class T>
__device__ __forceinline__ void inertia_contrib(const Layout &L, int v, const typename RT<R>::R4 &xt, T idt2,
                                                const T (&xa)[3], T (&f)[3], T (&A)[6]) {
    const T m = T(ld(reinterpret_cast<const R *>(L.mass) + v)) * idt2;
    f[0] -= m * (xa[0] - T(xt.x));
    f[1] -= m * (xa[1] - T(xt.y));
    f[2] -= m * (xa[2] - T(xt.z));
    A[0] += m;
    A[1] += m;
    A[2] += m;
}

// weak-constraint terms for vertex v: f -= d K C_c, A += d^2 K
// (gat(node) returns another node's position)
template <class R, class T, bool HESS, class Gat>
__device__ __forceinline__ void wc_terms(const Layout &L, const Gat &gat, int v, const T (&xa)[3], T (&f)[3],
                                         T (&A)[6]) {
    using R4 = typename RT<R>::R4;
    const int e0 = ld(L.wc_off + v), e1 = ld(L.wc_off + v + 1);
    for (int e = e0; e < e1; ++e) {
        const int cid = ld(L.wc_cid + e);
        const T d = T(ld(reinterpret_cast<const R *>(L.wc_d) + e));
        const R4 an = ld(reinterpret_cast<const R4 *>(L.c_anchor) + cid);
        T C[3] = {-T(an.x), -T(an.y), -T(an.z)};
        const int nn = ld(L.c_n + cid);
        for (int q = 0; q < nn; ++q) {
            const int node = ld(L.c_node + kWcMaxNodes * cid + q);
            const T w = T(ld(reinterpret_cast<const R *>(L.c_w) + kWcMaxNodes * cid + q));
            if (node == v) {
                C[0] += w * xa[0]; C[1] += w * xa[1]; C[2] += w * xa[2];
            } else {
                const R4 y = gat(node);
                C[0] += w * T(y.x); C[1] += w * T(y.y); C[2] += w * T(y.z);
            }
        }
        const R *Kp = reinterpret_cast<const R *>(L.c_K) + kWcMaxNodes * cid;
        const T kxx = T(ld(Kp + 0)), kyy = T(ld(Kp + 1)), kzz = T(ld(Kp + 2));
        const T kxy = T(ld(Kp + 3)), kyz = T(ld(Kp + 4)), kxz = T(ld(Kp + 5));
        f[0] -= d * (kxx * C[0] + kxy * C[1] + kxz * C[2]);
        f[1] -= d * (kxy * C[0] + kyy * C[1] + kyz * C[2]);
        f[2] -= d * (kxz * C[0] + kyz * C[1] + kzz * C[2]);
        if (HESS) {
            const T d2 = d * d;
            A[0] += d2 * kxx; A[1] += d2 * kyy; A[2] += d2 * kzz;
            A[3] += d2 * kxy; A[4] += d2 * kyz; A[5] += d2 * kxz;
        }
    }
}
template <class R, class T, bool HESS, int G = GATHER_NC>
__device__ __forceinline__ void wc_contrib(const Layout &L, const typename RT<R>::R4 *x, const int sh, int v,
                                           const T (&xa)[3], T (&f)[3], T (&A)[6]) {
    wc_terms<R, T, HESS>(L, [&](int node) { return gather<G>(x + ((int64_t)node << sh)); }, v, xa, f, A);
}
// the same terms with positions read through the layout accessor (sample b of any position layout)
template <class R, class T, bool HESS>
__device__ __forceinline__ void wc_contrib_at(const Layout &L, const void *buf, int64_t b, int64_t xs, int sh, int v,
                                              const T (&xa)[3], T (&f)[3], T (&A)[6]) {
    wc_terms<R, T, HESS>(L, [&](int node) { return pos_load<R>(buf, b, node, xs, sh); }, v, xa, f, A);
}

// ------------------------------------------------------------------------------------------------
// colour sweep
// ------------------------------------------------------------------------------------------------
template <class R>
__device__ __forceinline__ void sub3(const typename RT<R>::R4 &p, const R (&xa)[3], R (&d)[3]) {
    d[0] = p.x - xa[0];
    d[1] = p.y - xa[1];
    d[2] = p.z - xa[2];
}

// one modified-Newton step from a zero initial guess (eq:pbgn_dx): dx = A^{-1} (f_i + f^ext_i) by
// Cholesky in registers (A is SPD); then the fused acceleration blend and the stores.
template <class R, int ACCEL>
__device__ __forceinline__ void finish_vertex(const Layout &L, typename RT<R>::R4 *__restrict__ work, const int64_t xs,
                                              const int64_t v, const int oi, const int hi,
                                              const typename RT<R>::R4 &xa4, const R (&f)[3], const R (&A)[6],
                                              const R omega, const R gamma) {
    using R4 = typename RT<R>::R4;
    const R xa[3] = {xa4.x, xa4.y, xa4.z};
    const R i00 = rsq(A[0]);
    const R l10 = A[3] * i00, l20 = A[5] * i00;
    const R i11 = rsq(A[1] - l10 * l10);
    const R l21 = (A[4] - l20 * l10) * i11;
    const R i22 = rsq(A[2] - l20 * l20 - l21 * l21);
    const R z0 = f[0] * i00;
    const R z1 = (f[1] - l10 * z0) * i11;
    const R z2 = (f[2] - l20 * z0 - l21 * z1) * i22;
    const R x2 = z2 * i22;
    const R x1 = (z1 - l21 * x2) * i11;
    const R x0 = (z0 - l10 * x1 - l20 * x2) * i00;
    const R p[3] = {xa[0] + x0, xa[1] + x1, xa[2] + x2};
    if (!(isfinite(p[0]) && isfinite(p[1]) && isfinite(p[2]))) atomicOr(L.flag, 1);

    work[v] = mk4<R>(p[0], p[1], p[2]);
    if (ACCEL != ACCEL_NONE) {
        R4 *__restrict__ out = reinterpret_cast<R4 *>(L.xbuf[oi]) + xs;
        R4 *__restrict__ hist = reinterpret_cast<R4 *>(L.xbuf[hi]) + xs;
        const R4 h4 = hist[v];
        const R h[3] = {h4.x, h4.y, h4.z};
        R o[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            if (ACCEL == ACCEL_SOR)  // x^{l+1} = omega (x_PBNG - x^{l-1}) + x^{l-1}
                o[c] = omega * (p[c] - h[c]) + h[c];
            else  // x^{l+1} = omega_{l+1} (gamma (x_PBNG - x^l) + x^l - x^{l-1}) + x^{l-1}
                o[c] = omega * (gamma * (p[c] - xa[c]) + xa[c] - h[c]) + h[c];
        }
        out[v] = mk4<R>(o[0], o[1], o[2]);
        hist[v] = xa4;
    }
}

#ifndef PBNG_SWEEP_UNROLL
#define PBNG_SWEEP_UNROLL 2
#endif
constexpr int kSweepUnroll = PBNG_SWEEP_UNROLL;  // pair-loop unroll (loads of record k+1 issued early)
#ifndef PBNG_SWEEP_PREFETCH
#define PBNG_SWEEP_PREFETCH 4
#endif
constexpr int kSweepPrefetch = PBNG_SWEEP_PREFETCH;  // L2 prefetch distance of the record stream (0: off)
#ifndef PBNG_TAB_PREFETCH
#define PBNG_TAB_PREFETCH 2
#endif
#ifndef PBNG_TAB_UNROLL
#define PBNG_TAB_UNROLL 1
#endif
constexpr int kTabUnroll = PBNG_TAB_UNROLL;  // table records: unroll of the 4-record group loop
constexpr int kTabPrefetch = PBNG_TAB_PREFETCH;  // table records: L2 prefetch distance in 4-record groups (2 best, 4: +1.3%)
// table records: the group tail (slots k + q >= deg) is processed without a branch.  Those slots are padding
// {code 0, VE 0} (pbng_host.cpp group_table_records / SELL padding): V E = 0 makes Vmu = Vlam = 0, so the
// slot adds exactly zero to f and A (finite table entry, finite positions), and the pushes it makes into
// the position slots happen after the vertex's last record.
#ifndef PBNG_TAB_NOBRANCH
#define PBNG_TAB_NOBRANCH 0
#endif
constexpr bool kTabNoBranch = PBNG_TAB_NOBRANCH;
// table records: the colour-launch sweep copies the n_tab table entries into shared memory once per CTA
// (before waiting on the previous colour) and reads them with LDS instead of L1-cached LDG
#ifndef PBNG_TAB_SMEM
#define PBNG_TAB_SMEM 0
#endif
constexpr bool kTabSmem = PBNG_TAB_SMEM;
// table records: L1 prefetch of the lane's next record group (its 32-B sector) one group ahead, so the
// group load hits L1 instead of waiting on L2 (PBNG_TAB_L1PF); register double-buffering of the next
// group's record load instead (PBNG_TAB_PIPE)
#ifndef PBNG_TAB_L1PF
#define PBNG_TAB_L1PF 0
#endif
constexpr bool kTabL1Pf = PBNG_TAB_L1PF;
#ifndef PBNG_TAB_PIPE
#define PBNG_TAB_PIPE 0
#endif
constexpr bool kTabPipe = PBNG_TAB_PIPE;
#ifndef PBNG_SWEEP_MINB
#define PBNG_SWEEP_MINB 1
#endif

#ifndef PBNG_SPLIT_PREFETCH
#define PBNG_SPLIT_PREFETCH 2
#endif
#ifndef PBNG_SPLIT_UNROLL
#define PBNG_SPLIT_UNROLL 1
#endif
constexpr int kSplitPrefetch = PBNG_SPLIT_PREFETCH;  // split warps: L2 prefetch distance in own records (2: config 5 -1.5%, config 2 -3%)
constexpr int kSplitUnroll = PBNG_SPLIT_UNROLL;
// partial sums of warp `sub` of a SPLIT-warp group over records k = sub, sub + SPLIT, ... (ascending)
template <class R, int MODEL, int G, int SPLIT>
__device__ __forceinline__ void split_partial(const Layout &L, const typename RT<R>::R4 *work, const R (&xa)[3],
                                              const int64_t base, const int deg, const int sub, const R cmu,
                                              const R clam, R (&f)[3], R (&A)[6]) {
#pragma unroll kSplitUnroll
    for (int k = sub; k < deg; k += SPLIT) {
        if (kSplitPrefetch > 0 && k + SPLIT * kSplitPrefetch < deg)
            prefetch_pair<R, MODEL>(L, base + (int64_t)(k + SPLIT * kSplitPrefetch) * kChunk);
        Pair<R, MODEL> pr;
        load_pair<true>(L, base + (int64_t)k * kChunk, pr);
        R d1[3], d2[3], d3[3];
        sub3<R>(gather<G>(work + pr.id.x), xa, d1);
        sub3<R>(gather<G>(work + pr.id.y), xa, d2);
        sub3<R>(gather<G>(work + pr.id.z), xa, d3);
        contrib<true>(d1, d2, d3, pr, cmu, clam, f, A);
    }
}

// resident CTAs sweep_kernel is compiled for (PBNG_SWEEP_MINB: fp32; PBNG_SWEEP_MINB_F64: fp64)
#ifndef PBNG_SWEEP_MINB_F64
#define PBNG_SWEEP_MINB_F64 1
#endif
template <class R> struct SweepMinBlocks { static constexpr int n = sizeof(R) == 4 ? PBNG_SWEEP_MINB : PBNG_SWEEP_MINB_F64; };
// table records (8 B, no rest data streamed through L1): more resident warps pay, unlike the stored layouts
// (fp32 64 registers / 32 warps per SM measured best)
#ifndef PBNG_SWEEP_MINB_TAB
#define PBNG_SWEEP_MINB_TAB 8
#endif
#ifndef PBNG_SWEEP_MINB_TAB64
#define PBNG_SWEEP_MINB_TAB64 1
#endif
template <class R, int PATH> struct SweepMinBlocksP {
    static constexpr int n = PATH != 3 ? SweepMinBlocks<R>::n : sizeof(R) == 4 ? PBNG_SWEEP_MINB_TAB : PBNG_SWEEP_MINB_TAB64;
};

// One free vertex's PBNG update: accumulate over its records in ascending tet order,
// weak constraints, inertia, then solve + blend + store (finish_vertex).
template <class R, int MODEL, int ACCEL, bool FEXT, bool WC, int G>
__device__ __forceinline__ void update_vertex(const Layout &L, typename RT<R>::R4 *__restrict__ work, const int64_t xs,
                                              const int v, const int64_t base, const int deg, const int oi,
                                              const int hi, const R cmu, const R clam, const R omega, const R gamma,
                                              const R idt2) {
    using R4 = typename RT<R>::R4;
    const R4 xa4 = work[v];
    const R xa[3] = {xa4.x, xa4.y, xa4.z};
    R f[3] = {R(0), R(0), R(0)};
    if (FEXT) {
        const R4 fe = ld(reinterpret_cast<const R4 *>(L.fext) + v);
        f[0] = fe.x; f[1] = fe.y; f[2] = fe.z;
    }
    R A[6] = {R(0), R(0), R(0), R(0), R(0), R(0)};

#pragma unroll kSweepUnroll
    for (int k = 0; k < deg; ++k) {
        if (kSweepPrefetch > 0 && k + kSweepPrefetch < deg)
            prefetch_pair<R, MODEL>(L, base + (int64_t)(k + kSweepPrefetch) * kChunk);
        Pair<R, MODEL> pr;
        load_pair<true>(L, base + (int64_t)k * kChunk, pr);
        R d1[3], d2[3], d3[3];
        sub3<R>(gather<G>(work + pr.id.x), xa, d1);
        sub3<R>(gather<G>(work + pr.id.y), xa, d2);
        sub3<R>(gather<G>(work + pr.id.z), xa, d3);
        contrib<true>(d1, d2, d3, pr, cmu, clam, f, A);
    }
    if (WC) wc_contrib<R, R, true, G>(L, work, 0, v, xa, f, A);
    if (idt2 > R(0)) inertia_contrib<R, R>(L, v, ld(reinterpret_cast<const R4 *>(L.xtilde) + xs + v), idt2, xa, f, A);
    finish_vertex<R, ACCEL>(L, work, xs, v, oi, hi, xa4, f, A, omega, gamma);
}

// update_vertex for path records (Neo-Hookean, Problem::path): one neighbour gather per record
// (MODE 1: stored records; 2: rest-recompute records, one more gather of the neighbour's rest position per
// record; 3: table records, the rest data read from the small table of distinct tuples)
template <class R, int ACCEL, bool FEXT, bool WC, int G, int MODE = 1, bool TS = false>
__device__ __forceinline__ void update_vertex_path(const Layout &L, typename RT<R>::R4 *__restrict__ work,
                                                   const int64_t xs, const int v, const int64_t base, const int deg,
                                                   const int oi, const int hi, const R cmu, const R clam,
                                                   const R omega, const R gamma, const R idt2,
                                                   const typename RT<R>::R4 *stab = nullptr) {
    using R4 = typename RT<R>::R4;
    const R4 xa4 = work[v];
    const R xa[3] = {xa4.x, xa4.y, xa4.z};
    R f[3] = {R(0), R(0), R(0)};
    if (FEXT) {
        const R4 fe = ld(reinterpret_cast<const R4 *>(L.fext) + v);
        f[0] = fe.x; f[1] = fe.y; f[2] = fe.z;
    }
    R A[6] = {R(0), R(0), R(0), R(0), R(0), R(0)};
    const int2 p0 = ld(L.path0 + v);
    // difference slots: S_k holds d = x_k - x_i, computed once when the neighbour is pushed (the same
    // subtraction the contribution would repeat for every record that keeps the neighbour: bitwise equal)
    auto dif = [&](const R4 &q) { return mk4<R>(q.x - xa[0], q.y - xa[1], q.z - xa[2]); };
    R4 S0 = mk4<R>(R(0), R(0), R(0)), S1 = dif(gather<G>(work + p0.x)), S2 = dif(gather<G>(work + p0.y));
    constexpr bool REST = MODE == 2;
    R4 T0, T1, T2;  // REST: the slots' rest positions
    R Xi[3];
    if constexpr (REST) {
        T0 = rest_at<R>(L, v);
        T1 = rest_at<R>(L, p0.x);
        T2 = rest_at<R>(L, p0.y);
        Xi[0] = T0.x; Xi[1] = T0.y; Xi[2] = T0.z;
    }
    if constexpr (MODE == 3) {
        // table records: RG records per step, their RG neighbour gathers issued together
        const int64_t b4 = group_base(base);
        RecGroup<R> gn;
        if (kTabPipe && deg > 0) load_group(L, b4, gn);
#pragma unroll kTabUnroll
        for (int k = 0; k < deg; k += RG) {
            if (kTabPrefetch > 0 && k + RG * kTabPrefetch < deg)
                pf_l2(reinterpret_cast<const int2 *>(L.rec_id) + b4 + (int64_t)(k + RG * kTabPrefetch) * kChunk);
            if (kTabL1Pf && k + RG < deg) pf_l1(reinterpret_cast<const int2 *>(L.rec_id) + b4 + (int64_t)(k + RG) * kChunk);
            RecGroup<R> g;
            if (kTabPipe) {
                g = gn;
                if (k + RG < deg) load_group(L, b4 + (int64_t)(k + RG) * kChunk, gn);
            } else {
                load_group(L, b4 + (int64_t)k * kChunk, g);
            }
            R4 nw[RG];
#pragma unroll
            for (int q = 0; q < RG; ++q) nw[q] = gather<G>(work + (g.code[q] & 0x3fffff));
#pragma unroll
            for (int q = 0; q < RG; ++q) nw[q] = dif(nw[q]);
#pragma unroll
            for (int q = 0; q < RG; ++q) {
                if (kTabNoBranch || k + q < deg) {
                    Pair<R, MODEL_NH> pr;
                    const int code = TS ? table_pair_smem<R>(stab, g.code[q], g.VE[q], pr)
                                        : table_pair<R>(L, g.code[q], g.VE[q], pr);
                    PBNG_CHECK((code & 0x3fffffff) < L.n_vertices);
                    path_push(S0, S1, S2, nw[q], code);
                    const R d1[3] = {S0.x, S0.y, S0.z}, d2[3] = {S1.x, S1.y, S1.z}, d3[3] = {S2.x, S2.y, S2.z};
                    contrib<true>(d1, d2, d3, pr, cmu, clam, f, A);
                }
            }
        }
    } else {
#pragma unroll kSweepUnroll
    for (int k = 0; k < deg; ++k) {
        Pair<R, MODEL_NH> pr;
        int code;
        if constexpr (REST) {
            if (kSweepPrefetch > 0 && k + kSweepPrefetch < deg)
                pf_l2(reinterpret_cast<const int2 *>(L.rec_id) + base + (int64_t)(k + kSweepPrefetch) * kChunk);
            R E6;
            code = load_rest_rec<true>(L, base + (int64_t)k * kChunk, E6);
            const int j = code & 0x3fffffff;
            const R4 nw = dif(gather<G>(work + j)), nr = rest_at<R>(L, j);
            path_push(S0, S1, S2, nw, code);
            path_push(T0, T1, T2, nr, code);
            rest_pair<R>(T0, T1, T2, Xi, E6, pr);
        } else {
            if (kSweepPrefetch > 0 && k + kSweepPrefetch < deg) {
                if constexpr (MODE == 3) pf_l2(reinterpret_cast<const int2 *>(L.rec_id) + base + (int64_t)(k + kSweepPrefetch) * kChunk);
                else prefetch_path<R>(L, base + (int64_t)(k + kSweepPrefetch) * kChunk);
            }
            code = load_path_rec<true, MODE == 3>(L, base + (int64_t)k * kChunk, pr);
            const R4 nw = dif(gather<G>(work + (code & 0x3fffffff)));
            path_push(S0, S1, S2, nw, code);
        }
        const R d1[3] = {S0.x, S0.y, S0.z}, d2[3] = {S1.x, S1.y, S1.z}, d3[3] = {S2.x, S2.y, S2.z};
        contrib<true>(d1, d2, d3, pr, cmu, clam, f, A);
    }
    }
    if (WC) wc_contrib<R, R, true, G>(L, work, 0, v, xa, f, A);
    if (idt2 > R(0)) inertia_contrib<R, R>(L, v, ld(reinterpret_cast<const R4 *>(L.xtilde) + xs + v), idt2, xa, f, A);
    finish_vertex<R, ACCEL>(L, work, xs, v, oi, hi, xa4, f, A, omega, gamma);
}

#ifndef PBNG_SWEEP_TMA
#define PBNG_SWEEP_TMA 0
#endif
#ifndef PBNG_TMA_GROUP
#define PBNG_TMA_GROUP 2
#endif
#ifndef PBNG_TMA_GROUPS
#define PBNG_TMA_GROUPS 3
#endif
// record stream of sweep_kernel through a TMA ring (1) or register loads + L2 prefetch (0, default).
// Measured on config 3: the ring's shared memory is carved out of the L1 that
// serves the neighbour gathers, and every ring depth tried was slower (0.42-0.60 vs 0.39 ms/iteration).
constexpr bool kSweepTma = PBNG_SWEEP_TMA;
#ifndef PBNG_PDL
#define PBNG_PDL 1
#endif
constexpr bool kPdl = PBNG_PDL;
#ifndef PBNG_ONE_WAVE
#define PBNG_ONE_WAVE 1
#endif
constexpr bool kOneWave = PBNG_ONE_WAVE;  // register-capped sweep instance for colours of ~1 wave  // colour launches as programmatic dependent launches (register path)
constexpr int kGroup = PBNG_TMA_GROUP;      // record steps per bulk copy
constexpr int kGroups = PBNG_TMA_GROUPS;    // ring depth in groups
template <class R, int MODEL> struct StageSmem {  // per warp: [ring][kGroups mbarriers, padded]
    static constexpr int group_bytes = kGroup * RecFmt<R, MODEL>::stage_bytes;
    static constexpr int per_warp = kSweepTma ? kGroups * group_bytes + 128 : 0;
};

// One thread per free vertex of the colour; a warp owns one 32-vertex SELL chunk.  The chunk's record
// stream is contiguous (record step k of the 32 lanes is one run of 32 slots per field, consecutive
// steps adjacent), so lane 0 streams it into a ring of kGroups groups of kGroup steps with bulk copies
// (TMA), one mbarrier per group: HBM latency is hidden without holding registers, and the lanes only
// gather their neighbour positions (through L1; they belong to other colours, read-only in this
// launch).  The per-vertex summation order is ascending tet index, as in the oracle.
template <class R, int MODEL, int ACCEL, bool FEXT, bool WC, bool ONE_WAVE = false, int PATH = 0>
__global__ void __launch_bounds__(kSweepBlock, (ONE_WAVE ? 1024 / kSweepBlock : SweepMinBlocksP<R, PATH>::n)) sweep_kernel(const Layout L, const int32_t v_begin, const int32_t n_v,
                                                            const int64_t chunk_begin, const int64_t x_stride,
                                                            const int wi, const int oi, const int hi, const R cmu,
                                                            const R clam, const R omega, const R gamma, const R idt2) {
    using R4 = typename RT<R>::R4;
    if (!kSweepTma) {
        // programmatic dependent launch: let the next colour's CTAs start in this launch's tail; before
        // waiting for the previous colour they touch only static data (offsets, degree) and prefetch their
        // first records into L2 (the record stream does not depend on any position)
        if (kPdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        extern __shared__ __align__(128) unsigned char tsm[];
        R4 *stab = reinterpret_cast<R4 *>(tsm);
        if constexpr (PATH == 3 && kTabSmem) {  // static table: copied before the wait on the previous colour
            for (int q = threadIdx.x; q < L.n_tab; q += kSweepBlock) stab[q] = ld(reinterpret_cast<const R4 *>(L.rec_a) + q);
            __syncthreads();
        }
        const int t = blockIdx.x * kSweepBlock + threadIdx.x;
        if (t >= n_v) return;
        const int v = v_begin + t;
        const int64_t base = ld(L.chunk_off + chunk_begin + (t >> 5)) + (t & 31);
        const int deg = ld(L.deg + v);
        if (kPdl) {
            for (int k = 0; k < kSweepPrefetch && k < deg; ++k) {
                if constexpr (PATH == 3) {
                    if (k < kTabPrefetch && RG * k < deg)
                        pf_l2(reinterpret_cast<const int2 *>(L.rec_id) + group_base(base) + (int64_t)(RG * k) * kChunk);
                }
                else if constexpr (PATH == 2) pf_l2(reinterpret_cast<const int2 *>(L.rec_id) + base + (int64_t)k * kChunk);
                else if constexpr (PATH) prefetch_path<R>(L, base + (int64_t)k * kChunk);
                else prefetch_pair<R, MODEL>(L, base + (int64_t)k * kChunk);
            }
            asm volatile("griddepcontrol.wait;" ::: "memory");
        }
        const int64_t xs = (int64_t)blockIdx.y * x_stride;
        R4 *__restrict__ work = reinterpret_cast<R4 *>(L.xbuf[wi]) + xs;
        if constexpr (PATH && MODEL == MODEL_NH)
            update_vertex_path<R, ACCEL, FEXT, WC, GATHER_NC, PATH, PATH == 3 && kTabSmem>(
                L, work, xs, v, base, deg, oi, hi, cmu, clam, omega, gamma, idt2, stab);
        else
            update_vertex<R, MODEL, ACCEL, FEXT, WC, GATHER_NC>(L, work, xs, v, base, deg, oi, hi, cmu, clam, omega,
                                                                gamma, idt2);
        return;
    }
    using F = RecFmt<R, MODEL>;
    using SS = StageSmem<R, MODEL>;
    extern __shared__ __align__(128) unsigned char dsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cw = blockIdx.x * (kSweepBlock / 32) + warp;  // chunk within the colour
    if (cw * kChunk >= n_v) return;                         // warp-uniform
    unsigned char *ring = dsm + (size_t)warp * SS::per_warp;
    const uint32_t bar0 = smem_u32(ring + kGroups * SS::group_bytes);
    const int64_t ch = chunk_begin + cw;
    const int64_t r0 = ld(L.chunk_off + ch);
    const int W = (int)((ld(L.chunk_off + ch + 1) - r0) >> 5);  // records per lane incl. padding
    const int NGRP = (W + kGroup - 1) / kGroup;
    uint64_t pol = 0;
    auto issue = [&](int g) {  // lane 0: record steps [g kGroup, (g + 1) kGroup) into ring slot g % kGroups
        const int k0 = g * kGroup, n = min(kGroup, W - k0);
        const uint32_t bar = bar0 + 8 * (g % kGroups);
        const uint32_t dst = smem_u32(ring + (g % kGroups) * SS::group_bytes);
        mbar_expect_tx(bar, n * F::stage_bytes);
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (F::size(q) > 0)
                bulk_g2s(dst + kGroup * F::off(q),
                         static_cast<const char *>(rec_field<R, MODEL>(L, q)) + (r0 + (int64_t)k0 * kChunk) * F::size(q),
                         n * kChunk * F::size(q), bar, pol);
    };
    if (lane == 0) {
        for (int g = 0; g < kGroups; ++g) mbar_init(bar0 + 8 * g, 1);
        mbar_fence_init();
        pol = l2_evict_first();
        for (int g = 0; g < min(kGroups, NGRP); ++g) issue(g);
    }
    __syncwarp();
    const int t = cw * kChunk + lane;
    const bool valid = t < n_v;
    const int v = v_begin + t;
    const int64_t xs = (int64_t)blockIdx.y * x_stride;
    R4 *__restrict__ work = reinterpret_cast<R4 *>(L.xbuf[wi]) + xs;
    const R4 xa4 = valid ? work[v] : mk4<R>(R(0), R(0), R(0));
    const R xa[3] = {xa4.x, xa4.y, xa4.z};
    const int deg = valid ? ld(L.deg + v) : 0;
    R f[3] = {R(0), R(0), R(0)};
    if (FEXT && valid) {
        const R4 fe = ld(reinterpret_cast<const R4 *>(L.fext) + v);
        f[0] = fe.x; f[1] = fe.y; f[2] = fe.z;
    }
    R A[6] = {R(0), R(0), R(0), R(0), R(0), R(0)};
    for (int g = 0; g < NGRP; ++g) {
        const unsigned char *grp = ring + (g % kGroups) * SS::group_bytes;
        mbar_wait(bar0 + 8 * (g % kGroups), (g / kGroups) & 1);
        const int kd = deg - g * kGroup;
#pragma unroll
        for (int j = 0; j < kGroup; ++j) {
            if (j < kd) {
                Pair<R, MODEL> pr;
                decode_stage(grp, kGroup, j, lane, pr);
                R d1[3], d2[3], d3[3];
                sub3<R>(ld(work + pr.id.x), xa, d1);
                sub3<R>(ld(work + pr.id.y), xa, d2);
                sub3<R>(ld(work + pr.id.z), xa, d3);
                contrib<true>(d1, d2, d3, pr, cmu, clam, f, A);
            }
        }
        // group g is consumed by every lane: refill its ring slot with group g + kGroups
        __syncwarp();
        if (lane == 0 && g + kGroups < NGRP) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(g + kGroups);
        }
    }
    if (!valid) return;
    if (WC) wc_contrib<R, R, true>(L, work, 0, v, xa, f, A);
    if (idt2 > R(0)) inertia_contrib<R, R>(L, v, ld(reinterpret_cast<const R4 *>(L.xtilde) + xs + v), idt2, xa, f, A);
    finish_vertex<R, ACCEL>(L, work, xs, v, oi, hi, xa4, f, A, omega, gamma);
}

// ------------------------------------------------------------------------------------------------
// Pipelined (dataflow) sweep: ONE persistent launch runs up to kPipeMaxIter whole iterations.  Work
// items are (iteration l, chunk X, sample b) in lexicographic order -- iteration-major, then colour-
// major chunk order -- taken by warps from a global counter.  Instead of a grid-wide barrier between
// colours, a chunk waits only for the chunks holding its stencil neighbours (host-built list,
// pbng_host.cpp build_pipeline): a neighbour chunk of an EARLIER colour must have finished iteration
// l (done >= l + 1), one of a LATER colour (and the chunk itself) iteration l - 1 (done >= l).  This
// is exactly the order the per-colour launches impose on every (reader, writer) pair of positions
// -- including the work/out buffer swap of the accelerated blends -- so every vertex reads the same
// values and the results are bitwise those of the barrier schedule.  No deadlock: an item only waits
// for items earlier in the counter order, which running warps already hold.
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ int ld_acquire(const int32_t *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_relaxed(const int32_t *p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void red_release_add(int32_t *p, int v) {
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// windowed batched schedule: relaxed polling + one acquire fence per item, release reduction (1), or
// acquire polling + __threadfence in every thread (0)
#ifndef PBNG_B2_LIGHTSYNC
#define PBNG_B2_LIGHTSYNC 1
#endif
constexpr bool kB2LightSync = PBNG_B2_LIGHTSYNC;
__device__ __forceinline__ void st_release(int32_t *p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void group_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// threads per CTA of the split and pipelined kernels: whole SPLIT-warp groups, at least kSweepBlock
template <int SPLIT> struct SplitBlock { static constexpr int n = SPLIT * 32 > kSweepBlock ? SPLIT * 32 : kSweepBlock; };
// resident CTAs the split kernel is compiled for: fp32 at 64 registers (32 warps per SM; without the hint
// ptxas picks 91 registers for the fixed-corotated kernel and config 5 runs 25% slower), fp64 unconstrained
#ifndef PBNG_SPLIT_WARPS_F32
#define PBNG_SPLIT_WARPS_F32 32
#endif
template <class R, int SPLIT> struct SplitMinBlocks {
    static constexpr int n = sizeof(R) == 4 ? PBNG_SPLIT_WARPS_F32 * 32 / SplitBlock<SPLIT>::n : 1;
};

// SPLIT warps form a group that owns one item at a time (SPLIT = 1: update_vertex, the arithmetic of
// sweep_kernel; SPLIT > 1: the partial sums and fixed-order combination of sweep_split_kernel), so the
// per-vertex summation order -- and the result -- is that of the colour-launch schedule with the same
// split (pbng_host.cpp problem_split).
template <class R, int MODEL, int ACCEL, bool FEXT, bool WC, int SPLIT, int PATH = 0>
__global__ void __launch_bounds__(SplitBlock<SPLIT>::n, (MODEL == MODEL_FCR && SPLIT == 8) ? 3 : PBNG_SWEEP_MINB)
    sweep_pipe_kernel(const Layout L, const PipeLaunch P,
                                                                 const int64_t x_stride, const int32_t n_batch,
                                                                 const int64_t n_chunks, const R cmu, const R clam,
                                                                 const R idt2) {
    using R4 = typename RT<R>::R4;
    constexpr int GROUPS = SplitBlock<SPLIT>::n / (32 * SPLIT);
    static_assert(GROUPS >= 1 && GROUPS * SPLIT * 32 == SplitBlock<SPLIT>::n, "block must hold whole groups");
    __shared__ R red[GROUPS][SPLIT > 1 ? SPLIT - 1 : 1][9][32];
    __shared__ int64_t item_sh[GROUPS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int grp = warp / SPLIT, sub = warp % SPLIT;
    const int64_t per_iter = n_chunks * n_batch;
    const int64_t n_items = per_iter * P.n_iter;
    auto gsync = [&] {
        if (SPLIT == 1) __syncwarp();
        else group_sync(1 + grp, SPLIT * 32);
    };
    for (;;) {
        if (sub == 0 && lane == 0)
            item_sh[grp] = (int64_t)atomicAdd(reinterpret_cast<unsigned long long *>(L.pipe_counter), 1ull);
        gsync();
        const int64_t q = item_sh[grp];
        if (q >= n_items) return;
        int l, b;
        int64_t X;
        if (n_items < (int64_t(1) << 31)) {  // 32-bit division (64-bit integer division is a slow subroutine)
            const uint32_t qq = (uint32_t)q, pi = (uint32_t)per_iter, nb = (uint32_t)n_batch;
            l = (int)(qq / pi);
            const uint32_t rem = qq - (uint32_t)l * pi;
            X = rem / nb;
            b = (int)(rem - (uint32_t)X * nb);
        } else {
            l = (int)(q / per_iter);
            const int64_t rem = q - (int64_t)l * per_iter;
            X = rem / n_batch;
            b = (int)(rem - X * n_batch);
        }
        int32_t *flags = L.pipe_flags + (int64_t)b * n_chunks;
        if (sub == 0) {  // wait for the neighbour chunks (one dependency per lane)
            const int d0 = ld(L.dep_off + X), d1 = ld(L.dep_off + X + 1);
            for (int d = d0 + lane; d < d1; d += 32) {
                const int dep = ld(L.deps + d);
                const int target = l + (dep & 1);
                const int32_t *fl = flags + (dep >> 1);
                while (ld_acquire(fl) < target) __nanosleep(32);
            }
        }
        gsync();
        __threadfence();
        const int wi = (ACCEL != ACCEL_NONE && (l & 1)) ? P.out : P.work;
        const int oi = (ACCEL != ACCEL_NONE && (l & 1)) ? P.work : P.out;
        const R omega = R(P.omega[l]), gamma = R(P.gamma);
        const int2 cv = ld(L.chunk_v + X);
        const bool valid = lane < cv.y;
        const int v = cv.x + lane;
        const int64_t xs = (int64_t)b * x_stride;
        R4 *__restrict__ work = reinterpret_cast<R4 *>(L.xbuf[wi]) + xs;
        const int64_t base = ld(L.chunk_off + X) + lane;
        if (SPLIT == 1) {
            if (valid) {
                if constexpr (PATH && MODEL == MODEL_NH)
                    update_vertex_path<R, ACCEL, FEXT, WC, GATHER_COHERENT, PATH>(
                        L, work, xs, v, base, ld(L.deg + v), oi, P.hist, cmu, clam, omega, gamma, idt2);
                else
                    update_vertex<R, MODEL, ACCEL, FEXT, WC, GATHER_COHERENT>(L, work, xs, v, base, ld(L.deg + v), oi,
                                                                              P.hist, cmu, clam, omega, gamma, idt2);
            }
        } else {
            R f[3] = {R(0), R(0), R(0)};
            R A[6] = {R(0), R(0), R(0), R(0), R(0), R(0)};
            R4 xa4 = mk4<R>(R(0), R(0), R(0));
            if (valid) {
                xa4 = work[v];
                const R xa[3] = {xa4.x, xa4.y, xa4.z};
                split_partial<R, MODEL, GATHER_COHERENT, SPLIT>(L, work, xa, base, ld(L.deg + v), sub, cmu, clam, f, A);
            }
            if (sub > 0) {
#pragma unroll
                for (int c = 0; c < 3; ++c) red[grp][sub - 1][c][lane] = f[c];
#pragma unroll
                for (int c = 0; c < 6; ++c) red[grp][sub - 1][3 + c][lane] = A[c];
            }
            gsync();
            if (sub == 0 && valid) {
#pragma unroll
                for (int t = 0; t < SPLIT - 1; ++t) {
#pragma unroll
                    for (int c = 0; c < 3; ++c) f[c] += red[grp][t][c][lane];
#pragma unroll
                    for (int c = 0; c < 6; ++c) A[c] += red[grp][t][3 + c][lane];
                }
                if (FEXT) {
                    const R4 fe = ld(reinterpret_cast<const R4 *>(L.fext) + v);
                    f[0] += fe.x; f[1] += fe.y; f[2] += fe.z;
                }
                const R xa[3] = {xa4.x, xa4.y, xa4.z};
                if (WC) wc_contrib<R, R, true, GATHER_COHERENT>(L, work, 0, v, xa, f, A);
                if (idt2 > R(0))
                    inertia_contrib<R, R>(L, v, ld(reinterpret_cast<const R4 *>(L.xtilde) + xs + v), idt2, xa, f, A);
                finish_vertex<R, ACCEL>(L, work, xs, v, oi, P.hist, xa4, f, A, omega, gamma);
            }
        }
        if (sub == 0) {
            __threadfence();
            __syncwarp();
            if (lane == 0) st_release(flags + X, l + 1);
        }
    }
}

// Split variant for compute-heavy pairs (fixed-corotated: a polar decomposition per pair) and small
// colours: SPLIT warps share one 32-vertex chunk, warp s takes records k = s, s + SPLIT, ...; the nine
// partial sums (f: 3, A: 6) are combined through shared memory in fixed warp order (deterministic),
// and warp 0 solves and stores.  Block = SPLIT * 32 * CPB threads, CPB chunks per block.
template <class R, int MODEL, int ACCEL, bool FEXT, bool WC, int SPLIT>
__global__ void __launch_bounds__(SplitBlock<SPLIT>::n, (SplitMinBlocks<R, SPLIT>::n)) sweep_split_kernel(const Layout L, const int32_t v_begin, const int32_t n_v,
                                                                  const int64_t chunk_begin, const int64_t x_stride,
                                                                  const int wi, const int oi, const int hi, const R cmu,
                                                                  const R clam, const R omega, const R gamma,
                                                                  const R idt2) {
    using R4 = typename RT<R>::R4;
    constexpr int CPB = SplitBlock<SPLIT>::n / (32 * SPLIT);
    static_assert(CPB >= 1 && CPB * SPLIT * 32 == SplitBlock<SPLIT>::n, "block must hold whole chunk groups");
    __shared__ R red[CPB][SPLIT - 1][9][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cl = warp / SPLIT, sub = warp % SPLIT;
    const int tc = (blockIdx.x * CPB + cl) * 32 + lane;  // vertex index within the colour
    const bool valid = tc < n_v;
    const int v = v_begin + tc;
    const int64_t xs = (int64_t)blockIdx.y * x_stride;
    R4 *__restrict__ work = reinterpret_cast<R4 *>(L.xbuf[wi]) + xs;
    R f[3] = {R(0), R(0), R(0)};
    R A[6] = {R(0), R(0), R(0), R(0), R(0), R(0)};
    R4 xa4 = mk4<R>(R(0), R(0), R(0));
    if (kPdl) {  // as sweep_kernel: static data and a record prefetch before waiting for the previous colour
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        if (valid) prefetch_pair<R, MODEL>(L, ld(L.chunk_off + chunk_begin + (tc >> 5)) + lane + (int64_t)sub * kChunk);
        asm volatile("griddepcontrol.wait;" ::: "memory");
    }
    if (valid) {
        const int64_t base = ld(L.chunk_off + chunk_begin + (tc >> 5)) + lane;
        const int deg = ld(L.deg + v);
        xa4 = work[v];
        const R xa[3] = {xa4.x, xa4.y, xa4.z};
        split_partial<R, MODEL, GATHER_NC, SPLIT>(L, work, xa, base, deg, sub, cmu, clam, f, A);
    }
    if (sub > 0) {
#pragma unroll
        for (int q = 0; q < 3; ++q) red[cl][sub - 1][q][lane] = f[q];
#pragma unroll
        for (int q = 0; q < 6; ++q) red[cl][sub - 1][3 + q][lane] = A[q];
    }
    __syncthreads();
    if (sub != 0 || !valid) return;
#pragma unroll
    for (int s = 0; s < SPLIT - 1; ++s) {
#pragma unroll
        for (int q = 0; q < 3; ++q) f[q] += red[cl][s][q][lane];
#pragma unroll
        for (int q = 0; q < 6; ++q) A[q] += red[cl][s][3 + q][lane];
    }
    if (FEXT) {
        const R4 fe = ld(reinterpret_cast<const R4 *>(L.fext) + v);
        f[0] += fe.x; f[1] += fe.y; f[2] += fe.z;
    }
    const R xa[3] = {xa4.x, xa4.y, xa4.z};
    if (WC) wc_contrib<R, R, true>(L, work, 0, v, xa, f, A);
    if (idt2 > R(0)) inertia_contrib<R, R>(L, v, ld(reinterpret_cast<const R4 *>(L.xtilde) + xs + v), idt2, xa, f, A);
    finish_vertex<R, ACCEL>(L, work, xs, v, oi, hi, xa4, f, A, omega, gamma);
}

// a pair record held by lane `src`, broadcast to the warp (32-bit words)
template <class P> __device__ __forceinline__ P shfl_pair(const P &p, int src) {
    static_assert(sizeof(P) % 4 == 0, "pair records are whole words");
    P out;
    const uint32_t *a = reinterpret_cast<const uint32_t *>(&p);
    uint32_t *o = reinterpret_cast<uint32_t *>(&out);
#pragma unroll
    for (int k = 0; k < (int)(sizeof(P) / 4); ++k) o[k] = __shfl_sync(0xffffffffu, a[k], src);
    return out;
}

// Batched samples (n_batch >= 32): positions are stored sample-minor,
// x[(group * x_stride + v) * 32 + lane] with sample = 32 * group + lane.  A warp updates ONE vertex for
// 32 samples: lane k loads the vertex's record k once (shared rest mesh), each pair's record is then a
// warp shuffle, so the neighbour gathers -- each one coalesced 512 B (f32) line -- of consecutive pairs
// are independent of any load and overlap (unrolled x4).  Same arithmetic and per-vertex order as
// sweep_kernel.
template <class R, int MODEL, int ACCEL, bool FEXT, bool WC>
__global__ void __launch_bounds__(kSweepBlock) sweep_batched_kernel(const Layout L, const int32_t v_begin,
                                                                    const int32_t n_v, const int64_t chunk_begin,
                                                                    const int64_t x_stride, const int32_t n_batch,
                                                                    const int wi, const int oi, const int hi,
                                                                    const R cmu, const R clam, const R omega,
                                                                    const R gamma, const R idt2) {
    using R4 = typename RT<R>::R4;
    constexpr int WPB = kSweepBlock / 32;
    const int lane = threadIdx.x & 31;
    const int t = blockIdx.x * WPB + (threadIdx.x >> 5);  // vertex index within the colour
    const int b = blockIdx.y * 32 + lane;                  // sample (lanes past n_batch compute, never store)
    if (t >= n_v) return;                                  // warp-uniform
    const int v = v_begin + t;
    const int64_t base = ld(L.chunk_off + chunk_begin + (t >> 5)) + (t & 31);
    const int deg = ld(L.deg + v);
    const int64_t xs = ((int64_t)blockIdx.y * x_stride << 5) + lane;  // this lane's sample offset
    R4 *__restrict__ work = reinterpret_cast<R4 *>(L.xbuf[wi]) + xs;
    const R4 xa4 = work[(int64_t)v << 5];
    const R xa[3] = {xa4.x, xa4.y, xa4.z};
    R f[3] = {R(0), R(0), R(0)};
    if (FEXT) {
        const R4 fe = ld(reinterpret_cast<const R4 *>(L.fext) + v);
        f[0] = fe.x; f[1] = fe.y; f[2] = fe.z;
    }
    R A[6] = {R(0), R(0), R(0), R(0), R(0), R(0)};
    for (int k0 = 0; k0 < deg; k0 += 32) {
        Pair<R, MODEL> mine = {};
        if (k0 + lane < deg) load_pair<false>(L, base + (int64_t)(k0 + lane) * kChunk, mine);
        const int n = min(32, deg - k0);
#pragma unroll 4
        for (int j = 0; j < n; ++j) {
            const Pair<R, MODEL> pr = shfl_pair(mine, j);
            R d1[3], d2[3], d3[3];
            sub3<R>(ld(work + ((int64_t)pr.id.x << 5)), xa, d1);
            sub3<R>(ld(work + ((int64_t)pr.id.y << 5)), xa, d2);
            sub3<R>(ld(work + ((int64_t)pr.id.z << 5)), xa, d3);
            contrib<true>(d1, d2, d3, pr, cmu, clam, f, A);
        }
    }
    if (b >= n_batch) return;
    if (WC) wc_contrib<R, R, true>(L, work, 5, v, xa, f, A);
    if (idt2 > R(0))
        inertia_contrib<R, R>(L, v, ld(reinterpret_cast<const R4 *>(L.xtilde) + xs + ((int64_t)v << 5)), idt2, xa, f, A);
    finish_vertex<R, ACCEL>(L, work, xs, (int64_t)v << 5, oi, hi, xa4, f, A, omega, gamma);
}

// ------------------------------------------------------------------------------------------------
// Batched samples, two groups per warp (fp32 Neo-Hookean, n_batch >= 64): lane holds samples
// 64 g + lane and 64 g + 32 + lane, and every pair's arithmetic runs in packed FP32x2 instructions
// (FFMA2 / FADD2 / FMUL2: two fused multiply-adds per lane per instruction on sm_100), which halves the
// issued instructions of this issue-bound kernel.  The record is shared by both samples (one shuffle).
// Same per-vertex order as sweep_kernel; the rounding of the packed expressions differs from the
// compiler's scalar contraction by an ulp per operation.
// ------------------------------------------------------------------------------------------------

// eq:nh pair term for two samples at once (see contrib<..., Pair<R, MODEL_NH>>)
__device__ __forceinline__ void contrib_nh2(const float2 (&d1)[3], const float2 (&d2)[3], const float2 (&d3)[3],
                                            const Pair<float, MODEL_NH> &p, float cmu, float clam, float2 (&f)[3],
                                            float2 (&A)[6]) {
    const float2 e1[3] = {sub2(d2[0], d1[0]), sub2(d2[1], d1[1]), sub2(d2[2], d1[2])};
    const float2 e2[3] = {sub2(d3[0], d1[0]), sub2(d3[1], d1[1]), sub2(d3[2], d1[2])};
    const float2 n[3] = {fma2(e1[1], e2[2], ng(mul2(e1[2], e2[1]))), fma2(e1[2], e2[0], ng(mul2(e1[0], e2[2]))),
                         fma2(e1[0], e2[1], ng(mul2(e1[1], e2[0])))};
    const float2 J = mul2(fma2(d1[0], n[0], fma2(d1[1], n[1], mul2(d1[2], n[2]))), bc(p.detB));
    const float Vmu = p.VE * cmu, Vlam = p.VE * clam, lh = Vmu + Vlam;
    const float2 sc = fma2(bc(lh), J, bc(-lh - Vmu));  // lamhat (J - 1) - mu, times V
    const float dg = -2.f * Vmu * (p.s[0] + p.s[1] + p.s[2]);
    float2 w[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        w[r] = mul2(bc(-p.detB), n[r]);
        const float2 Fg = fma2(bc(p.s[2]), d3[r], fma2(bc(p.s[1]), d2[r], mul2(bc(p.s[0]), d1[r])));
        f[r] = fma2(ng(sc), w[r], fma2(bc(-Vmu), Fg, f[r]));
    }
    const float2 t0 = mul2(bc(Vlam), w[0]), t1 = mul2(bc(Vlam), w[1]), t2 = mul2(bc(Vlam), w[2]);
    A[0] = fma2(t0, w[0], add2(A[0], bc(dg)));
    A[1] = fma2(t1, w[1], add2(A[1], bc(dg)));
    A[2] = fma2(t2, w[2], add2(A[2], bc(dg)));
    A[3] = fma2(t0, w[1], A[3]);
    A[4] = fma2(t1, w[2], A[4]);
    A[5] = fma2(t0, w[2], A[5]);
}

// contrib_nh2 with the record's material scalars precomputed on the host (batched sh-6 records, rec_b:
// {V mu, V lambda, V (mu + lambda), 2 V mu |g_i|^2} in fp64, rounded): the same terms without the ~10 scalar
// instructions per record that derive them from VE
__device__ __forceinline__ void contrib_nh2v(const float2 (&d1)[3], const float2 (&d2)[3], const float2 (&d3)[3],
                                             const float4 sd, const float4 vv, float2 (&f)[3], float2 (&A)[6]) {
    const float2 e1[3] = {sub2(d2[0], d1[0]), sub2(d2[1], d1[1]), sub2(d2[2], d1[2])};
    const float2 e2[3] = {sub2(d3[0], d1[0]), sub2(d3[1], d1[1]), sub2(d3[2], d1[2])};
    const float2 n[3] = {fma2(e1[1], e2[2], ng(mul2(e1[2], e2[1]))), fma2(e1[2], e2[0], ng(mul2(e1[0], e2[2]))),
                         fma2(e1[0], e2[1], ng(mul2(e1[1], e2[0])))};
    const float2 J = mul2(fma2(d1[0], n[0], fma2(d1[1], n[1], mul2(d1[2], n[2]))), bc(sd.w));
    const float Vmu = vv.x, Vlam = vv.y, lh = vv.z;
    const float2 sc = fma2(bc(lh), J, bc(-lh - Vmu));  // lamhat (J - 1) - mu, times V
    float2 w[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        w[r] = mul2(bc(-sd.w), n[r]);
        const float2 Fg = fma2(bc(sd.z), d3[r], fma2(bc(sd.y), d2[r], mul2(bc(sd.x), d1[r])));
        f[r] = fma2(ng(sc), w[r], fma2(bc(-Vmu), Fg, f[r]));
    }
    const float2 t0 = mul2(bc(Vlam), w[0]), t1 = mul2(bc(Vlam), w[1]), t2 = mul2(bc(Vlam), w[2]);
    A[0] = fma2(t0, w[0], add2(A[0], bc(vv.w)));
    A[1] = fma2(t1, w[1], add2(A[1], bc(vv.w)));
    A[2] = fma2(t2, w[2], add2(A[2], bc(vv.w)));
    A[3] = fma2(t0, w[1], A[3]);
    A[4] = fma2(t1, w[2], A[4]);
    A[5] = fma2(t0, w[2], A[5]);
}

#ifndef PBNG_B2_MINB
#define PBNG_B2_MINB 5  // 96 registers / 20 warps per SM measured best (config 4: 0.970 ms per iteration; 4: 1.158, 6: 1.068 with unroll 6)
#endif
#ifndef PBNG_B2_UNROLL
#define PBNG_B2_UNROLL 12
#endif
constexpr int kB2Unroll = PBNG_B2_UNROLL;
#ifndef PBNG_B2_PF
#define PBNG_B2_PF 0
#endif
constexpr int kB2Prefetch = PBNG_B2_PF;  // records ahead whose neighbour slot is prefetched into L1 (0: off; 4: 7% slower)
// the packed positions of a lane's two samples at one vertex (sh 6 slot {x0 x1 y0 y1 | z0 z1 . .})
struct P6 {
    float2 x, y, z;
};
template <bool COH = false>
__device__ __forceinline__ P6 ld_p6(const float *p) {
    const float4 a = COH ? *reinterpret_cast<const float4 *>(p) : ld(reinterpret_cast<const float4 *>(p));
    const float2 b = COH ? *reinterpret_cast<const float2 *>(p + 4) : ld(reinterpret_cast<const float2 *>(p + 4));
    return {make_float2(a.x, a.y), make_float2(a.z, a.w), b};
}

// dx = A^{-1} f by the same register Cholesky as finish_vertex
__device__ __forceinline__ void chol_solve3(const float (&A)[6], const float (&f)[3], float (&x)[3]) {
    const float i00 = rsq(A[0]);
    const float l10 = A[3] * i00, l20 = A[5] * i00;
    const float i11 = rsq(A[1] - l10 * l10);
    const float l21 = (A[4] - l20 * l10) * i11;
    const float i22 = rsq(A[2] - l20 * l20 - l21 * l21);
    const float z0 = f[0] * i00;
    const float z1 = (f[1] - l10 * z0) * i11;
    const float z2 = (f[2] - l20 * z0 - l21 * z1) * i22;
    x[2] = z2 * i22;
    x[1] = (z1 - l21 * x[2]) * i11;
    x[0] = (z0 - l10 * x[1] - l20 * x[2]) * i00;
}

// Position layout sh = 6 (pos6_elem): the lane's 32 B slot of vertex u in group pair gp starts at float
// ((gp * x_stride + u) << 8) + 8 lane and holds {x0 x1 y0 y1 | z0 z1 . .} -- the packed operands of its
// two samples, loaded with one LDG.128 + one LDG.64 (no repacking moves).  The warp's records are staged
// in shared memory (lane k stores record k) and read back as warp-broadcast LDS.128 pairs.
// One vertex (index t of its colour) for the 64 samples of group pair gp, by one warp (COH: positions are
// written by other CTAs of the same launch -- the windowed persistent kernel -- so they are read with
// plain loads after an acquire instead of the read-only path).
template <int ACCEL, bool FEXT, bool WC, bool COH>
__device__ __forceinline__ void b2_vertex(const Layout &L, const int t, const int32_t v_begin, const int64_t chunk_begin,
                                          const int64_t gp, const int64_t x_stride, const int32_t n_batch, const int wi,
                                          const int oi, const int hi, const float cmu, const float clam,
                                          const float omega, const float gamma, const float idt2, int2 (&s_id)[32],
                                          float4 (&s_sd)[32], float4 (&s_vv)[32]) {
    const int lane = threadIdx.x & 31;
    const int v = v_begin + t;
    const int64_t base = ld(L.chunk_off + chunk_begin + (t >> 5)) + (t & 31);
    const int deg = ld(L.deg + v);
    const int64_t slot = ((gp * x_stride) << 8) + 8 * lane;  // this lane's float offset at vertex 0
    const float *__restrict__ wk = reinterpret_cast<const float *>(L.xbuf[wi]) + slot;
    const int64_t vo = (int64_t)v << 8;
    const float4 a01 = *reinterpret_cast<const float4 *>(wk + vo);  // own row: written only by this warp
    const float2 a2 = *reinterpret_cast<const float2 *>(wk + vo + 4);
    const float2 xa[3] = {make_float2(a01.x, a01.y), make_float2(a01.z, a01.w), a2};
    float2 f[3] = {bc(0.f), bc(0.f), bc(0.f)};
    if (FEXT) {
        const float4 fe = ld(reinterpret_cast<const float4 *>(L.fext) + v);
        f[0] = bc(fe.x); f[1] = bc(fe.y); f[2] = bc(fe.z);
    }
    float2 A[6] = {bc(0.f), bc(0.f), bc(0.f), bc(0.f), bc(0.f), bc(0.f)};
    // path records (the host always orders sh-6 records along link paths): three slots of packed
    // positions {x, y, z} x 2 samples; each record gathers one new neighbour (one LDG.128 + one LDG.64)
    // the slots hold the differences d = x_j - x_i (computed once when a neighbour is pushed)
    P6 S0, S1, S2;
    auto diff = [&](const P6 &q) { return P6{sub2(q.x, xa[0]), sub2(q.y, xa[1]), sub2(q.z, xa[2])}; };
    {
        const int2 p0 = ld(L.path0 + v);
        S0 = {bc(0.f), bc(0.f), bc(0.f)};
        S1 = diff(ld_p6<COH>(wk + ((int64_t)p0.x << 8)));
        S2 = diff(ld_p6<COH>(wk + ((int64_t)p0.y << 8)));
    }
    for (int k0 = 0; k0 < deg; k0 += 32) {
        if (k0 + lane < deg) {
            const int64_t r = base + (int64_t)(k0 + lane) * kChunk;
            s_id[lane] = ld(reinterpret_cast<const int2 *>(L.rec_id) + r);
            s_sd[lane] = ld(reinterpret_cast<const float4 *>(L.rec_a) + r);
            s_vv[lane] = ld(reinterpret_cast<const float4 *>(L.rec_b) + r);
            PBNG_CHECK(r < L.n_slots && (s_id[lane].x & 0x3fffffff) < L.n_vertices);
        }
        __syncwarp();
        const int n = min(32, deg - k0);
#pragma unroll kB2Unroll
        for (int j = 0; j < n; ++j) {
            if (kB2Prefetch > 0 && j + kB2Prefetch < n)  // the gather of record j + PF: L2 -> L1 now
                pf_l1(wk + ((int64_t)(s_id[j + kB2Prefetch].x & 0x3fffffff) << 8));
            const int2 id = s_id[j];
            const P6 nw = diff(ld_p6<COH>(wk + ((int64_t)(id.x & 0x3fffffff) << 8)));
            path_push(S0, S1, S2, nw, id.x);
            const float2 d1[3] = {S0.x, S0.y, S0.z};
            const float2 d2[3] = {S1.x, S1.y, S1.z};
            const float2 d3[3] = {S2.x, S2.y, S2.z};
            contrib_nh2v(d1, d2, d3, s_sd[j], s_vv[j], f, A);
        }
        __syncwarp();
    }
    // per sample: weak constraints, inertia, solve, blend (scalar); then one interleaved store per buffer
    float p[2][3], o[2][3];
    const float *hs = reinterpret_cast<const float *>(L.xbuf[hi]) + slot + vo;
    float4 h01 = make_float4(0.f, 0.f, 0.f, 0.f);
    float2 h2 = make_float2(0.f, 0.f);
    if (ACCEL != ACCEL_NONE) {
        h01 = *reinterpret_cast<const float4 *>(hs);
        h2 = *reinterpret_cast<const float2 *>(hs + 4);
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const int64_t b = gp * 64 + q * 32 + lane;
        const float xs3[3] = {q ? xa[0].y : xa[0].x, q ? xa[1].y : xa[1].x, q ? xa[2].y : xa[2].x};
        const float h[3] = {q ? h01.y : h01.x, q ? h01.w : h01.z, q ? h2.y : h2.x};
        float fs[3], As[6];
#pragma unroll
        for (int r = 0; r < 3; ++r) fs[r] = q ? f[r].y : f[r].x;
#pragma unroll
        for (int r = 0; r < 6; ++r) As[r] = q ? A[r].y : A[r].x;
        if (b < n_batch) {
            if (WC) wc_contrib_at<float, float, true>(L, L.xbuf[wi], b, x_stride, 6, v, xs3, fs, As);
            if (idt2 > 0.f) inertia_contrib<float, float>(L, v, pos_load<float>(L.xtilde, b, v, x_stride, 6), idt2, xs3, fs, As);
            float dx[3];
            chol_solve3(As, fs, dx);
#pragma unroll
            for (int c = 0; c < 3; ++c) p[q][c] = xs3[c] + dx[c];
            if (!(isfinite(p[q][0]) && isfinite(p[q][1]) && isfinite(p[q][2]))) atomicOr(L.flag, 1);
        } else {  // padding sample: keep its (finite) values
#pragma unroll
            for (int c = 0; c < 3; ++c) p[q][c] = xs3[c];
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            if (ACCEL == ACCEL_SOR)  // x^{l+1} = omega (x_PBNG - x^{l-1}) + x^{l-1}
                o[q][c] = omega * (p[q][c] - h[c]) + h[c];
            else if (ACCEL == ACCEL_CHEB)  // x^{l+1} = omega_{l+1} (gamma (x_PBNG - x^l) + x^l - x^{l-1}) + x^{l-1}
                o[q][c] = omega * (gamma * (p[q][c] - xs3[c]) + xs3[c] - h[c]) + h[c];
        }
    }
    float *ws = reinterpret_cast<float *>(L.xbuf[wi]) + slot + vo;
    *reinterpret_cast<float4 *>(ws) = make_float4(p[0][0], p[1][0], p[0][1], p[1][1]);
    *reinterpret_cast<float2 *>(ws + 4) = make_float2(p[0][2], p[1][2]);
    if (ACCEL != ACCEL_NONE) {
        float *os = reinterpret_cast<float *>(L.xbuf[oi]) + slot + vo;
        *reinterpret_cast<float4 *>(os) = make_float4(o[0][0], o[1][0], o[0][1], o[1][1]);
        *reinterpret_cast<float2 *>(os + 4) = make_float2(o[0][2], o[1][2]);
        float *hw = reinterpret_cast<float *>(L.xbuf[hi]) + slot + vo;
        *reinterpret_cast<float4 *>(hw) = a01;
        *reinterpret_cast<float2 *>(hw + 4) = a2;
    }
}

template <int ACCEL, bool FEXT, bool WC>
__global__ void __launch_bounds__(kSweepBlock, PBNG_B2_MINB) sweep_batched2_kernel(const Layout L, const int32_t v_begin,
                                                                     const int32_t n_v, const int64_t chunk_begin,
                                                                     const int64_t x_stride, const int32_t n_batch,
                                                                     const int wi, const int oi, const int hi,
                                                                     const float cmu, const float clam,
                                                                     const float omega, const float gamma,
                                                                     const float idt2, const int reverse) {
    constexpr int WPB = kSweepBlock / 32;
    __shared__ int2 s_id[WPB][32];
    __shared__ float4 s_sd[WPB][32];
    __shared__ float4 s_vv[WPB][32];
    const int wq = threadIdx.x >> 5;
    const int t = blockIdx.x * WPB + wq;  // vertex index within the colour
    if (t >= n_v) return;                  // warp-uniform (only warp-level synchronisation below)
    const int64_t gp = reverse ? gridDim.y - 1 - blockIdx.y : blockIdx.y;
    b2_vertex<ACCEL, FEXT, WC, false>(L, t, v_begin, chunk_begin, gp, x_stride, n_batch, wi, oi, hi, cmu, clam, omega,
                                      gamma, idt2, s_id[wq], s_sd[wq], s_vv[wq]);
}

// Windowed persistent schedule for the batched fp32 Neo-Hookean layout (sh 6).  The sample-group pairs are
// independent problems, so a colour pass of one group pair needs only the previous colour pass of the SAME
// group pair.  Items (iteration, window of W group pairs, colour, group pair, block of WPB vertices) are
// taken in that order from a global counter; an item waits (acquire) until its group pair's previous colour
// pass has released all its blocks.  A window's positions (W x 3 buffers x ~5 MB) stay in L2 through its 8
// colour passes, instead of every colour launch re-reading all 4096 samples from DRAM.  Every vertex reads
// exactly what the colour launches give it -> bitwise-identical iterates.
template <int ACCEL, bool FEXT, bool WC>
__global__ void __launch_bounds__(kSweepBlock, PBNG_B2_MINB) sweep_batched2_window_kernel(
    const Layout L, const B2Window P, const int64_t x_stride, const int32_t n_batch, const float cmu, const float clam,
    const float idt2) {
    constexpr int WPB = kSweepBlock / 32;
    __shared__ int2 s_id[WPB][32];
    __shared__ float4 s_sd[WPB][32];
    __shared__ float4 s_vv[WPB][32];
    __shared__ int64_t item_sh;
    const int wq = threadIdx.x >> 5;
    const int64_t n_gp = (n_batch + 63) / 64;
    const int64_t per_gp = P.blk_off[P.ncol];  // blocks of one group pair in one iteration
    const int64_t per_iter = n_gp * per_gp;
    const int64_t n_items = per_iter * P.n_iter;
    int32_t *done = L.pipe_flags;  // [n_gp][ncol] blocks finished (all iterations of this launch)
    for (;;) {
        if (threadIdx.x == 0) item_sh = (int64_t)atomicAdd(reinterpret_cast<unsigned long long *>(L.pipe_counter), 1ull);
        __syncthreads();
        const int64_t q = item_sh;
        __syncthreads();
        if (q >= n_items) return;
        const int it = (int)(q / per_iter);
        int64_t r = q - (int64_t)it * per_iter;
        const int64_t wsz = (int64_t)P.window * per_gp;
        const int64_t w = r / wsz;
        r -= w * wsz;
        const int64_t gp0 = w * P.window;
        const int64_t W = min((int64_t)P.window, n_gp - gp0);  // group pairs in this window
        int c = 0;
        while (c + 1 < P.ncol && r >= W * P.blk_off[c + 1]) ++c;
        r -= W * P.blk_off[c];
        const int nblk = P.blk_off[c + 1] - P.blk_off[c];
        const int64_t gp = gp0 + r / nblk;
        const int blk = (int)(r % nblk);
        if (threadIdx.x == 0) {  // the group pair's previous (non-empty) colour pass, this or the previous iteration
            const int pc = P.prev[c];
            const int target = (pc < c ? it + 1 : it) * (P.blk_off[pc + 1] - P.blk_off[pc]);
            const int32_t *fl = done + gp * P.ncol + pc;
            if (kB2LightSync) {
                // relaxed polling, then ONE acquire fence: every acquire invalidates the SM's whole L1
                // (CCTL.IVALL), so acquiring per poll and fencing in every thread wiped the gathers that
                // the other resident warps had cached
                while (ld_relaxed(fl) < target) __nanosleep(32);
                fence_acq_rel_gpu();
            } else {
                while (ld_acquire(fl) < target) __nanosleep(32);
            }
        }
        __syncthreads();  // the CTA's loads below are ordered after thread 0's acquire
        if (!kB2LightSync) __threadfence();
        const int wi = (ACCEL != ACCEL_NONE && (it & 1)) ? P.out : P.work;
        const int oi = (ACCEL != ACCEL_NONE && (it & 1)) ? P.work : P.out;
#pragma unroll 1
        for (int u = 0; u < kB2WinVpw; ++u) {
            const int t = (blk * kB2WinVpw + u) * WPB + wq;
            if (t < P.n_v[c])
                b2_vertex<ACCEL, FEXT, WC, true>(L, t, P.v_begin[c], P.chunk_begin[c], gp, x_stride, n_batch, wi, oi,
                                                 P.hist, cmu, clam, float(P.omega[it]), float(P.gamma), idt2, s_id[wq],
                                                 s_sd[wq], s_vv[wq]);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            if (kB2LightSync) {
                red_release_add(done + gp * P.ncol + c, 1);  // cumulative over the CTA's stores (bar.sync above)
            } else {
                __threadfence();
                atomicAdd(done + gp * P.ncol + c, 1);
            }
        }
    }
}

#ifndef PBNG_BATCHED2
#define PBNG_BATCHED2 1
#endif

template <class R, int MODEL, int ACCEL, bool FE, bool W, int S>
cudaError_t split_launch(const Problem &p, const Layout &L, const SweepLaunch &s, cudaStream_t st) {
    constexpr int B = SplitBlock<S>::n, VPB = B / S;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)((s.n_v + VPB - 1) / VPB), (unsigned)p.n_batch);
    cfg.blockDim = dim3(B);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = kPdl ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, sweep_split_kernel<R, MODEL, ACCEL, FE, W, S>, L, s.v_begin, s.n_v,
                              s.chunk_begin, p.x_stride, s.work, s.out, s.hist, R(p.cmu), R(p.clam), R(s.omega),
                              R(s.gamma), R(p.inv_dt2));
}

template <class R, int MODEL, int ACCEL, bool FE, bool W>
cudaError_t sweep_dispatch4(const Problem &p, const Layout &L, const SweepLaunch &s, cudaStream_t st) {
    const R cmu = R(p.cmu), clam = R(p.clam), om = R(s.omega), ga = R(s.gamma), idt2 = R(p.inv_dt2);
    if constexpr (sizeof(R) == 4 && MODEL == MODEL_NH) {
      if (p.lane_shift == 6) {  // fp32 Neo-Hookean batches (the host picks sh 6)
        constexpr int WPB = kSweepBlock / 32;
        dim3 grid((unsigned)((s.n_v + WPB - 1) / WPB), (unsigned)((p.n_batch + 63) / 64));
        sweep_batched2_kernel<ACCEL, FE, W><<<grid, kSweepBlock, 0, st>>>(L, s.v_begin, s.n_v, s.chunk_begin,
                                                                          p.x_stride, p.n_batch, s.work, s.out,
                                                                          s.hist, float(cmu), float(clam), float(om),
                                                                          float(ga), float(idt2), s.reverse);
        return cudaGetLastError();
    }
    }
    if (p.lane_shift == 5) {
        constexpr int WPB = kSweepBlock / 32;
        dim3 grid((unsigned)((s.n_v + WPB - 1) / WPB), (unsigned)((p.n_batch + 31) / 32));
        sweep_batched_kernel<R, MODEL, ACCEL, FE, W><<<grid, kSweepBlock, 0, st>>>(
            L, s.v_begin, s.n_v, s.chunk_begin, p.x_stride, p.n_batch, s.work, s.out, s.hist, cmu, clam, om, ga, idt2);
        return cudaGetLastError();
    }
    if (s.split <= 1) {
        constexpr int smem = (kSweepBlock / 32) * StageSmem<R, MODEL>::per_warp;
        // function attributes are per device: one flag per ordinal (setting one twice is harmless)
        static std::atomic<bool> attr[kMaxDevices];
        if (smem > 48 * 1024 && !attr[p.device % kMaxDevices].load(std::memory_order_acquire)) {
            cudaError_t e = cudaFuncSetAttribute(sweep_kernel<R, MODEL, ACCEL, FE, W>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            if (e != cudaSuccess) return e;
            attr[p.device % kMaxDevices].store(true, std::memory_order_release);
        }
        dim3 grid((unsigned)((s.n_v + kSweepBlock - 1) / kSweepBlock), (unsigned)p.n_batch);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(kSweepBlock);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = (kPdl && !kSweepTma) ? 1 : 0;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        // a colour that fits in one wave only at full occupancy (the two small colours of config 3) runs a
        // register-capped instance so that it does not leave a second, almost empty wave
        const int sms = p.sm_count > 0 ? p.sm_count : 148;
        const int64_t blocks = (int64_t)grid.x * grid.y;
        // L1 / shared-memory split of the register path (PBNG_CARVEOUT = percent of the unified array
        // given to shared memory; unset: the driver's choice)
        static const int carve = [] {
            const char *e = getenv("PBNG_CARVEOUT");
            return e ? atoi(e) : -1;
        }();
        static std::atomic<bool> carved[kMaxDevices];
        if (!kSweepTma && carve >= 0 && !carved[p.device % kMaxDevices].load(std::memory_order_acquire)) {
            cudaFuncSetAttribute(sweep_kernel<R, MODEL, ACCEL, FE, W>, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
            cudaFuncSetAttribute(sweep_kernel<R, MODEL, ACCEL, FE, W, true>, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
            carved[p.device % kMaxDevices].store(true, std::memory_order_release);
        }
        const bool one_wave = kOneWave && sizeof(R) == 4 && !kSweepTma && blocks > (int64_t)sms * 6 &&
                              blocks <= (int64_t)sms * (1024 / kSweepBlock);
        if constexpr (MODEL == MODEL_NH) {
            if (p.path && p.path_mode == 3) {
                if (kTabSmem) cfg.dynamicSmemBytes = (size_t)L.n_tab * sizeof(typename RT<R>::R4);
                if (one_wave)
                    return cudaLaunchKernelEx(&cfg, sweep_kernel<R, MODEL, ACCEL, FE, W, true, 3>, L, s.v_begin,
                                              s.n_v, s.chunk_begin, p.x_stride, s.work, s.out, s.hist, cmu, clam, om, ga,
                                              idt2);
                return cudaLaunchKernelEx(&cfg, sweep_kernel<R, MODEL, ACCEL, FE, W, false, 3>, L, s.v_begin, s.n_v,
                                          s.chunk_begin, p.x_stride, s.work, s.out, s.hist, cmu, clam, om, ga, idt2);
            }
            if (p.path && p.path_mode == 2) {
                if (one_wave)
                    return cudaLaunchKernelEx(&cfg, sweep_kernel<R, MODEL, ACCEL, FE, W, true, 2>, L, s.v_begin,
                                              s.n_v, s.chunk_begin, p.x_stride, s.work, s.out, s.hist, cmu, clam, om, ga,
                                              idt2);
                return cudaLaunchKernelEx(&cfg, sweep_kernel<R, MODEL, ACCEL, FE, W, false, 2>, L, s.v_begin, s.n_v,
                                          s.chunk_begin, p.x_stride, s.work, s.out, s.hist, cmu, clam, om, ga, idt2);
            }
            if (p.path) {
                if (one_wave)
                    return cudaLaunchKernelEx(&cfg, sweep_kernel<R, MODEL, ACCEL, FE, W, true, 1>, L, s.v_begin,
                                              s.n_v, s.chunk_begin, p.x_stride, s.work, s.out, s.hist, cmu, clam, om, ga,
                                              idt2);
                return cudaLaunchKernelEx(&cfg, sweep_kernel<R, MODEL, ACCEL, FE, W, false, 1>, L, s.v_begin, s.n_v,
                                          s.chunk_begin, p.x_stride, s.work, s.out, s.hist, cmu, clam, om, ga, idt2);
            }
        }
        if (one_wave)
            return cudaLaunchKernelEx(&cfg, sweep_kernel<R, MODEL, ACCEL, FE, W, true>, L, s.v_begin, s.n_v,
                                      s.chunk_begin, p.x_stride, s.work, s.out, s.hist, cmu, clam, om, ga, idt2);
        return cudaLaunchKernelEx(&cfg, sweep_kernel<R, MODEL, ACCEL, FE, W>, L, s.v_begin, s.n_v, s.chunk_begin,
                                  p.x_stride, s.work, s.out, s.hist, cmu, clam, om, ga, idt2);
    }
    if (s.split == 2) return split_launch<R, MODEL, ACCEL, FE, W, 2>(p, L, s, st);
    if (s.split == 8) return split_launch<R, MODEL, ACCEL, FE, W, 8>(p, L, s, st);
    return split_launch<R, MODEL, ACCEL, FE, W, 4>(p, L, s, st);
}

// persistent grid: every SM filled to the kernel's occupancy (queried once per instantiation and device;
// racing threads compute and store the same value)
template <class R, int MODEL, int ACCEL, bool FE, bool W, int SPLIT, int PATH = 0>
cudaError_t pipe_launch(const Problem &p, const Layout &L, const PipeLaunch &s, cudaStream_t st) {
    static std::atomic<int> cache[kMaxDevices];
    int blocks = cache[p.device % kMaxDevices].load(std::memory_order_acquire);
    if (blocks == 0) {
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_pipe_kernel<R, MODEL, ACCEL, FE, W, SPLIT, PATH>,
                                                      SplitBlock<SPLIT>::n, 0);
        blocks = std::max(1, (p.sm_count > 0 ? p.sm_count : 148) * std::max(1, per_sm));
        cache[p.device % kMaxDevices].store(blocks, std::memory_order_release);
    }
    constexpr int GROUPS = SplitBlock<SPLIT>::n / (32 * SPLIT);
    const int64_t items = p.n_chunks * p.n_batch * s.n_iter;
    const int64_t g = std::min<int64_t>(blocks, (items + GROUPS - 1) / GROUPS);
    if (g <= 0) return cudaSuccess;
    sweep_pipe_kernel<R, MODEL, ACCEL, FE, W, SPLIT, PATH><<<(unsigned)g, SplitBlock<SPLIT>::n, 0, st>>>(
        L, s, p.x_stride, p.n_batch, p.n_chunks, R(p.cmu), R(p.clam), R(p.inv_dt2));
    return cudaGetLastError();
}

template <class R, int MODEL, int ACCEL, bool FE, bool W>
cudaError_t pipe_dispatch4(const Problem &p, const Layout &L, const PipeLaunch &s, cudaStream_t st) {
    if (s.split == 2) return pipe_launch<R, MODEL, ACCEL, FE, W, 2>(p, L, s, st);
    if (s.split == 4) return pipe_launch<R, MODEL, ACCEL, FE, W, 4>(p, L, s, st);
    if (s.split == 8) return pipe_launch<R, MODEL, ACCEL, FE, W, 8>(p, L, s, st);
    if constexpr (MODEL == MODEL_NH) {
        if (p.path && p.path_mode == 3) return pipe_launch<R, MODEL, ACCEL, FE, W, 1, 3>(p, L, s, st);
        if (p.path && p.path_mode == 2) return pipe_launch<R, MODEL, ACCEL, FE, W, 1, 2>(p, L, s, st);
        if (p.path) return pipe_launch<R, MODEL, ACCEL, FE, W, 1, 1>(p, L, s, st);
    }
    return pipe_launch<R, MODEL, ACCEL, FE, W, 1>(p, L, s, st);
}

template <class R, int MODEL, int ACCEL>
cudaError_t pipe_dispatch3(const Problem &p, const Layout &L, const PipeLaunch &s, cudaStream_t st) {
    if (p.has_fext) {
        if (p.has_wc) return pipe_dispatch4<R, MODEL, ACCEL, true, true>(p, L, s, st);
        return pipe_dispatch4<R, MODEL, ACCEL, true, false>(p, L, s, st);
    }
    if (p.has_wc) return pipe_dispatch4<R, MODEL, ACCEL, false, true>(p, L, s, st);
    return pipe_dispatch4<R, MODEL, ACCEL, false, false>(p, L, s, st);
}

template <class R, int MODEL>
cudaError_t pipe_dispatch2(const Problem &p, const Layout &L, const PipeLaunch &s, cudaStream_t st) {
    switch (s.accel) {
        case ACCEL_SOR: return pipe_dispatch3<R, MODEL, ACCEL_SOR>(p, L, s, st);
        case ACCEL_CHEB: return pipe_dispatch3<R, MODEL, ACCEL_CHEB>(p, L, s, st);
        default: return pipe_dispatch3<R, MODEL, ACCEL_NONE>(p, L, s, st);
    }
}

template <class R, int MODEL, int ACCEL>
cudaError_t sweep_dispatch3(const Problem &p, const Layout &L, const SweepLaunch &s, cudaStream_t st) {
    if (p.has_fext) {
        if (p.has_wc) return sweep_dispatch4<R, MODEL, ACCEL, true, true>(p, L, s, st);
        return sweep_dispatch4<R, MODEL, ACCEL, true, false>(p, L, s, st);
    }
    if (p.has_wc) return sweep_dispatch4<R, MODEL, ACCEL, false, true>(p, L, s, st);
    return sweep_dispatch4<R, MODEL, ACCEL, false, false>(p, L, s, st);
}

template <class R, int MODEL>
cudaError_t sweep_dispatch2(const Problem &p, const Layout &L, const SweepLaunch &s, cudaStream_t st) {
    switch (s.accel) {
        case ACCEL_SOR: return sweep_dispatch3<R, MODEL, ACCEL_SOR>(p, L, s, st);
        case ACCEL_CHEB: return sweep_dispatch3<R, MODEL, ACCEL_CHEB>(p, L, s, st);
        default: return sweep_dispatch3<R, MODEL, ACCEL_NONE>(p, L, s, st);
    }
}

// ------------------------------------------------------------------------------------------------
// positions: original <-> internal order
// ------------------------------------------------------------------------------------------------
template <class R>
__global__ void set_positions_kernel(const Layout L, const int64_t nv, const int64_t n_global, const int64_t n_free,
                                     const int64_t n_pin, const int64_t x_stride, const int nbuf,
                                     const int sh) {
    using R4 = typename RT<R>::R4;
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= nv) return;
    const int64_t b = blockIdx.y;
    R4 val;
    if (v < n_free || nbuf < 0) {
        const R *s = reinterpret_cast<const R *>(L.stage) + (b * n_global + L.int2orig[v]) * 3;
        val = mk4<R>(s[0], s[1], s[2]);
    } else {
        val = reinterpret_cast<const R4 *>(L.targets)[b * n_pin + (v - n_free)];
    }
    if (nbuf < 0) {  // backward-Euler inertial target xtilde (pbng_set_inertia)
        pos_store<R>(L.xtilde, b, v, x_stride, sh, val);
        return;
    }
    for (int k = 0; k < nbuf; ++k) pos_store<R>(L.xbuf[k], b, v, x_stride, sh, val);
}

template <class R>
__global__ void get_positions_kernel(const Layout L, const int64_t nv, const int64_t n_global, const int64_t x_stride,
                                     const int wi, const int sh) {
    using R4 = typename RT<R>::R4;
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= nv) return;
    const int64_t b = blockIdx.y;
    const R4 x = pos_load<R>(wi < 0 ? L.xtilde : L.xbuf[wi], b, v, x_stride, sh);  // wi < 0: the inertial target
    R *d = reinterpret_cast<R *>(L.stage) + (b * n_global + L.int2orig[v]) * 3;
    d[0] = x.x;
    d[1] = x.y;
    d[2] = x.z;
}

// halo exchange (domain decomposition): pack the listed vertices' work (, out, hist) values into a
// contiguous [n_batch][n][n_fields] Real4 buffer, or scatter such a buffer into the ghost rows
template <class R>
__global__ void halo_pack_kernel(const Layout L, const int32_t *__restrict__ idx, const int64_t n, const int nf,
                                 const int64_t x_stride, const int b0, const int b1, const int b2, void *buf,
                                 const int sh) {
    using R4 = typename RT<R>::R4;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t b = blockIdx.y;
    R4 *o = reinterpret_cast<R4 *>(buf) + (b * n + i) * nf;
    const int bb[3] = {b0, b1, b2};
    for (int k = 0; k < nf; ++k) o[k] = pos_load<R>(L.xbuf[bb[k]], b, idx[i], x_stride, sh);
}

template <class R>
__global__ void halo_unpack_kernel(const Layout L, const int32_t *__restrict__ idx, const int64_t n, const int nf,
                                   const int64_t x_stride, const int b0, const int b1, const int b2, const void *buf,
                                   const int sh) {
    using R4 = typename RT<R>::R4;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t b = blockIdx.y;
    const R4 *o = reinterpret_cast<const R4 *>(buf) + (b * n + i) * nf;
    const int bb[3] = {b0, b1, b2};
    for (int k = 0; k < nf; ++k) pos_store<R>(L.xbuf[bb[k]], b, idx[i], x_stride, sh, o[k]);
}

// ------------------------------------------------------------------------------------------------
// Peer-store halo transport (pbng_enable_peer_halo / pbng_group_set_transport; PAPER.md:693-705 colour
// order): after a colour's part-1 vertices are final, ONE kernel per neighbour rank reads
// this rank's send rows and stores them straight into the neighbour's ghost rows through a peer mapping
// (NVLink P2P between processes, plain device pointers in the one-GPU loopback group) -- no pack buffer,
// no library copy, no unpack.  Ordering between ranks is carried by two epoch flags per neighbour pair in
// the receiver's memory, E = 1 + pass index within the pbng_iterate call (pass = iteration * colours + colour):
//   pushed[q] = E   rank q's rows of pass E have landed here            (written by q's push kernel)
//   done[q]   = E   rank q has finished every read of pass E            (written by q's signal kernel)
// Rank r's pass E: part 1 -> per neighbour q on the side stream { wait done[q] >= E-1 ; store rows ;
// pushed_on_q[r] = E } || part 2 -> join -> ONE sync kernel { done_on_q[r] = E ; wait pushed[q] >= E for the
// neighbours that send rows of this colour }.  The block's last pass signals, then waits done[q] >= E.
// A wait of pass E refers to what a neighbour does in passes <= E before its own wait of pass E, so by
// induction on E there is no cycle; tests/test_peer_protocol.py model-checks the rules under random rank
// speeds (and shows that dropping either wait breaks the serial colour order).
// ------------------------------------------------------------------------------------------------

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t *p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t global_timer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// bounded spin: a neighbour that never signals (a rank died, mismatched iterate calls) raises bit 1 of
// the context's flag word instead of hanging the GPU; the host reports it as PBNG_E_CUDA
__device__ __forceinline__ void peer_wait(const uint32_t *flag, uint32_t want, int32_t *err, uint64_t timeout_ns) {
    if ((int32_t)(ld_acquire_sys(flag) - want) >= 0) return;
    if (*reinterpret_cast<volatile int32_t *>(err) & 2) return;  // an earlier wait already timed out: fail fast
    const uint64_t t0 = global_timer_ns();
    while ((int32_t)(ld_acquire_sys(flag) - want) < 0) {
        __nanosleep(200);
        if (global_timer_ns() - t0 > timeout_ns) {
            atomicOr(err, 2);
            return;
        }
    }
}

template <class R>
__global__ void __launch_bounds__(256) halo_push_kernel(const Layout L, const PeerPush P) {
    using R4 = typename RT<R>::R4;
    if (P.wait_flag) {  // the neighbour must be done reading pass E-1 before its ghost rows change
        if (threadIdx.x == 0) peer_wait(P.wait_flag, P.wait_val, L.flag, P.timeout_ns);
        __syncthreads();
    }
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t b = blockIdx.y;
    if (i < P.n) {
        const int32_t src = P.idx[i], dst = P.rows[i];
        PBNG_CHECK(src >= 0 && src < L.n_vertices);          // an owned row of this rank
        PBNG_CHECK(dst >= 0 && dst < P.peer_n_vertices);     // a row the neighbour holds (its ghost)
#pragma unroll
        for (int k = 0; k < 3; ++k)
            if (k < P.nf) {
                const R4 x = pos_load<R>(L.xbuf[P.buf[k]], b, src, P.x_stride, P.sh);
                pos_store<R>(P.peer_x[P.buf[k]], b, dst, P.peer_stride, P.peer_sh, x);
            }
    }
    if (P.sig_flag) {
        // the CTA barrier orders every thread's peer stores before thread 0's system-scope fence (fences are
        // cumulative over what the barrier made visible to thread 0), so ONE fence.sys per CTA -- not one per
        // thread -- puts the block's rows before its count; the last block's release store then publishes all
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned total = gridDim.x * gridDim.y;
            if (total == 1) {  // one CTA (the usual halo size): the release store alone publishes its rows
                st_release_sys(P.sig_flag, P.sig_val);
                return;
            }
            __threadfence_system();
            if (atomicAdd(P.counter, 1u) == total - 1) {  // last block: every block's rows have landed
                *P.counter = 0;
                __threadfence_system();  // pairs with the other blocks' fences through the counter
                st_release_sys(P.sig_flag, P.sig_val);
            }
        }
    }
}

// end of pass E on the main stream, one launch: publish done = E in every neighbour's flag words, then wait
// for the rows the neighbours stored in pass E (their pushed flags) before the next pass starts
__global__ void halo_sync_kernel(const PeerSignal S, const PeerWait W, int32_t *err) {
    // the next pass's part-1 sweep is a programmatic dependent launch: its CTAs may start now, prefetch their
    // records (static data) and block in griddepcontrol.wait until this kernel -- i.e. the flag wait -- is done
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int t = threadIdx.x;
    if (t < S.n) st_release_sys(S.flag[t], S.val);  // release: after everything earlier in the stream
    if (t < W.n) peer_wait(W.flags + W.slot[t], W.want, err, W.timeout_ns);
}

// one thread per neighbour: wait until flags[slot[t]] >= want (pushed / done epochs of the neighbours)
__global__ void halo_wait_kernel(const PeerWait W, int32_t *err) {
    const int t = threadIdx.x;
    if (t < W.n) peer_wait(W.flags + W.slot[t], W.want, err, W.timeout_ns);
}

// one thread per neighbour: publish `val` in the neighbour's flag word (all earlier work of the stream,
// this rank's reads of pass E included, is complete at the kernel boundary)
__global__ void halo_signal_kernel(const PeerSignal S) {
    const int t = threadIdx.x;
    if (t < S.n) {
        __threadfence_system();
        st_release_sys(S.flag[t], S.val);
    }
}

// ------------------------------------------------------------------------------------------------
// contact detection (pbng_detect_contacts): a uniform hash grid of the boundary
// triangles (cell size = largest triangle extent + 2 thickness, so a triangle's thickness-inflated box
// covers at most 2 cells per axis), then one thread per free boundary vertex walks its cell's bucket and
// keeps the closest triangle of another body, lexicographically (|p - q|^2, triangle index) -- the
// result does not depend on the bucket order.  fp64 arithmetic for both dtypes.
// ------------------------------------------------------------------------------------------------
template <class R>
__device__ __forceinline__ double3 pos_d(const Layout &L, int work, int64_t b, int64_t v, int64_t xs, int sh) {
    const typename RT<R>::R4 x = pos_load<R>(L.xbuf[work], b, v, xs, sh);
    return make_double3(double(x.x), double(x.y), double(x.z));
}
__device__ __forceinline__ double3 sub(double3 a, double3 b) { return make_double3(a.x - b.x, a.y - b.y, a.z - b.z); }
__device__ __forceinline__ double dot(double3 a, double3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ double3 cross(double3 a, double3 b) {
    return make_double3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ int64_t cell_of(double x, double cs) { return (int64_t)floor(x / cs); }
__device__ __forceinline__ int64_t bucket_of(int64_t i, int64_t j, int64_t k, int64_t nb) {
    const uint64_t h = (uint64_t)i * 73856093ull ^ (uint64_t)j * 19349663ull ^ (uint64_t)k * 83492791ull;
    return (int64_t)(h & (uint64_t)(nb - 1));
}

// closest point of triangle (a, b, c) to p as barycentric weights: the plane projection when it falls
// inside the triangle, else the closest of the three edge-segment projections
__device__ __forceinline__ void closest_on_triangle(double3 p, double3 a, double3 b, double3 c, double (&w)[3]) {
    const double3 e0 = sub(b, a), e1 = sub(c, a), d = sub(p, a);
    const double d00 = dot(e0, e0), d01 = dot(e0, e1), d11 = dot(e1, e1);
    const double den = d00 * d11 - d01 * d01;
    if (den > 0.0) {
        const double d20 = dot(d, e0), d21 = dot(d, e1);
        const double v = (d11 * d20 - d01 * d21) / den, t = (d00 * d21 - d01 * d20) / den;
        if (v >= 0.0 && t >= 0.0 && v + t <= 1.0) {
            w[0] = 1.0 - v - t; w[1] = v; w[2] = t;
            return;
        }
    }
    const double3 P[3] = {a, b, c};
    double best = -1.0;
    for (int k = 0; k < 3; ++k) {  // edge P[k] -> P[k+1]
        const double3 s0 = P[k], s1 = P[(k + 1) % 3], e = sub(s1, s0);
        const double ee = dot(e, e);
        double t = ee > 0.0 ? dot(sub(p, s0), e) / ee : 0.0;
        t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
        const double3 q = make_double3(s0.x + t * e.x, s0.y + t * e.y, s0.z + t * e.z);
        const double dd = dot(sub(p, q), sub(p, q));
        if (best < 0.0 || dd < best) {
            best = dd;
            w[0] = w[1] = w[2] = 0.0;
            w[k] = 1.0 - t;
            w[(k + 1) % 3] = t;
        }
    }
}

template <class R>
__global__ void contact_extent_kernel(const Layout L, const int64_t n_surf, const int work, const int64_t b,
                                      const int64_t xs, const int sh) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_surf) return;
    const int4 tr = L.surf[t];
    const double3 a = pos_d<R>(L, work, b, tr.x, xs, sh), p = pos_d<R>(L, work, b, tr.y, xs, sh),
                  c = pos_d<R>(L, work, b, tr.z, xs, sh);
    const double ex = fmax(fmax(a.x, p.x), c.x) - fmin(fmin(a.x, p.x), c.x);
    const double ey = fmax(fmax(a.y, p.y), c.y) - fmin(fmin(a.y, p.y), c.y);
    const double ez = fmax(fmax(a.z, p.z), c.z) - fmin(fmin(a.z, p.z), c.z);
    atomicMax(L.c_scal, __float_as_uint(__double2float_ru(fmax(fmax(ex, ey), ez))));
}

template <class R>
__global__ void contact_insert_kernel(const Layout L, const int64_t n_surf, const int work, const int64_t b,
                                      const int64_t xs, const int sh, const double thick, const int64_t nb) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_surf) return;
    const double cs = double(__uint_as_float(L.c_scal[0])) + 2.0 * thick;
    const int4 tr = L.surf[t];
    const double3 a = pos_d<R>(L, work, b, tr.x, xs, sh), p = pos_d<R>(L, work, b, tr.y, xs, sh),
                  c = pos_d<R>(L, work, b, tr.z, xs, sh);
    const int64_t i0 = cell_of(fmin(fmin(a.x, p.x), c.x) - thick, cs), i1 = cell_of(fmax(fmax(a.x, p.x), c.x) + thick, cs);
    const int64_t j0 = cell_of(fmin(fmin(a.y, p.y), c.y) - thick, cs), j1 = cell_of(fmax(fmax(a.y, p.y), c.y) + thick, cs);
    const int64_t k0 = cell_of(fmin(fmin(a.z, p.z), c.z) - thick, cs), k1 = cell_of(fmax(fmax(a.z, p.z), c.z) + thick, cs);
    int e = 0;
    for (int64_t i = i0; i <= i1 && i <= i0 + 1; ++i)
        for (int64_t j = j0; j <= j1 && j <= j0 + 1; ++j)
            for (int64_t k = k0; k <= k1 && k <= k0 + 1; ++k, ++e) {
                const int32_t slot = (int32_t)(t * 8 + e);
                const int32_t old = atomicExch(L.c_head + bucket_of(i, j, k, nb), slot);
                L.c_next[slot] = make_int2((int32_t)t, old);
            }
}

template <class R>
__global__ void contact_query_kernel(const Layout L, const int64_t n_sv, const int work, const int64_t b,
                                     const int64_t xs, const int sh, const double thick, const int64_t nb) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n_sv) return;
    const double cs = double(__uint_as_float(L.c_scal[0])) + 2.0 * thick;
    const int2 sv = L.sv[q];
    const double3 p = pos_d<R>(L, work, b, sv.x, xs, sh);
    const double t2 = thick * thick;
    const int32_t head = L.c_head[bucket_of(cell_of(p.x, cs), cell_of(p.y, cs), cell_of(p.z, cs), nb)];
    // pass 0: the least squared distance; pass 1: the lowest triangle index within 1e-10 thickness^2 of
    // it (closest points on shared edges / vertices are ties; include/pbng.h)
    double best = 0.0, bw[3] = {0.0, 0.0, 0.0};
    bool any = false;
    int32_t bt = -1;
    for (int pass = 0; pass < 2 && (pass == 0 || any); ++pass)
        for (int32_t e = head; e >= 0;) {
            const int2 en = L.c_next[e];
            e = en.y;
            const int4 tr = L.surf[en.x];
            if (tr.w == sv.y) continue;  // same body
            const double3 a = pos_d<R>(L, work, b, tr.x, xs, sh), bb = pos_d<R>(L, work, b, tr.y, xs, sh),
                          c = pos_d<R>(L, work, b, tr.z, xs, sh);
            double w[3];
            closest_on_triangle(p, a, bb, c, w);
            const double3 d = make_double3(p.x - (w[0] * a.x + w[1] * bb.x + w[2] * c.x),
                                           p.y - (w[0] * a.y + w[1] * bb.y + w[2] * c.y),
                                           p.z - (w[0] * a.z + w[1] * bb.z + w[2] * c.z));
            const double d2 = dot(d, d);
            if (d2 > t2) continue;
            if (pass == 0) {
                if (!any || d2 < best) best = d2;
                any = true;
            } else if (d2 <= best + 1e-10 * t2 && (bt < 0 || en.x < bt)) {
                bt = en.x;
                bw[0] = w[0]; bw[1] = w[1]; bw[2] = w[2];
            }
        }
    ContactHit h;
    h.tri = bt;
    if (bt >= 0) {
        const int4 tr = L.surf[bt];
        const double3 a = pos_d<R>(L, work, b, tr.x, xs, sh), bb = pos_d<R>(L, work, b, tr.y, xs, sh),
                      c = pos_d<R>(L, work, b, tr.z, xs, sh);
        const double3 n = cross(sub(bb, a), sub(c, a));
        const double nn = sqrt(dot(n, n));
        for (int k = 0; k < 3; ++k) h.bary[k] = bw[k];
        h.normal[0] = nn > 0.0 ? n.x / nn : 0.0;
        h.normal[1] = nn > 0.0 ? n.y / nn : 0.0;
        h.normal[2] = nn > 0.0 ? n.z / nn : 0.0;
    }
    L.c_res[q] = h;
}

// ------------------------------------------------------------------------------------------------
// energy and residual (fp64 arithmetic for both dtypes; fixed-order reductions)
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ double block_sum(double v, double *sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double r = 0.0;
    if (w == 0) {
        r = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
    }
    return r;  // valid in thread 0
}

// Item loops of the energy / residual kernels.  NS = 0: one sample per grid row (blockIdx.y), one item per
// thread.  NS = 1 (sample-minor sh 5): one group of 32 samples per grid row, lane = sample, one item per
// WARP.  NS = 2 (two-sample sh 6): one group pair of 64 samples per grid row, lane = its two samples (the
// two halves of one 32 B slot), one item per warp.  In the warp modes the item's records are warp-uniform
// (broadcast) loads and the position loads of a warp are the item's contiguous sample-minor lines.  All
// reduce in a fixed order (deterministic).
template <int NS>
__device__ __forceinline__ void item_range(int64_t (&b)[2], int64_t &i0, int64_t &step) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (NS > 0) {
        b[0] = (int64_t)blockIdx.y * (32 * NS) + lane;
        b[1] = b[0] + 32;
        i0 = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
        step = (int64_t)gridDim.x * (blockDim.x >> 5);
    } else {
        b[0] = b[1] = blockIdx.y;
        i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        step = (int64_t)gridDim.x * blockDim.x;
    }
}
// the block's partial of sample b: the warp modes sum the block's warps lane by lane (lane = sample)
template <int NS>
__device__ __forceinline__ void store_partial(double acc, double *part, int64_t b, int g, int32_t n_batch,
                                              double *red_sh) {
    if (NS == 0) {
        const double s = block_sum(acc, red_sh);
        if (threadIdx.x == 0) part[b * g + blockIdx.x] = s;
        return;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();  // red_sh may still be read by a previous call
    red_sh[warp * 32 + lane] = acc;
    __syncthreads();
    if (warp == 0) {
        double s = 0.0;
        for (int w = 0; w < nw; ++w) s += red_sh[w * 32 + lane];
        if (b < n_batch) part[b * g + blockIdx.x] = s;
    }
}

template <class R, int MODEL, int NS>
__global__ void __launch_bounds__(kRedBlock) energy_kernel(const Layout L, const int64_t nt, const int64_t n_cons,
                                                           const int64_t x_stride, const int wi, const double cmu,
                                                           const double clam, const double rgx, const double rgy,
                                                           const double rgz, const int ge, const int sh,
                                                           const int64_t n_own, const double idt2,
                                                           const int32_t n_batch) {
    using R4 = typename RT<R>::R4;
    __shared__ double red_sh[kRedBlock];
    int64_t bq[2], i0, istep;
    item_range<NS>(bq, i0, istep);
    constexpr int NQ = NS == 2 ? 2 : 1;
    const void *x = L.xbuf[wi];
    const double r_mu = cmu / (cmu + clam);  // mu / lambdahat, independent of E
    double accq[2] = {0.0, 0.0};
    const int64_t n_items = nt + n_cons + (idt2 > 0.0 ? n_own : 0);
    for (int64_t item = i0; item < n_items; item += istep)
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const int64_t b = bq[q];
        double &acc = accq[q];
        if (item >= nt + n_cons) {  // backward Euler: inertia m_i/(2 dt^2) |x_i - xtilde_i|^2 of owned free nodes
            const int64_t v = item - nt - n_cons;
            const R4 xv = pos_load<R>(x, b, v, x_stride, sh);
            const R4 xt = pos_load<R>(L.xtilde, b, v, x_stride, sh);
            const double dx = double(xv.x) - xt.x, dy = double(xv.y) - xt.y, dz = double(xv.z) - xt.z;
            acc += 0.5 * idt2 * double(ld(reinterpret_cast<const R *>(L.mass) + v)) * (dx * dx + dy * dy + dz * dz);
        } else if (item < nt) {
            const int4 id = ld(L.tet_id + item);
            const R4 ta = ld(reinterpret_cast<const R4 *>(L.tet_a) + item);
            const R4 tb = ld(reinterpret_cast<const R4 *>(L.tet_b) + item);
            const R4 tc = ld(reinterpret_cast<const R4 *>(L.tet_c) + item);
            const R4 q0 = pos_load<R>(x, b, id.x, x_stride, sh), q1 = pos_load<R>(x, b, id.y, x_stride, sh),
                     q2 = pos_load<R>(x, b, id.z, x_stride, sh), q3 = pos_load<R>(x, b, id.w, x_stride, sh);
            const double Bm[3][3] = {{ta.x, ta.y, ta.z}, {ta.w, tb.x, tb.y}, {tb.z, tb.w, tc.x}};
            const double VE = tc.y, V = tc.z;
            const double d[3][3] = {{double(q1.x) - q0.x, double(q1.y) - q0.y, double(q1.z) - q0.z},
                                    {double(q2.x) - q0.x, double(q2.y) - q0.y, double(q2.z) - q0.z},
                                    {double(q3.x) - q0.x, double(q3.y) - q0.y, double(q3.z) - q0.z}};
            double F[3][3];
#pragma unroll
            for (int r = 0; r < 3; ++r)
#pragma unroll
                for (int c = 0; c < 3; ++c) F[r][c] = d[0][r] * Bm[0][c] + d[1][r] * Bm[1][c] + d[2][r] * Bm[2][c];
            const double J = F[0][0] * (F[1][1] * F[2][2] - F[1][2] * F[2][1]) -
                             F[0][1] * (F[1][0] * F[2][2] - F[1][2] * F[2][0]) +
                             F[0][2] * (F[1][0] * F[2][1] - F[1][1] * F[2][0]);
            const double Vmu = VE * cmu, Vlam = VE * clam;
            double e;
            if (MODEL == MODEL_NH) {
                double fro = 0.0;
#pragma unroll
                for (int r = 0; r < 3; ++r)
#pragma unroll
                    for (int c = 0; c < 3; ++c) fro += F[r][c] * F[r][c];
                const double t = J - 1.0 - r_mu;
                e = 0.5 * Vmu * (fro - 3.0) + 0.5 * (Vmu + Vlam) * t * t - 0.5 * Vmu * r_mu;
            } else if (MODEL == MODEL_SNH) {
                double ic = 0.0;
#pragma unroll
                for (int r = 0; r < 3; ++r)
#pragma unroll
                    for (int c = 0; c < 3; ++c) ic += F[r][c] * F[r][c];
                const double Vms = 4.0 / 3.0 * Vmu, Vls = Vlam + 5.0 / 6.0 * Vmu;
                const double al = 1.0 + 3.0 * Vms / (4.0 * Vls);
                // shifted so that Psi(I) = 0 (as Z1 for eq:nh)
                e = 0.5 * Vms * (ic - 3.0) + 0.5 * Vls * (J - al) * (J - al) - 0.5 * Vms * log(1.0 + ic) -
                    (0.5 * Vls * (1.0 - al) * (1.0 - al) - 0.5 * Vms * log(4.0));
            } else {
                double Rm[3][3];
                polar_rotation(F, Rm);
                double s = 0.0;
#pragma unroll
                for (int r = 0; r < 3; ++r)
#pragma unroll
                    for (int c = 0; c < 3; ++c) s += (F[r][c] - Rm[r][c]) * (F[r][c] - Rm[r][c]);
                e = Vmu * s + 0.5 * Vlam * (J - 1.0) * (J - 1.0);
            }
            // - x . f^ext with f^ext_i = sum_e rho g V_e / 4, distributed per tet
            const double sx = double(q0.x) + q1.x + q2.x + q3.x, sy = double(q0.y) + q1.y + q2.y + q3.y,
                         sz = double(q0.z) + q1.z + q2.z + q3.z;
            e -= 0.25 * V * (rgx * sx + rgy * sy + rgz * sz);
            acc += e;
        } else {
            const int64_t c = item - nt;
            const R4 an = ld(reinterpret_cast<const R4 *>(L.c_anchor) + c);
            double C[3] = {-double(an.x), -double(an.y), -double(an.z)};
            const int nn = ld(L.c_n + c);
            for (int q = 0; q < nn; ++q) {
                const R4 y = pos_load<R>(x, b, ld(L.c_node + kWcMaxNodes * c + q), x_stride, sh);
                const double w = ld(reinterpret_cast<const R *>(L.c_w) + kWcMaxNodes * c + q);
                C[0] += w * y.x; C[1] += w * y.y; C[2] += w * y.z;
            }
            const R *Kp = reinterpret_cast<const R *>(L.c_K) + kWcMaxNodes * c;
            const double kxx = ld(Kp + 0), kyy = ld(Kp + 1), kzz = ld(Kp + 2), kxy = ld(Kp + 3), kyz = ld(Kp + 4),
                         kxz = ld(Kp + 5);
            acc += 0.5 * (C[0] * (kxx * C[0] + kxy * C[1] + kxz * C[2]) + C[1] * (kxy * C[0] + kyy * C[1] + kyz * C[2]) +
                          C[2] * (kxz * C[0] + kyz * C[1] + kzz * C[2]));
        }
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) store_partial<NS>(accq[q], L.part_e, bq[q], ge, n_batch, red_sh);
}

template <class R, int MODEL, bool FEXT, bool WC, int NS>
__global__ void __launch_bounds__(kRedBlock) residual_kernel(const Layout L, const int64_t n_chunks,
                                                             const int64_t x_stride, const int wi, const double cmu,
                                                             const double clam, const int gr, const int sh,
                                                             const double idt2, const bool path,
                                                             const int32_t n_batch) {
    using R4 = typename RT<R>::R4;
    __shared__ double red_sh[kRedBlock];
    int64_t bq[2], i0, istep;
    item_range<NS>(bq, i0, istep);
    constexpr int NQ = NS == 2 ? 2 : 1;
    const void *x = L.xbuf[wi];
    double accq[2] = {0.0, 0.0};
    for (int64_t t = i0; t < n_chunks * kChunk; t += istep)
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const int64_t b = bq[q];
        double &acc = accq[q];
        const int64_t chunk = t >> 5;
        const int cl = (int)(t & 31);  // the vertex's lane in its chunk
        const int2 cv = L.chunk_v[chunk];
        if (cl >= cv.y) continue;
        const int v = cv.x + cl;
        const int64_t base = L.chunk_off[chunk] + cl;
        const int deg = L.deg[v];
        const R4 xa4 = pos_load<R>(x, b, v, x_stride, sh);
        const double xa[3] = {xa4.x, xa4.y, xa4.z};
        double f[3] = {0.0, 0.0, 0.0}, A[6];
        if (FEXT) {
            const R4 fe = reinterpret_cast<const R4 *>(L.fext)[v];
            f[0] = fe.x; f[1] = fe.y; f[2] = fe.z;
        }
        bool done = false;
        if constexpr (MODEL == MODEL_NH) {
            if (path) {  // path records: three slots, one new neighbour per record
                const int2 p0 = L.path0[v];
                R4 S0 = xa4, S1 = pos_load<R>(x, b, p0.x, x_stride, sh), S2 = pos_load<R>(x, b, p0.y, x_stride, sh);
                const bool rest = L.path_mode == 2;  // rest-recompute records: the sweep's own rebuild
                R4 T0 = xa4, T1 = xa4, T2 = xa4;
                R Xi[3] = {R(0), R(0), R(0)};
                if (rest) {
                    T0 = rest_at<R>(L, v);
                    T1 = rest_at<R>(L, p0.x);
                    T2 = rest_at<R>(L, p0.y);
                    Xi[0] = T0.x; Xi[1] = T0.y; Xi[2] = T0.z;
                }
                for (int k = 0; k < deg; ++k) {
                    Pair<R, MODEL_NH> pr;
                    int code;
                    if (rest) {
                        R E6;
                        code = load_rest_rec<true>(L, base + (int64_t)k * kChunk, E6);
                        path_push(T0, T1, T2, rest_at<R>(L, code & 0x3fffffff), code);
                        rest_pair<R>(T0, T1, T2, Xi, E6, pr);
                    } else if (L.path_mode == 3) {
                        const int64_t r = group_base(base) + (int64_t)(k - k % RG) * kChunk + k % RG;
                        code = load_path_rec<true, true>(L, r, pr);
                    } else {
                        code = load_path_rec<true>(L, base + (int64_t)k * kChunk, pr);
                    }
                    path_push(S0, S1, S2, pos_load<R>(x, b, code & 0x3fffffff, x_stride, sh), code);
                    const double d1[3] = {S0.x - xa[0], S0.y - xa[1], S0.z - xa[2]};
                    const double d2[3] = {S1.x - xa[0], S1.y - xa[1], S1.z - xa[2]};
                    const double d3[3] = {S2.x - xa[0], S2.y - xa[1], S2.z - xa[2]};
                    contrib<false>(d1, d2, d3, pr, cmu, clam, f, A);
                }
                done = true;
            }
        }
        for (int k = 0; k < deg && !done; ++k) {
            Pair<R, MODEL> pr;
            load_pair<true>(L, base + (int64_t)k * kChunk, pr);
            const R4 p1 = pos_load<R>(x, b, pr.id.x, x_stride, sh), p2 = pos_load<R>(x, b, pr.id.y, x_stride, sh),
                     p3 = pos_load<R>(x, b, pr.id.z, x_stride, sh);
            const double d1[3] = {p1.x - xa[0], p1.y - xa[1], p1.z - xa[2]};
            const double d2[3] = {p2.x - xa[0], p2.y - xa[1], p2.z - xa[2]};
            const double d3[3] = {p3.x - xa[0], p3.y - xa[1], p3.z - xa[2]};
            contrib<false>(d1, d2, d3, pr, cmu, clam, f, A);
        }
        if (WC) wc_contrib_at<R, double, false>(L, x, b, x_stride, sh, v, xa, f, A);
        if (idt2 > 0.0) inertia_contrib<R, double>(L, v, pos_load<R>(L.xtilde, b, v, x_stride, sh), idt2, xa, f, A);
        acc += f[0] * f[0] + f[1] * f[1] + f[2] * f[2];
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) store_partial<NS>(accq[q], L.part_r, bq[q], gr, n_batch, red_sh);
}

__global__ void __launch_bounds__(kRedBlock) reduce_kernel(const Layout L, const int ge, const int gr) {
    __shared__ double red_sh[32];
    const int64_t b = blockIdx.x;
    double e = 0.0, r = 0.0;
    for (int k = threadIdx.x; k < ge; k += blockDim.x) e += L.part_e[b * ge + k];
    for (int k = threadIdx.x; k < gr; k += blockDim.x) r += L.part_r[b * gr + k];
    e = block_sum(e, red_sh);
    __syncthreads();
    r = block_sum(r, red_sh);
    if (threadIdx.x == 0) {
        L.results[2 * b] = e;
        L.results[2 * b + 1] = sqrt(r);
    }
}

template <class R, int MODEL, int NS>
cudaError_t energy_residual_launch(const Problem &p, const Layout &L, int wi, cudaStream_t st) {
    const unsigned rows = NS > 0 ? (unsigned)((p.n_batch + 32 * NS - 1) / (32 * NS)) : (unsigned)p.n_batch;
    energy_kernel<R, MODEL, NS><<<dim3(p.ge, rows), kRedBlock, 0, st>>>(
        L, p.n_tets, p.n_cons, p.x_stride, wi, p.cmu, p.clam, p.rho_g[0], p.rho_g[1], p.rho_g[2], p.ge, p.lane_shift,
        p.n_own, p.inv_dt2, p.n_batch);
    dim3 gr(p.gr, rows);
    const auto a = std::make_tuple(L, p.n_chunks, p.x_stride, wi, p.cmu, p.clam, p.gr, p.lane_shift, p.inv_dt2, p.path,
                                   p.n_batch);
    auto go = [&](auto kern) {
        std::apply([&](auto... xs) { kern<<<gr, kRedBlock, 0, st>>>(xs...); }, a);
    };
    if (p.has_fext) {
        if (p.has_wc) go(residual_kernel<R, MODEL, true, true, NS>);
        else go(residual_kernel<R, MODEL, true, false, NS>);
    } else {
        if (p.has_wc) go(residual_kernel<R, MODEL, false, true, NS>);
        else go(residual_kernel<R, MODEL, false, false, NS>);
    }
    reduce_kernel<<<p.n_batch, kRedBlock, 0, st>>>(L, p.ge, p.gr);
    return cudaGetLastError();
}

template <class R, int MODEL>
cudaError_t energy_dispatch(const Problem &p, const Layout &L, int wi, cudaStream_t st) {
    // batched layouts: a warp covers one item for 32 (sh 5) or 64 (sh 6) samples
    if (p.lane_shift == 6) return energy_residual_launch<R, MODEL, 2>(p, L, wi, st);
    if (p.lane_shift == 5) return energy_residual_launch<R, MODEL, 1>(p, L, wi, st);
    return energy_residual_launch<R, MODEL, 0>(p, L, wi, st);
}

// test hook: R(F) of the device polar decomposition for n matrices (pbng_test_polar)
template <class R>
__global__ void polar_test_kernel(const double *F, double *Rout, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    R Fm[3][3], Rm[3][3];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) Fm[a][b] = R(F[9 * i + 3 * a + b]);
    R C[3][3];
    C[0][0] = Fm[1][1] * Fm[2][2] - Fm[1][2] * Fm[2][1];
    C[0][1] = Fm[1][2] * Fm[2][0] - Fm[1][0] * Fm[2][2];
    C[0][2] = Fm[1][0] * Fm[2][1] - Fm[1][1] * Fm[2][0];
    C[1][0] = Fm[0][2] * Fm[2][1] - Fm[0][1] * Fm[2][2];
    C[1][1] = Fm[0][0] * Fm[2][2] - Fm[0][2] * Fm[2][0];
    C[1][2] = Fm[0][1] * Fm[2][0] - Fm[0][0] * Fm[2][1];
    C[2][0] = Fm[0][1] * Fm[1][2] - Fm[0][2] * Fm[1][1];
    C[2][1] = Fm[0][2] * Fm[1][0] - Fm[0][0] * Fm[1][2];
    C[2][2] = Fm[0][0] * Fm[1][1] - Fm[0][1] * Fm[1][0];
    const R J = Fm[0][0] * C[0][0] + Fm[0][1] * C[0][1] + Fm[0][2] * C[0][2];
    polar_fcr(Fm, C, J, Rm);  // the routine the fixed-corotated sweep uses for this dtype
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) Rout[9 * i + 3 * a + b] = double(Rm[a][b]);
}

}  // namespace

// Per-(dtype, model) entry points.  build.py compiles this file once per (dtype, model) with
// PBNG_TU_R / PBNG_TU_MODEL set (the sweep and energy/residual instantiations of that pair, compiled in
// parallel) and once without them (the dispatchers and the model-independent kernels).
template <class R, int MODEL>
cudaError_t sweep_entry(const Problem &p, const Layout &L, const SweepLaunch &s, cudaStream_t st);
template <class R, int MODEL>
cudaError_t energy_entry(const Problem &p, const Layout &L, int work, cudaStream_t st);
template <class R, int MODEL>
cudaError_t pipe_entry(const Problem &p, const Layout &L, const PipeLaunch &s, cudaStream_t st);
template <class R, int MODEL>
cudaError_t b2win_entry(const Problem &p, const Layout &L, const B2Window &w, int accel, cudaStream_t st);

#if defined(PBNG_TU_R)
template <class R, int MODEL>
cudaError_t b2win_entry(const Problem &p, const Layout &L, const B2Window &w, int accel, cudaStream_t st) {
    if constexpr (sizeof(R) == 4 && MODEL == MODEL_NH) {
        // persistent grid: every SM filled to the instance's occupancy (items are taken in order by running
        // CTAs and only wait for earlier items, so a larger grid could not deadlock either)
        const bool fe = p.has_fext, wcn = p.has_wc;
        auto go = [&](auto kern) -> cudaError_t {
            int per_sm = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSweepBlock, 0);
            const int blocks = std::max(1, (p.sm_count > 0 ? p.sm_count : 148) * std::max(1, per_sm));
            kern<<<(unsigned)blocks, kSweepBlock, 0, st>>>(L, w, p.x_stride, p.n_batch, float(p.cmu), float(p.clam),
                                                          float(p.inv_dt2));
            return cudaGetLastError();
        };
#define PBNG_B2W(A)                                                                   \
    if (fe && wcn) return go(sweep_batched2_window_kernel<A, true, true>);          \
    if (fe) return go(sweep_batched2_window_kernel<A, true, false>);                \
    if (wcn) return go(sweep_batched2_window_kernel<A, false, true>);               \
    return go(sweep_batched2_window_kernel<A, false, false>);
        if (accel == ACCEL_SOR) { PBNG_B2W(ACCEL_SOR) }
        if (accel == ACCEL_CHEB) { PBNG_B2W(ACCEL_CHEB) }
        PBNG_B2W(ACCEL_NONE)
#undef PBNG_B2W
    } else {
        (void)p; (void)L; (void)w; (void)accel; (void)st;
        return cudaErrorInvalidValue;
    }
}
template cudaError_t b2win_entry<PBNG_TU_R, PBNG_TU_MODEL>(const Problem &, const Layout &, const B2Window &, int,
                                                           cudaStream_t);
template <class R, int MODEL>
cudaError_t pipe_entry(const Problem &p, const Layout &L, const PipeLaunch &s, cudaStream_t st) {
    return pipe_dispatch2<R, MODEL>(p, L, s, st);
}
template cudaError_t pipe_entry<PBNG_TU_R, PBNG_TU_MODEL>(const Problem &, const Layout &, const PipeLaunch &,
                                                          cudaStream_t);
template <class R, int MODEL>
cudaError_t sweep_entry(const Problem &p, const Layout &L, const SweepLaunch &s, cudaStream_t st) {
    return sweep_dispatch2<R, MODEL>(p, L, s, st);
}
template <class R, int MODEL>
cudaError_t energy_entry(const Problem &p, const Layout &L, int work, cudaStream_t st) {
    return energy_dispatch<R, MODEL>(p, L, work, st);
}
template cudaError_t sweep_entry<PBNG_TU_R, PBNG_TU_MODEL>(const Problem &, const Layout &, const SweepLaunch &,
                                                           cudaStream_t);
template cudaError_t energy_entry<PBNG_TU_R, PBNG_TU_MODEL>(const Problem &, const Layout &, int, cudaStream_t);
#else

cudaError_t launch_b2_window(const Problem &p, const Layout &L, const B2Window &w, int accel, cudaStream_t st) {
    if (w.n_iter <= 0 || p.n_chunks <= 0) return cudaSuccess;
    return b2win_entry<float, MODEL_NH>(p, L, w, accel, st);
}

cudaError_t launch_sweep_pipe(const Problem &p, const Layout &L, const PipeLaunch &s, cudaStream_t st) {
    if (s.n_iter <= 0 || p.n_chunks <= 0) return cudaSuccess;
    if (p.dtype == DT_F64) {
        if (p.model == MODEL_FCR) return pipe_entry<double, MODEL_FCR>(p, L, s, st);
        if (p.model == MODEL_SNH) return pipe_entry<double, MODEL_SNH>(p, L, s, st);
        return pipe_entry<double, MODEL_NH>(p, L, s, st);
    }
    if (p.model == MODEL_FCR) return pipe_entry<float, MODEL_FCR>(p, L, s, st);
    if (p.model == MODEL_SNH) return pipe_entry<float, MODEL_SNH>(p, L, s, st);
    return pipe_entry<float, MODEL_NH>(p, L, s, st);
}

cudaError_t launch_sweep(const Problem &p, const Layout &L, const SweepLaunch &s, cudaStream_t st) {
    if (s.n_v <= 0) return cudaSuccess;
    if (p.dtype == DT_F64) {
        if (p.model == MODEL_FCR) return sweep_entry<double, MODEL_FCR>(p, L, s, st);
        if (p.model == MODEL_SNH) return sweep_entry<double, MODEL_SNH>(p, L, s, st);
        return sweep_entry<double, MODEL_NH>(p, L, s, st);
    }
    if (p.model == MODEL_FCR) return sweep_entry<float, MODEL_FCR>(p, L, s, st);
    if (p.model == MODEL_SNH) return sweep_entry<float, MODEL_SNH>(p, L, s, st);
    return sweep_entry<float, MODEL_NH>(p, L, s, st);
}

// n_buffers = -1: write the staged array into the backward-Euler target xtilde instead
cudaError_t launch_set_positions(const Problem &p, const Layout &L, int n_buffers, cudaStream_t st) {
    if (p.n_vertices <= 0) return cudaSuccess;
    dim3 grid((unsigned)((p.n_vertices + 255) / 256), (unsigned)p.n_batch);
    if (p.dtype == DT_F64)
        set_positions_kernel<double><<<grid, 256, 0, st>>>(L, p.n_vertices, p.n_global, p.n_free, p.n_pinned, p.x_stride, n_buffers, p.lane_shift);
    else
        set_positions_kernel<float><<<grid, 256, 0, st>>>(L, p.n_vertices, p.n_global, p.n_free, p.n_pinned, p.x_stride, n_buffers, p.lane_shift);
    return cudaGetLastError();
}

cudaError_t launch_get_positions(const Problem &p, const Layout &L, int work, cudaStream_t st) {
    if (p.n_vertices <= 0) return cudaSuccess;
    dim3 grid((unsigned)((p.n_vertices + 255) / 256), (unsigned)p.n_batch);
    if (p.dtype == DT_F64)
        get_positions_kernel<double><<<grid, 256, 0, st>>>(L, p.n_vertices, p.n_global, p.x_stride, work, p.lane_shift);
    else
        get_positions_kernel<float><<<grid, 256, 0, st>>>(L, p.n_vertices, p.n_global, p.x_stride, work, p.lane_shift);
    return cudaGetLastError();
}

cudaError_t launch_halo_pack(const Problem &p, const Layout &L, const int32_t *idx, int64_t n, int n_fields,
                             const int (&bufs)[3], void *buf, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    dim3 grid((unsigned)((n + 255) / 256), (unsigned)p.n_batch);
    if (p.dtype == DT_F64)
        halo_pack_kernel<double><<<grid, 256, 0, st>>>(L, idx, n, n_fields, p.x_stride, bufs[0], bufs[1], bufs[2], buf, p.lane_shift);
    else
        halo_pack_kernel<float><<<grid, 256, 0, st>>>(L, idx, n, n_fields, p.x_stride, bufs[0], bufs[1], bufs[2], buf, p.lane_shift);
    return cudaGetLastError();
}

cudaError_t launch_halo_unpack(const Problem &p, const Layout &L, const int32_t *idx, int64_t n, int n_fields,
                               const int (&bufs)[3], const void *buf, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    dim3 grid((unsigned)((n + 255) / 256), (unsigned)p.n_batch);
    if (p.dtype == DT_F64)
        halo_unpack_kernel<double><<<grid, 256, 0, st>>>(L, idx, n, n_fields, p.x_stride, bufs[0], bufs[1], bufs[2], buf, p.lane_shift);
    else
        halo_unpack_kernel<float><<<grid, 256, 0, st>>>(L, idx, n, n_fields, p.x_stride, bufs[0], bufs[1], bufs[2], buf, p.lane_shift);
    return cudaGetLastError();
}

cudaError_t launch_halo_push(const Problem &p, const Layout &L, const PeerPush &P, cudaStream_t st) {
    if (P.n <= 0 && !P.sig_flag) return cudaSuccess;
    dim3 grid((unsigned)std::max<int64_t>((P.n + 255) / 256, 1), (unsigned)p.n_batch);
    if (p.dtype == DT_F64)
        halo_push_kernel<double><<<grid, 256, 0, st>>>(L, P);
    else
        halo_push_kernel<float><<<grid, 256, 0, st>>>(L, P);
    return cudaGetLastError();
}

cudaError_t launch_halo_wait(const Layout &L, const PeerWait &W, cudaStream_t st) {
    if (W.n <= 0) return cudaSuccess;
    halo_wait_kernel<<<1, 64, 0, st>>>(W, L.flag);
    return cudaGetLastError();
}

cudaError_t launch_halo_sync(const Layout &L, const PeerSignal &S, const PeerWait &W, cudaStream_t st) {
    if (S.n <= 0 && W.n <= 0) return cudaSuccess;
    halo_sync_kernel<<<1, 64, 0, st>>>(S, W, L.flag);
    return cudaGetLastError();
}

cudaError_t launch_halo_signal(const PeerSignal &S, cudaStream_t st) {
    if (S.n <= 0) return cudaSuccess;
    halo_signal_kernel<<<1, 64, 0, st>>>(S);
    return cudaGetLastError();
}

cudaError_t launch_energy_residual(const Problem &p, const Layout &L, int work, cudaStream_t st) {
    if (p.dtype == DT_F64) {
        if (p.model == MODEL_FCR) return energy_entry<double, MODEL_FCR>(p, L, work, st);
        if (p.model == MODEL_SNH) return energy_entry<double, MODEL_SNH>(p, L, work, st);
        return energy_entry<double, MODEL_NH>(p, L, work, st);
    }
    if (p.model == MODEL_FCR) return energy_entry<float, MODEL_FCR>(p, L, work, st);
    if (p.model == MODEL_SNH) return energy_entry<float, MODEL_SNH>(p, L, work, st);
    return energy_entry<float, MODEL_NH>(p, L, work, st);
}

int kernels_per_energy_residual() { return 3; }

template <class R>
cudaError_t contacts_dispatch(const Problem &p, const Layout &L, int work, int sample, double thick, cudaStream_t st) {
    const unsigned g1 = (unsigned)((p.n_surf + 255) / 256), g2 = (unsigned)((p.n_sv + 255) / 256);
    cudaError_t e = cudaMemsetAsync(L.c_scal, 0, 4, st);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(L.c_head, 0xff, (size_t)p.n_cbuckets * 4, st);
    if (e != cudaSuccess) return e;
    contact_extent_kernel<R><<<g1, 256, 0, st>>>(L, p.n_surf, work, sample, p.x_stride, p.lane_shift);
    contact_insert_kernel<R><<<g1, 256, 0, st>>>(L, p.n_surf, work, sample, p.x_stride, p.lane_shift, thick, p.n_cbuckets);
    contact_query_kernel<R><<<g2, 256, 0, st>>>(L, p.n_sv, work, sample, p.x_stride, p.lane_shift, thick, p.n_cbuckets);
    return cudaGetLastError();
}

cudaError_t launch_contacts(const Problem &p, const Layout &L, int work, int sample, double thickness, cudaStream_t st) {
    if (p.n_surf <= 0 || p.n_sv <= 0) return cudaSuccess;
    return p.dtype == DT_F64 ? contacts_dispatch<double>(p, L, work, sample, thickness, st)
                             : contacts_dispatch<float>(p, L, work, sample, thickness, st);
}

int kernels_per_contacts() { return 3; }

cudaError_t launch_polar_test(int dtype, const double *F, double *R, int64_t n, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const unsigned g = (unsigned)((n + 127) / 128);
    if (dtype == DT_F64) polar_test_kernel<double><<<g, 128, 0, st>>>(F, R, n);
    else polar_test_kernel<float><<<g, 128, 0, st>>>(F, R, n);
    return cudaGetLastError();
}

#endif  // PBNG_TU_R

}  // namespace pbng
