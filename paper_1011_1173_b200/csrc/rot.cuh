// rot.cuh -- device building blocks of the sweep: the row Compute (diagonal
// chain) and the scaled 2-FMA Apply.  Shared by every algorithm of the library.
//
// Paper, for row j, update column e, column m > j:
//   Compute: w = sqrt(d^2 + sigma v^2), c = w/d, s = v/d, L_jj <- w
//   Apply:   L_jm <- (L_jm + sigma s V_me)/c ;  V_me <- c V_me - s L_jm(new)
// Restatement used here (exact in real arithmetic,
// rounding-only differences; keeps the paper's mixed form: V uses the NEW L):
//   x_{j,e}   = L_jj^2 + sigma sum_{e'<=e} v_{j,e'}^2  (= w_{j,e}^2, no sqrt on the chain)
//   mu_{j,e}  = prod_{rows j' of the block, j'<=j} w_{j',e-1}/w_{j',e} = prod 1/c
//   Vt        = mu_{j-1,e} V   (scaled V state; mu = 1 at the start of a row block)
//   Lh        = (w_{j,e}/L_jj) L^{(e)}  (scaled L, starts as the raw L_jm)
//   Apply(j,e,m):  Lh += gamma_{j,e} Vt_e ;  Vt_e -= delta_{j,e} Lh      (2 FMA)
//   with gamma = sigma vt IM_{j-1,e} / L_jj,  delta = vt L_jj / x_{j,e},
//   IM = 1/mu^2, vt = mu_{j-1,e} v_{j,e};  finally L_jm = Lh * rho_j,
//   rho_j = L_jj / w_{j,k-1};  at the end of the block V = Vt * nu_e,
//   nu_e = sqrt(IM_{last,e}) = 1/mu_{last,e}.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "internal.h"

namespace gcm {

constexpr unsigned kFull = 0xffffffffu;

// Reciprocal and reciprocal square root on the chain: the MUFU approximation
// plus two Newton steps (quadratic convergence from ~2^-23: fully accurate to a
// couple of ulp) instead of the IEEE division/sqrt sequences with their
// slow-path branches (rounding-only difference).
__device__ __forceinline__ double fast_rcp(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}
__device__ __forceinline__ double fast_rsqrt(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double h = 0.5 * x;
    y = y * fma(-h * y, y, 1.5);
    return y * fma(-h * y, y, 1.5);
}

// fp32 counterparts (the single-precision path, GCM fp32 entry points; PAPER.md 111 ran
// both precisions): IEEE round-to-nearest reciprocal, rsqrt + one Newton step
__device__ __forceinline__ float fast_rcp(float x) { return __frcp_rn(x); }
__device__ __forceinline__ float fast_rsqrt(float x) {
    const float y = rsqrtf(x);
    return y * fmaf(-0.5f * x * y, y, 1.5f);
}
template <typename T>
struct V2;
template <>
struct V2<double> {
    using type = double2;
    static __device__ __forceinline__ double2 make(double a, double b) { return make_double2(a, b); }
};
template <>
struct V2<float> {
    using type = float2;
    static __device__ __forceinline__ float2 make(float a, float b) { return make_float2(a, b); }
};
template <typename T>
__device__ __forceinline__ T qnan();
template <>
__device__ __forceinline__ double qnan<double>() { return __longlong_as_double(0x7ff8000000000000ll); }
template <>
__device__ __forceinline__ float qnan<float>() { return __int_as_float(0x7fc00000); }

__device__ __forceinline__ void record_failure(unsigned long long *key, int64_t e, int64_t row, int code) {
    atomicMin(key, info_key(e, row, code));
}

// Row Compute for one row j, executed by ONE full warp (lane = update column
// within a chunk of 32).  Inputs: d0 = L_jj on entry, vrow[e] = vt_{j,e}
// (scaled residual, shared memory), IM[e] = 1/mu^2_{j-1,e} (shared, updated
// in place to 1/mu^2_{j,e}).  Outputs: cs[e] = (gamma, delta) in shared memory,
// optionally mirrored to gpanel[2e..2e+1] (global), V_exit[e*ldv] = v_{j,e}
// (true residual, PAPER.md 105) if vexit != nullptr.  Returns w = L~_jj on all
// lanes.  grow = global row index, ebase = index of update column 0 of this
// pass (for failure reports).
template <typename T>
__device__ __forceinline__ T compute_row_warp(int lane, T d0, const T *vrow, T *IM, typename V2<T>::type *cs,
                                              T *gpanel, T *vexit, int64_t ldv, int k, int sigma, int64_t grow,
                                              int64_t ebase, unsigned long long *key) {
    T d = d0;
    if (!(d > T(0))) {  // non-positive pivot on entry (R5)
        if (lane == 0) record_failure(key, ebase, grow, 2);
        d = qnan<T>();
    }
    const T invd = fast_rcp(d);
    T base = d * d;  // x_{j,-1}
    T rbase = invd * invd;
    for (int c0 = 0; c0 < k; c0 += 32) {
        const int e = c0 + lane;
        const bool valid = e < k;
        const T vt = valid ? vrow[e] : T(0);
        const T im = valid ? IM[e] : T(1);
        const T a = sigma > 0 ? vt * im : -(vt * im);  // sigma vt IM
        // inclusive scan over lanes of a*vt  ->  x_{j,e} = x_{j,c0-1} + scan
        T s = a * vt;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const T y = __shfl_up_sync(kFull, s, off);
            if (lane >= off) s += y;
        }
        T x = base + s;
        const bool bad = valid && !(x > T(0));
        const unsigned badmask = __ballot_sync(kFull, bad);
        if (badmask) {
            const int first = __ffs(badmask) - 1;
            if (lane == first) record_failure(key, ebase + e, grow, 1);
            if (lane >= first) x = qnan<T>();
        }
        const T rx = fast_rcp(x);
        T rxp = __shfl_up_sync(kFull, rx, 1);
        if (lane == 0) rxp = rbase;
        if (valid) {
            const T gam = a * invd;
            const T del = vt * d * rx;
            IM[e] = im * x * rxp;
            cs[e] = V2<T>::make(gam, del);
            if (gpanel) {
                gpanel[2 * e] = gam;
                gpanel[2 * e + 1] = del;
            }
            if (vexit) vexit[(int64_t)e * ldv] = vt * sqrt(im);
        }
        base = __shfl_sync(kFull, x, 31);
        rbase = __shfl_sync(kFull, rx, 31);
    }
    return sqrt(base);
}

// Apply the k rotations of one row (coefficients cs[0..k-1] in shared memory)
// to one (L element, V state) pair held by this thread; returns the final L.
template <int KMAX, typename T>
__device__ __forceinline__ T apply_row(T l, T (&v)[KMAX], const typename V2<T>::type *cs, T rho, int k) {
#pragma unroll
    for (int e = 0; e < KMAX; ++e) {
        if (e < k) {
            const auto gd = cs[e];
            l = fma(gd.x, v[e], l);
            v[e] = fma(-gd.y, l, v[e]);
        }
    }
    return l * rho;
}

// The in-block sweep of one D-row diagonal block (PAPER.md lines 24-30
// restricted to rows/columns r0 .. r0+Db-1), run by a CTA whose threads
// tbase .. tbase+Db-1 own the block's columns: thread tbase+m owns column r0+m
// with its V state v[] (TRUE values on entry, i.e. mu = 1); Ls[m][j] =
// L(r0+j, r0+m) in shared memory.  The warp starting at thread tbase (tbase a
// multiple of 32, Db <= blockDim - tbase) computes the rows' coefficients.
// Emits the block's coefficient panel (gamma/delta, rho, nu; layout in
// internal.h, panel may be shared or global memory), V_exit rows r0..
// (vexit + e*ldv), and leaves L~ in Ls.  Must be called by ALL threads of the CTA.
template <int KMAX, int LD, typename T>
__device__ __forceinline__ void block_sweep(T (*Ls)[LD], T (&v)[KMAX], int Db, int k, int sigma, int64_t r0,
                                            T *panel, T *vexit, int64_t ldv, unsigned long long *key, int64_t ebase,
                                            T *vrow, T *IM, typename V2<T>::type *cs, T *rho_s, int tbase = 0) {
    const int t = threadIdx.x;
    const int m = t - tbase;  // own column within the block (valid if 0 <= m < Db)
    const int lane = t & 31;
    for (int e = t; e < k; e += blockDim.x) IM[e] = T(1);
    T *rho_g = panel + 2ll * kD * k;
    for (int j = 0; j < Db; ++j) {
        if (m == j) {
#pragma unroll
            for (int e = 0; e < KMAX; ++e)
                if (e < k) vrow[e] = v[e];
        }
        __syncthreads();
        if (m >= 0 && m < 32) {
            const T d0 = Ls[j][j];
            const T w = compute_row_warp<T>(lane, d0, vrow, IM, cs, panel + 2ll * j * k, vexit + j, ldv, k, sigma,
                                            r0 + j, ebase, key);
            if (lane == 0) {
                const T rho = d0 / w;
                *rho_s = rho;
                rho_g[j] = rho;
                Ls[j][j] = w;
            }
        }
        __syncthreads();
        if (m > j && m < Db) Ls[m][j] = apply_row<KMAX>(Ls[m][j], v, cs, *rho_s, k);
    }
    __syncthreads();
    T *nu_g = panel + 2ll * kD * k + kD;
    for (int e = t; e < k; e += blockDim.x) nu_g[e] = sqrt(IM[e]);
}

// Wavefront variant of block_sweep.  The Compute
// of (row j, column e) needs only (j, e-1) [through x] and (j-1, e) [through
// column j's V after row j-1's rotation e], so all (j, e) on an anti-diagonal
// j + e = tau are independent: tick tau computes them in one dedicated warp
// (lane = e) and, after one barrier, the column threads apply them.  The block
// costs Db + KB - 1 ticks instead of Db full rows.  The running L of element
// (j, m) lives in Ls[m][j] between ticks, so the KB rotations of a column can be
// split over NQ threads (thread (m, q) owns update columns q*KB/NQ ..) at no cost.
// The rank is padded to KB (update columns k..KB-1 have V = 0: identity
// rotations, gamma = delta = 0), so all indices are compile-time.
//   Vs[m*KB + e]   : column m's TRUE V state at block start (caller fills, smem, and
//                    synchronises the CTA before the call)
//   Ls[m][j]       : L(r0+j, r0+m) (smem), L~ on exit
//   threads tbase + q*kD + m (q < NQ, m < Db) : column parts; warp cwarp: coefficients
//   pan            : smem panel, (gamma, delta) at pan[2*(j*KB+e)], rho at 2*kD*KB, nu at +kD
// Scratch (smem): vx[kD*KB], dinv[kD], vt[kD*KB], imx[kD*KB].  Called by ALL threads.
#ifdef GCM_SWEEP_TRACE
__device__ long long gcm_sweep_trace[2048];
#endif
__host__ __device__ constexpr int wave_panel_doubles(int KB) { return 2 * kD * KB + kD + KB; }

template <int KB, int NQ, int LD>
__device__ __forceinline__ void wave_sweep(double (*Ls)[LD], const double *Vs, int Db, int k, int sigma, int64_t r0,
                                           double *pan, double *vexit, int64_t ldv, unsigned long long *key,
                                           int64_t ebase, double *vx, double *dinv, double *vt, double *imx,
                                           int tbase, int cwarp) {
    static_assert(KB <= 32 && KB % NQ == 0, "wave_sweep: KB <= 32 update columns, NQ | KB");
    constexpr int EPT = KB / NQ;
    const int t = threadIdx.x;
    const int rel = t - tbase;
    const int m = rel % kD, q = rel / kD;
    const bool colthr = rel >= 0 && rel < NQ * kD && m < Db;
    const bool cthr = (t >> 5) == cwarp;
    const int lane = t & 31;
    double *rho_g = pan + 2 * kD * KB;
    double *nu_g = rho_g + kD;
    const int e0 = q * EPT;
    double v[EPT];
    if (colthr) {
#pragma unroll
        for (int i = 0; i < EPT; ++i) v[i] = Vs[m * KB + e0 + i];
        if (m == 0)
#pragma unroll
            for (int i = 0; i < EPT; ++i) vx[e0 + i] = v[i];  // row 0 computes on the initial V
        if (q == 0) {
            double d = Ls[m][m];
            if (!(d > 0.0)) d = __longlong_as_double(0x7ff8000000000000ll);
            dinv[m] = fast_rcp(d);
        }
    }
    __syncthreads();
    double im = 1.0;             // compute lane e: 1/mu^2 of its previous row
    double xr = 0.0, rxr = 0.0;  // x_{j,e} and 1/x_{j,e} of the last tick (read by lane e+1)
    const int ticks = Db + KB - 1;
    for (int tau = 0; tau < ticks; ++tau) {
#ifdef GCM_SWEEP_TRACE
        if (blockIdx.x == 0 && t == 0) gcm_sweep_trace[tau * 4 + 0] = clock64();
#endif
        if (cthr) {
            const int e = lane;
            const int j = tau - e;
            const double xup = __shfl_up_sync(kFull, xr, 1);
            const double rxup = __shfl_up_sync(kFull, rxr, 1);
            if (e < KB && j >= 0 && j < Db) {
                const double d = Ls[j][j];
                const double id = dinv[j];
                const double vv = vx[j * KB + e];
                const double xp = e == 0 ? d * d : xup;
                const double rxp = e == 0 ? id * id : rxup;
                const double a = sigma > 0 ? vv * im : -(vv * im);
                double x = fma(a, vv, xp);
                const bool bad = !(x > 0.0) || !(d > 0.0);
                if (bad) {
                    if (e == 0 && !(d > 0.0)) record_failure(key, ebase, r0 + j, 2);
                    else if (e < k) record_failure(key, ebase + e, r0 + j, 1);
                    x = __longlong_as_double(0x7ff8000000000000ll);
                }
                const double rx = fast_rcp(x);
                double2 gd;
                gd.x = a * id;       // gamma
                gd.y = vv * d * rx;  // delta
                *reinterpret_cast<double2 *>(pan + 2 * (j * KB + e)) = gd;
                vt[j * KB + e] = vv;
                imx[j * KB + e] = im;
                im = im * x * rxp;
                if (e == KB - 1) rho_g[j] = d * fast_rsqrt(x);  // L_jj / L~_jj
                if (j == Db - 1) nu_g[e] = sqrt(im);
                xr = x;
                rxr = rx;
            }
#ifdef GCM_SWEEP_TRACE
            if (blockIdx.x == 0 && lane == 0) gcm_sweep_trace[tau * 4 + 1] = clock64();
#endif
        }
        __syncthreads();
        if (colthr) {
            const double *lrow = &Ls[m][0];
            double2 gd[EPT];
            double lv[EPT];
#pragma unroll
            for (int i = 0; i < EPT; ++i) {
                const int jc = min(max(tau - e0 - i, 0), Db - 1);
                gd[i] = *reinterpret_cast<const double2 *>(pan + 2 * (jc * KB + e0 + i));
                lv[i] = lrow[jc];
            }
            const int jlast = tau - (KB - 1);
            const double rl = (q == NQ - 1 && jlast >= 0 && jlast < m) ? rho_g[jlast] : 1.0;
#pragma unroll
            for (int i = 0; i < EPT; ++i) {
                const int j = tau - e0 - i;
                const double l = fma(gd[i].x, v[i], lv[i]);
                const double vn = fma(-gd[i].y, l, v[i]);
                if (j >= 0 && j < m) {
                    v[i] = vn;
                    Ls[m][j] = (q == NQ - 1 && i == EPT - 1) ? l * rl : l;
                    if (j == m - 1) vx[m * KB + e0 + i] = vn;  // column m after row m-1: row m may compute
                }
            }
#ifdef GCM_SWEEP_TRACE
            if (blockIdx.x == 0 && rel == 0) gcm_sweep_trace[tau * 4 + 3] = clock64();
#endif
        }
        __syncthreads();
    }
    // epilogue: L~_jj and V_exit (true residual v = vt / mu = vt sqrt(IM_{j-1}))
    for (int idx = t; idx < Db * k; idx += blockDim.x) {
        const int j = idx / k, e = idx % k;
        vexit[j + (int64_t)e * ldv] = vt[j * KB + e] * sqrt(imx[j * KB + e]);
    }
    if (colthr && q == 0) Ls[m][m] = Ls[m][m] / rho_g[m];  // w = L_jj / rho_j
    __syncthreads();
}

}  // namespace gcm
