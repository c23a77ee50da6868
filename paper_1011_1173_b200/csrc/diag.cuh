// diag.cuh -- the diagonal block of the sweep in closed form (DESIGN.md "closed-form
// diagonal block", reading R20).
//
// The paper's sweep (CholeskyModifyA, PAPER.md 24-30) visits the rows of a diagonal block
// one after another: row j's Compute (PAPER.md 44-49) needs column j's V state rotated by
// every earlier row, so a D-row block is a chain of D + k - 1 dependent Compute links
// (rot.cuh wave_sweep: one tick each, two CTA barriers per tick).  That V state has a
// closed form.  With Y = the columns' V states at block start (true values) and
// q = L_bb^{-T} Y (q_m = row m, k-vector), the block is the paper's sweep of the small
// problem [L_bb; Y^T], so (the blocked path's derivation, one level down)
//
//   y_j := V state of column j entering row j = chol_lower(I + sigma S_j)^{-1} (L_jj q_j),
//   S_j  = sum_{i < j} q_i q_i^T   (k x k, exclusive prefix over the block's rows),
//
// which is exact in real arithmetic.  Every row's V state, hence every row's rotations
// (c, s) of PAPER.md 45-48, is then independent of the other rows:
//   x_{j,-1} = L_jj^2,  x_{j,e} = x_{j,e-1} + sigma y_{j,e}^2,  w = sqrt(x),
//   c_{j,e} = w_{j,e}/w_{j,e-1},  s_{j,e} = y_{j,e}/w_{j,e-1},  L~_jj = w_{j,k-1},
// and y_j is exactly the V_exit row the sweep writes back (PAPER.md 105).  The panel is
// emitted in the scaled 2-FMA form rot.cuh documents (gamma, delta, rho, nu with the
// running scale mu_{j,e} = prod_{rows j' <= j} 1/c_{j',e}, a prefix product over rows),
// and the block's own upper triangle gets the ordinary Apply (PAPER.md 52-54) from Y.
//
// Cost: one small Cholesky per row (KB lanes per row, all rows in parallel), a prefix
// product over 64 rows, and the triangle Apply (a D + k wavefront of 2-FMA links) --
// no CTA barrier per row.  Failures: row j reports !(L_jj > 0) (code 2) or the first e
// with !(x_{j,e} > 0) (code 1); a failing leading block of I + sigma S_j only happens
// after an earlier row failed at the same e, so the lexicographic minimum is the
// sequential sweep's report (R5, R6).
#pragma once
#include "rot.cuh"

namespace gcm {

#ifdef GCM_BT_TRACE  // sub-step clocks of diag_closed (CTA 0, tools/batched_trace.py)
__device__ long long g_dc_trace[16 * 8];
#define DC_MARK(slot)                                                                        \
    do {                                                                                     \
        if (threadIdx.x == 0 && blockIdx.x == 0 && r0 / kD < 16) g_dc_trace[(r0 / kD) * 8 + (slot)] = clock64(); \
    } while (0)
#else
#define DC_MARK(slot) ((void)0)
#endif

// shared-memory scratch of diag_closed (doubles)
__host__ __device__ constexpr int diag_closed_scratch(int KB) { return 8 * KB * (KB + 1) + 2 * kD * (KB + 1) + 3 * kD; }

// q = L_bb^{-T} Y for the block's Db rows (k right-hand sides padded to KB; padding
// columns of Y are zero), IN PLACE: on entry Y[m*ldy + e], on exit q there.  Ls[m][i] =
// L(r0+i, r0+m).  One warp per right-hand side; lane l owns the consecutive rows 2l, 2l+1,
// so each step resolves a row PAIR inside one lane (q_{2l} = a_{2l}/L, q_{2l+1} from it
// with one more FMA) and broadcasts both by shuffle: 32 dependent steps of ~FMA + FMA +
// SHFL + 2 FMA instead of 64 of MUL + SHFL + FMA.  Called by ALL threads; synchronises.
template <int KB, int LD, int RPW = 1>
__device__ __forceinline__ void block_trsv(const double (*Ls)[LD], double *Y, int ldy, int Db, double *) {
    // RPW right-hand sides per warp: the L entries a lane loads feed all of them (a CTA with
    // many warps per block, e.g. dsolve's 32, would otherwise re-load every entry per warp and
    // saturate the shared-memory pipe)
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int nw = blockDim.x >> 5;
    const int m0 = 2 * lane, m1 = 2 * lane + 1;
    const bool v0 = m0 < Db, v1 = m1 < Db;
    // own rows: 1/L_mm and the in-pair coupling L(m0, m1)/L(m1, m1)
    const double i0 = v0 ? fast_rcp(Ls[m0][m0]) : 0.0;
    const double i1 = v1 ? fast_rcp(Ls[m1][m1]) : 0.0;
    const double c1 = v1 ? Ls[m1][m0] * i1 : 0.0;
    const int np = (Db + 1) >> 1;
    // the lane's L entries of the next pair are loaded a step ahead (off the shuffle chain);
    // entries past the block (Db < 64) or in the strictly lower part are read but masked out
    const int mr0 = v0 ? m0 : 0, mr1 = v1 ? m1 : 0;
    for (int eb = warp * RPW; eb < KB; eb += nw * RPW) {
        double a0[RPW], a1[RPW];
#pragma unroll
        for (int w = 0; w < RPW; ++w) {
            const int e = eb + w;
            a0[w] = (v0 && e < KB) ? Y[m0 * ldy + e] : 0.0;
            a1[w] = (v1 && e < KB) ? Y[m1 * ldy + e] : 0.0;
        }
        double l00 = Ls[mr0][0], l01 = Ls[mr0][1], l10 = Ls[mr1][0], l11 = Ls[mr1][1];
        for (int p = 0; p < np; ++p) {
            const int in = 2 * p + 2 < kD ? 2 * p + 2 : 0;
            const double n00 = Ls[mr0][in], n01 = Ls[mr0][in + 1], n10 = Ls[mr1][in], n11 = Ls[mr1][in + 1];
            const bool two = 2 * p + 1 < Db;  // odd Db: the last pair has one row
#pragma unroll
            for (int w = 0; w < RPW; ++w) {
                const double q0l = a0[w] * i0;
                const double q1l = fma(-c1, q0l, a1[w] * i1);
                const double q0 = __shfl_sync(kFull, q0l, p);
                double q1 = __shfl_sync(kFull, q1l, p);
                if (!two) q1 = 0.0;
                if (lane == p && eb + w < KB) {
                    Y[m0 * ldy + eb + w] = q0;
                    if (v1) Y[m1 * ldy + eb + w] = q1;
                }
                if (lane > p) {  // rows of later lanes: a_m -= L(2p, m) q_{2p} + L(2p+1, m) q_{2p+1}
                    a0[w] = fma(-l01, q1, fma(-l00, q0, a0[w]));
                    a1[w] = fma(-l11, q1, fma(-l10, q0, a1[w]));
                }
            }
            l00 = n00;
            l01 = n01;
            l10 = n10;
            l11 = n11;
        }
    }
    __syncthreads();
}

// The closed-form sweep of one diagonal block, rows part.  Inputs (shared memory): Ls
// (original block; only its diagonal is read here), q[m*ldq + e] (= L_bb^{-T} Y, zero in
// the padding columns e >= k).  Outputs: pan (gamma/delta at 2*(j*KB+e), rho at 2*kD*KB, nu
// at 2*kD*KB + kD), L~_jj on the diagonal of Ls, V_exit rows r0.. (vexit + e*ldv), failures
// into key.  The block's own upper triangle is then rotated by diag_triangle (each column
// from its block-start V state).  Called by ALL threads of the CTA; synchronises on exit.
template <int KB, int LD>
__device__ void diag_closed(double (*Ls)[LD], const double *q, int ldq, int Db, int k, int sigma, int64_t r0,
                            double *pan, double *vexit, int64_t ldv, unsigned long long *key, int64_t ebase,
                            double *scratch) {
    static_assert(KB == 4 || KB == 8 || KB == 16 || KB == 32, "rank bucket");
    constexpr int LY = KB + 1;
    double *S8 = scratch;                 // [8][KB][KB+1]: exclusive prefix Grams at rows 0, 8, .., 56
    double *yv = S8 + 8 * KB * (KB + 1);  // [kD][LY]: y_{j,e}
    double *mu = yv + kD * LY;         // [kD][LY]: w_{j,e-1}/w_{j,e}, then mu_{j-1,e}
    double *dj = mu + kD * LY;         // [kD]: L_jj (original)
    double *rj = dj + kD;              // [kD]: 1/L_jj
    double *rho_g = pan + 2 * kD * KB;
    double *nu_g = rho_g + kD;
    const int t = threadIdx.x, nt = blockDim.x;
    const double sg = sigma > 0 ? 1.0 : -1.0;
    DC_MARK(0);

    // A. Grams of 8-row groups, then their exclusive prefix
    // (row stride KB + 1: a row problem's KB lanes read one column of S8 without bank conflicts)
    for (int o = t; o < 8 * KB * KB; o += nt) {
        const int g = o / (KB * KB), i = (o / KB) % KB, c = o % KB;
        double s = 0.0;
        for (int r = 8 * g; r < 8 * g + 8 && r < Db; ++r) s = fma(q[r * ldq + i], q[r * ldq + c], s);
        S8[(g * KB + i) * (KB + 1) + c] = s;
    }
    for (int j = t; j < Db; j += nt) {
        const double d = Ls[j][j];
        dj[j] = d;
        rj[j] = fast_rcp(d);
    }
    __syncthreads();
    for (int o = t; o < KB * KB; o += nt) {
        const int oo = (o / KB) * (KB + 1) + o % KB;
        double run = 0.0;
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            const double b = S8[g * KB * (KB + 1) + oo];
            S8[g * KB * (KB + 1) + oo] = run;
            run += b;
        }
    }
    __syncthreads();
    DC_MARK(1);

    // B. per row j: y_j = chol_lower(I + sigma S_j)^{-1} (L_jj q_j).
    //    KB <= 8: one thread per row holds the lower triangle of H_j = I + sigma S_j in
    //    registers (KB(KB+1)/2 values) and runs the textbook Cholesky + forward substitution
    //    (no shuffles, no barriers).  KB >= 16: KB lanes per row (lane i holds row i of H_j;
    //    Gaussian elimination by shuffles within the KB-lane segment: H = U' D U'^T,
    //    y = D^{-1/2} U'^{-1} z).  In both, a column is only combined with the columns before
    //    it, so a NaN column cannot reach earlier columns (R5, R6).
#ifndef GCM_DIAG_THREAD_CHOL
#define GCM_DIAG_THREAD_CHOL 0  // per-thread KB x KB Cholesky for KB <= this (register-heavy; 0 = shuffle elimination for all)
#endif
    if constexpr (KB <= GCM_DIAG_THREAD_CHOL) {
        for (int j = t; j < Db; j += nt) {
            double h[KB * (KB + 1) / 2];  // packed lower triangle, row-major: (i, c) at i(i+1)/2 + c
            const int g8 = j >> 3;
#pragma unroll
            for (int i = 0; i < KB; ++i)
#pragma unroll
                for (int c = 0; c <= i; ++c) h[i * (i + 1) / 2 + c] = S8[(g8 * KB + i) * (KB + 1) + c];
            for (int r = 8 * g8; r < j; ++r) {
                double qr[KB];
#pragma unroll
                for (int i = 0; i < KB; ++i) qr[i] = q[r * ldq + i];
#pragma unroll
                for (int i = 0; i < KB; ++i)
#pragma unroll
                    for (int c = 0; c <= i; ++c) h[i * (i + 1) / 2 + c] = fma(qr[i], qr[c], h[i * (i + 1) / 2 + c]);
            }
            double z[KB];
            const double d = dj[j];
#pragma unroll
            for (int i = 0; i < KB; ++i) {
#pragma unroll
                for (int c = 0; c <= i; ++c) h[i * (i + 1) / 2 + c] = (i == c ? 1.0 : 0.0) + sg * h[i * (i + 1) / 2 + c];
                z[i] = d * q[j * ldq + i];
            }
            // H = C C^T (C lower), y = C^{-1} z, column by column (right-looking)
#pragma unroll
            for (int c = 0; c < KB; ++c) {
                const double piv = h[c * (c + 1) / 2 + c];
                const double rs = piv > 0.0 ? fast_rsqrt(piv) : __longlong_as_double(0x7ff8000000000000ll);
                z[c] *= rs;
#pragma unroll
                for (int i = c + 1; i < KB; ++i) {
                    h[i * (i + 1) / 2 + c] *= rs;  // C(i, c)
                    z[i] = fma(-h[i * (i + 1) / 2 + c], z[c], z[i]);
                }
#pragma unroll
                for (int i = c + 1; i < KB; ++i)
#pragma unroll
                    for (int c2 = c + 1; c2 <= i; ++c2)
                        h[i * (i + 1) / 2 + c2] = fma(-h[i * (i + 1) / 2 + c], h[c2 * (c2 + 1) / 2 + c],
                                                      h[i * (i + 1) / 2 + c2]);
            }
#pragma unroll
            for (int i = 0; i < KB; ++i) yv[j * LY + i] = z[i];
        }
    } else {
        // RPL rows of H_j per lane (LPP = KB / RPL lanes per row problem, rows li + LPP u):
        // each pivot-row shuffle feeds RPL rows, so the shuffles -- the throughput limit of
        // this step when every warp eliminates -- drop by RPL
        constexpr int RPL = KB >= 16 ? (KB >= 32 ? 2 : 4) : (KB >= 8 ? 2 : 1);
        constexpr int LPP = KB / RPL;
        constexpr int PPW = 32 / LPP;  // row problems per warp
        const int warp = t >> 5, lane = t & 31, nw = nt >> 5;
        const int li = lane % LPP, grp = lane / LPP;
        for (int base = warp * PPW; base < Db; base += nw * PPW) {
            const int j = base + grp;
            const bool act = j < Db;
            const int jj = act ? j : 0;
            double a[RPL][KB], z[RPL];
            const int g8 = jj >> 3;
#pragma unroll
            for (int u = 0; u < RPL; ++u)
#pragma unroll
                for (int c = 0; c < KB; ++c) a[u][c] = S8[(g8 * KB + li + LPP * u) * (KB + 1) + c];
            for (int r = 8 * g8; r < jj; ++r) {
                double qr[KB];
#pragma unroll
                for (int c = 0; c < KB; ++c) qr[c] = q[r * ldq + c];
#pragma unroll
                for (int u = 0; u < RPL; ++u) {
                    const double qi = q[r * ldq + li + LPP * u];
#pragma unroll
                    for (int c = 0; c < KB; ++c) a[u][c] = fma(qi, qr[c], a[u][c]);
                }
            }
#pragma unroll
            for (int u = 0; u < RPL; ++u) {
                const int i = li + LPP * u;
#pragma unroll
                for (int c = 0; c < KB; ++c) a[u][c] = (i == c ? 1.0 : 0.0) + sg * a[u][c];
                z[u] = dj[jj] * q[jj * ldq + i];
            }
#pragma unroll
            for (int c = 0; c < KB - 1; ++c) {
                const int pl = c % LPP, pu = c / LPP;  // the pivot row's lane and slot
                double f[RPL];
                const double rp = fast_rcp(__shfl_sync(kFull, a[pu][c], pl, LPP));
#pragma unroll
                for (int u = 0; u < RPL; ++u) f[u] = a[u][c] * rp;
#pragma unroll
                for (int c2 = c + 1; c2 < KB; ++c2) {
                    const double x = __shfl_sync(kFull, a[pu][c2], pl, LPP);
#pragma unroll
                    for (int u = 0; u < RPL; ++u)
                        if (li + LPP * u > c) a[u][c2] = fma(-f[u], x, a[u][c2]);
                }
                const double zc = __shfl_sync(kFull, z[pu], pl, LPP);
#pragma unroll
                for (int u = 0; u < RPL; ++u)
                    if (li + LPP * u > c) z[u] = fma(-f[u], zc, z[u]);
            }
#pragma unroll
            for (int u = 0; u < RPL; ++u) {
                const int i = li + LPP * u;
                double di = 0.0;
#pragma unroll
                for (int c = 0; c < KB; ++c)
                    if (c == i) di = a[u][c];
                // a non-positive pivot (an indefinite leading block: an earlier row failed) gives NaN
                const double y = di > 0.0 ? z[u] * fast_rsqrt(di) : __longlong_as_double(0x7ff8000000000000ll);
                if (act) yv[jj * LY + i] = y;
            }
        }
    }
    __syncthreads();
    DC_MARK(2);

    // C. row Compute (PAPER.md 45-48) from y: x_{j,e}, the ratio w_{e-1}/w_e = 1/c, failures,
    //    L~_jj, rho_j, the V_exit row, and the unscaled panel entries sigma y / L_jj and
    //    y L_jj / x (the mu scales are applied in D)
    for (int j = t; j < Db; j += nt) {
        double d = dj[j];
        if (!(d > 0.0)) {
            record_failure(key, ebase, r0 + j, 2);
            d = __longlong_as_double(0x7ff8000000000000ll);
        }
        const double id = rj[j];
        double v[KB], x[KB + 1];
#pragma unroll
        for (int e = 0; e < KB; ++e) v[e] = yv[j * LY + e];
        x[0] = d * d;
#pragma unroll
        for (int e = 0; e < KB; ++e) x[e + 1] = fma(sg * v[e], v[e], x[e]);  // the only chain
        int bad = KB;  // first e with !(x_{j,e} > 0) (NaN included); later ones NaN as well
#pragma unroll
        for (int e = KB - 1; e >= 0; --e)
            if (!(x[e + 1] > 0.0)) bad = e;
        if (bad < k && d == d) record_failure(key, ebase + bad, r0 + j, 1);
#pragma unroll
        for (int e = 0; e < KB; ++e) {
            const double xn = e >= bad ? __longlong_as_double(0x7ff8000000000000ll) : x[e + 1];
            const double rx = fast_rcp(xn);
            const double rs0 = fast_rsqrt(x[e]);
            mu[j * LY + e] = x[e] * rs0 * fast_rsqrt(xn);  // w_{e-1} / w_e = 1/c_{j,e}
            double2 gd;
            gd.x = sg * v[e] * id;
            gd.y = v[e] * d * rx;
            *reinterpret_cast<double2 *>(pan + 2 * (j * KB + e)) = gd;
            if (e < k) vexit[j + (int64_t)e * ldv] = v[e];
        }
        const double xl = bad < KB ? __longlong_as_double(0x7ff8000000000000ll) : x[KB];
        rho_g[j] = d * fast_rsqrt(xl);  // L_jj / L~_jj
        Ls[j][j] = sqrt(xl);            // L~_jj
    }
    __syncthreads();
    DC_MARK(3);
    // mu_{j-1,e}: exclusive prefix product over rows of 1/c, nu_e = 1/mu_last.  Eight
    // threads per e: each multiplies its 8-row segment (loads in flight together), the
    // segment products are scanned by shuffles within the 8 lanes, then applied.
    for (int o = t; o < 8 * KB; o += nt) {
        const int e = o >> 3, sgm = o & 7;  // 8 consecutive lanes per e
        double r[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int j = 8 * sgm + u;
            r[u] = j < Db ? mu[j * LY + e] : 1.0;
        }
        double p = 1.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) p *= r[u];
        double pre = p;  // inclusive scan of the segment products over the 8 lanes
#pragma unroll
        for (int off = 1; off < 8; off <<= 1) {
            const double y = __shfl_up_sync(kFull, pre, off, 8);
            if (sgm >= off) pre *= y;
        }
        double m = __shfl_up_sync(kFull, pre, 1, 8);  // exclusive
        if (sgm == 0) m = 1.0;
        if (sgm == 7) nu_g[e] = fast_rcp(pre);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int j = 8 * sgm + u;
            if (j < Db) mu[j * LY + e] = m;
            m *= r[u];
        }
    }
    __syncthreads();
    DC_MARK(4);
    // D. scaled panel (rot.cuh): gamma = sigma y / (mu L_jj), delta = mu y L_jj / x
    for (int o = t; o < Db * KB; o += nt) {
        const int j = o / KB, e = o % KB;
        const double m = mu[j * LY + e];
        double2 *gd = reinterpret_cast<double2 *>(pan + 2 * (j * KB + e));
        double2 g = *gd;
        g.x *= fast_rcp(m);
        g.y *= m;
        *gd = g;
    }
    __syncthreads();
    DC_MARK(5);
}

// The block's own upper triangle, column m (0 < m < Db) from its block-start V state v
// (TRUE values) through the rows j < m of the block's panel (scaled 2-FMA Apply, PAPER.md
// 52-54).  v is consumed (the column's V state after its own block is not needed).
template <int KB, int LD>
__device__ __forceinline__ void diag_triangle(double (*Ls)[LD], int m, double (&v)[KB], const double *pan) {
    const double2 *cs = reinterpret_cast<const double2 *>(pan);
    const double *rho = pan + 2 * kD * KB;
    // rows in groups of RG held in registers, (row, e) loops unrolled: row j+1's rotation e
    // only waits for row j's rotation e, so the rows pipeline (a wavefront of RG + KB links)
#ifndef GCM_TRI_RG
#define GCM_TRI_RG 4
#endif
    constexpr int RG = GCM_TRI_RG;
    int j0 = 0;
    for (; j0 + RG <= m; j0 += RG) {
        double l[RG];
#pragma unroll
        for (int u = 0; u < RG; ++u) l[u] = Ls[m][j0 + u];
#pragma unroll
        for (int u = 0; u < RG; ++u) {
            const double2 *g = cs + (j0 + u) * KB;
#pragma unroll
            for (int e = 0; e < KB; ++e) {
                const double2 gd = g[e];
                l[u] = fma(gd.x, v[e], l[u]);
                v[e] = fma(-gd.y, l[u], v[e]);
            }
        }
#pragma unroll
        for (int u = 0; u < RG; ++u) Ls[m][j0 + u] = l[u] * rho[j0 + u];
    }
    for (int j = j0; j < m; ++j) Ls[m][j] = apply_row<KB>(Ls[m][j], v, cs + j * KB, rho[j], KB);
}

}  // namespace gcm
