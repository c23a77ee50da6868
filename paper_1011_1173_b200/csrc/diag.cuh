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

// shared-memory scratch of diag_closed (doubles)
__host__ __device__ constexpr int diag_closed_scratch(int KB) {
    return 8 * KB * KB + 3 * kD * (KB + 1) + 2 * kD;
}

// q = L_bb^{-T} Y for the block's Db rows (k right-hand sides padded to KB; padding
// columns of Y are zero).  Ls[m][i] = L(r0+i, r0+m).  One warp per right-hand side (lane
// owns rows lane, lane+32): right-looking substitution, q_i broadcast by shuffle.
// Called by ALL threads; synchronises on exit.
template <int KB, int LD>
__device__ __forceinline__ void block_trsv(const double (*Ls)[LD], const double *Y, int ldy, double *q, int ldq,
                                           int Db, double *rinv) {
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int nw = blockDim.x >> 5;
    for (int i = t; i < Db; i += blockDim.x) rinv[i] = fast_rcp(Ls[i][i]);
    __syncthreads();
    for (int e = warp; e < KB; e += nw) {
        double acc0 = lane < Db ? Y[lane * ldy + e] : 0.0;
        double acc1 = lane + 32 < Db ? Y[(lane + 32) * ldy + e] : 0.0;
        for (int i = 0; i < Db; ++i) {
            const double mine = (i < 32 ? acc0 : acc1) * rinv[i];
            const double qi = __shfl_sync(kFull, mine, i & 31);
            if (lane == (i & 31)) q[i * ldq + e] = qi;
            if (lane > i) acc0 = fma(-Ls[lane][i], qi, acc0);
            if (lane + 32 > i && lane + 32 < Db) acc1 = fma(-Ls[lane + 32][i], qi, acc1);
        }
    }
    __syncthreads();
}

// The closed-form sweep of one diagonal block.  Inputs (shared memory): Ls (original block),
// q[m*ldq + e] (= L_bb^{-T} Y), Y[m*ldy + e] (true V states at block start), both zero in the
// padding columns e >= k.  Outputs: pan (gamma/delta at 2*(j*KB+e), rho at 2*kD*KB, nu at
// 2*kD*KB + kD), L~ in Ls (upper triangle incl. diagonal), V_exit rows r0.. (vexit + e*ldv),
// failures into key.  Called by ALL threads of the CTA (>= 64 threads); synchronises on exit.
template <int KB, int LD>
__device__ void diag_closed(double (*Ls)[LD], const double *q, int ldq, const double *Y, int ldy, int Db, int k,
                            int sigma, int64_t r0, double *pan, double *vexit, int64_t ldv,
                            unsigned long long *key, int64_t ebase, double *scratch) {
    static_assert(KB == 4 || KB == 8 || KB == 16 || KB == 32, "rank bucket");
    constexpr int LY = KB + 1;
    double *S8 = scratch;              // [8][KB][KB]: exclusive prefix Grams at rows 0, 8, .., 56
    double *yv = S8 + 8 * KB * KB;     // [kD][LY]: y_{j,e}
    double *xs = yv + kD * LY;         // [kD][LY]: x_{j,e}
    double *mu = xs + kD * LY;         // [kD][LY]: w_{j,e-1}/w_{j,e}, then mu_{j-1,e}
    double *dj = mu + kD * LY;         // [kD]: L_jj (original)
    double *rj = dj + kD;              // [kD]: 1/L_jj
    double *rho_g = pan + 2 * kD * KB;
    double *nu_g = rho_g + kD;
    const int t = threadIdx.x, nt = blockDim.x;
    const double sg = sigma > 0 ? 1.0 : -1.0;

    // A. Grams of 8-row groups, then their exclusive prefix
    for (int o = t; o < 8 * KB * KB; o += nt) {
        const int g = o / (KB * KB), i = (o / KB) % KB, c = o % KB;
        double s = 0.0;
        for (int r = 8 * g; r < 8 * g + 8 && r < Db; ++r) s = fma(q[r * ldq + i], q[r * ldq + c], s);
        S8[o] = s;
    }
    for (int j = t; j < Db; j += nt) {
        const double d = Ls[j][j];
        dj[j] = d;
        rj[j] = fast_rcp(d);
    }
    __syncthreads();
    for (int o = t; o < KB * KB; o += nt) {
        double run = 0.0;
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            const double b = S8[g * KB * KB + o];
            S8[g * KB * KB + o] = run;
            run += b;
        }
    }
    __syncthreads();

    // B. per row j: y_j = chol_lower(I + sigma S_j)^{-1} (L_jj q_j), KB lanes per row
    //    (lane i holds row i of the KB x KB matrix; Gaussian elimination by shuffles within
    //    the KB-lane segment: H = U' D U'^T, y = D^{-1/2} U'^{-1} z)
    {
        constexpr int G = 32 / (KB < 32 ? KB : 32);  // rows per warp
        const int warp = t >> 5, lane = t & 31, nw = nt >> 5;
        const int i = lane % KB, grp = lane / KB;
        for (int base = warp * G; base < Db; base += nw * G) {
            const int j = base + grp;
            const bool act = j < Db;
            const int jj = act ? j : 0;
            double a[KB];
            const int g8 = jj >> 3;
#pragma unroll
            for (int c = 0; c < KB; ++c) a[c] = S8[(g8 * KB + i) * KB + c];
            for (int r = 8 * g8; r < jj; ++r) {
                const double qi = q[r * ldq + i];
#pragma unroll
                for (int c = 0; c < KB; ++c) a[c] = fma(qi, q[r * ldq + c], a[c]);
            }
#pragma unroll
            for (int c = 0; c < KB; ++c) a[c] = (i == c ? 1.0 : 0.0) + sg * a[c];
            double z = dj[jj] * q[jj * ldq + i];
#pragma unroll
            for (int c = 0; c < KB - 1; ++c) {
                const bool below = i > c;
                const double f = a[c] * fast_rcp(__shfl_sync(kFull, a[c], c, KB));
#pragma unroll
                for (int c2 = c + 1; c2 < KB; ++c2) {
                    const double x = __shfl_sync(kFull, a[c2], c, KB);
                    if (below) a[c2] = fma(-f, x, a[c2]);
                }
                const double zc = __shfl_sync(kFull, z, c, KB);
                if (below) z = fma(-f, zc, z);
            }
            double di = 0.0;
#pragma unroll
            for (int c = 0; c < KB; ++c)
                if (c == i) di = a[c];
            // a non-positive pivot (an indefinite leading block: an earlier row failed) gives NaN
            const double y = di > 0.0 ? z * fast_rsqrt(di) : __longlong_as_double(0x7ff8000000000000ll);
            if (act) yv[jj * LY + i] = y;
        }
    }
    __syncthreads();

    // C. row Compute (PAPER.md 45-48) from y: x_{j,e}, the ratio w_{e-1}/w_e, failures,
    //    L~_jj, rho_j and the V_exit row
    for (int j = t; j < Db; j += nt) {
        double d = dj[j];
        if (!(d > 0.0)) {
            record_failure(key, ebase, r0 + j, 2);
            d = __longlong_as_double(0x7ff8000000000000ll);
        }
        double x = d * d;
        bool failed = false;
#pragma unroll
        for (int e = 0; e < KB; ++e) {
            const double v = yv[j * LY + e];
            double xn = fma(sg * v, v, x);
            if (!(xn > 0.0) && !failed) {
                if (e < k && d == d) record_failure(key, ebase + e, r0 + j, 1);
                failed = true;
            }
            if (failed) xn = __longlong_as_double(0x7ff8000000000000ll);
            const double ratio = sqrt(x) * fast_rsqrt(xn);  // w_{e-1} / w_e = 1/c
            xs[j * LY + e] = xn;
            mu[j * LY + e] = ratio;
            if (e < k) vexit[j + (int64_t)e * ldv] = v;
            x = xn;
        }
        rho_g[j] = d * fast_rsqrt(x);  // L_jj / L~_jj
        Ls[j][j] = sqrt(x);            // L~_jj
    }
    __syncthreads();
    // mu_{j-1,e} (exclusive prefix product over rows of 1/c) and nu_e = 1/mu_{last,e}
    for (int e = t; e < KB; e += nt) {
        double m = 1.0;
        for (int j = 0; j < Db; ++j) {
            const double r = mu[j * LY + e];
            mu[j * LY + e] = m;
            m *= r;
        }
        nu_g[e] = fast_rcp(m);
    }
    __syncthreads();
    // D. panel: gamma = sigma y / (mu L_jj), delta = mu y L_jj / x (rot.cuh, scaled Apply)
    for (int o = t; o < Db * KB; o += nt) {
        const int j = o / KB, e = o % KB;
        const double v = yv[j * LY + e], m = mu[j * LY + e], d = dj[j];
        double2 gd;
        gd.x = sg * v * fast_rcp(m) * rj[j];
        gd.y = m * v * d * fast_rcp(xs[j * LY + e]);
        *reinterpret_cast<double2 *>(pan + 2 * (j * KB + e)) = gd;
    }
    __syncthreads();
    // E. the block's own triangle: column m from its block-start state Y_m through rows j < m
    for (int m = 1 + t; m < Db; m += nt) {
        double v[KB];
#pragma unroll
        for (int e = 0; e < KB; ++e) v[e] = Y[m * ldy + e];
        const double2 *cs = reinterpret_cast<const double2 *>(pan);
        for (int j = 0; j < m; ++j) Ls[m][j] = apply_row<KB>(Ls[m][j], v, cs + j * KB, rho_g[j], KB);
    }
    __syncthreads();
}

}  // namespace gcm
