// panel.cu -- the column-sharded path (gcm_modify_dist, gcm_modify_dist_virtual) and its
// one-rank instance GCM_ALGO_PANEL (large single factors).
//
// The blocked single-factor path (blocked.cu) keeps the whole triangular solve P = L^{-T} V
// inside one persistent kernel whose helpers own every column strip; at n = 1e5 its helpers
// are throughput-bound and it cannot be split over GPUs.  This path runs the same method
// (P, prefix Grams G_b, U_b = chol_lower(I + sigma G_b), Apply tiles seeded
// by the checkpointed residuals U_b^{-1} r) as a right-looking block algorithm over column
// blocks of width nb, which shards by columns:
//
//   for every column block g (rows/columns [g nb, (g+1) nb)):
//     owner (rank g mod R):  P rows of block g = L_gg^{-T} r_g  (dsolve_kernel: 64-row
//                            sub-blocks, in-block residual updates + their checkpoints),
//                            written straight into EVERY rank's replicated P buffer
//                            (device-initiated puts; PEER mode adds a system-scope flag)
//                            -- or one ncclBroadcast in NCCL mode;
//     every rank:            residuals of its strips right of block g  -= L_{g,s}^T P_g,
//                            writing the Apply checkpoint of each 64-row tile (pupdate_kernel);
//   every rank: G_b prefix Grams from the replicated P (pgram/pscan), the diagonal sweeps of
//     its own 64-row diagonal blocks (bdiag_body: PAPER.md 24-30 Compute/Apply on the block,
//     seeded by U_b^{-1} L_bb^T P_b), then coefficient panels + U_b^{-1} to every rank;
//   every rank: the Apply (PAPER.md 52-54) of every panel to its own tiles (btma_body over a
//     tensor map of the LOCAL columns, 4 strips per CTA; ptile_kernel for the tiles of the
//     diagonal column block).
//
// The only exchanges are P (n k doubles per call, every owner's rows once) and the panels
// (~(2*64*k + 64 + k) doubles per 64-row block), both written by the producing kernel
// itself.  Layout: 1-D block-cyclic over columns (gcm.h), V rows follow their columns.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <tuple>
#include <vector>

#include "bparts.cuh"
#include "diag.cuh"
#include "internal.h"
#include "tma.cuh"

#ifdef GCM_WITH_NCCL
#include <nccl.h>
#endif

struct gcm_comm {
#ifdef GCM_WITH_NCCL
    ncclComm_t nc = nullptr;
#endif
    int rank = 0;
    int nranks = 1;
    int peer = 0;          // 1: device-initiated exchange through an IPC window (gcm_comm_set_peer)
    unsigned epoch = 0;    // peer mode: pass counter (identical on every rank)
    char *win = nullptr;   // this rank's window: [P | panels | U | flags | counter]
    size_t win_bytes = 0;
    char *peers[8] = {};   // every rank's window mapped into this process (peers[rank] = win)
    size_t offP = 0, offPan = 0, offU = 0, offFlag = 0, offCtr = 0;
};

namespace gcm {
namespace {

constexpr int kMaxRanks = 8;  // virtual ranks / peers a kernel writes to
constexpr int kPT = 256;      // pupdate threads
constexpr int kDsT = 512;     // dsolve threads (16 warps: 8 row tiles x 2 column groups)
constexpr int kPassK = 32;    // update columns per pass (k > 32: sequential passes, R3)

// -------------------------------------------------------------------------- layout (host)
int64_t local_cols(int64_t n, int64_t nb, int R, int r) {
    if (n < 0 || nb <= 0 || R <= 0 || r < 0 || r >= R) return -1;
    const int64_t nblk = (n + nb - 1) / nb;
    int64_t cols = 0;
    for (int64_t g = r; g < nblk; g += R) cols += std::min<int64_t>(nb, n - g * nb);
    return cols;
}
int64_t global_col(int64_t nb, int R, int r, int64_t lc) {
    const int64_t lb = lc / nb;
    return (lb * R + r) * nb + lc % nb;
}

// One rank's view: its factor columns, V rows, and workspace carve-up.
struct Plan {
    int64_t n, nb, nloc;
    int R, r, k, KB;
    int NB64, NBc, nsl;
    std::vector<int> gstrip;                // global 64-column strip of local strip sl
    std::vector<int64_t> chkoff;            // first checkpoint tile of local strip sl
    int64_t nchk = 0;
    std::vector<int> dl_b;                  // local diagonal 64-row blocks
    std::vector<int64_t> dl_lc;             //   and their first local column
    std::vector<int2> full;                 // TMA Apply items (b, first local strip of 4)
    std::vector<int> full_off, tiles_off;   // one rank: items sorted by b; row block b's are [off[b], off[b+1])
    std::vector<int2> tiles;                // single-tile Apply items (b, local strip)
    int64_t sb;                             // solve-block height (<= nb, dsolve's shared-memory cap)
    int NSB;                                // solve blocks
    std::vector<int> first_strip_after;     // per solve block: first local strip right of it
    unsigned char *img = nullptr;           // pinned host image of the device layout arrays (gstrip ..
    size_t img_bytes = 0;                   //   tiles at their carve offsets): one async upload per call
};

// rows of one dsolve launch: its residuals live in shared memory (kDsMaxRows x KB doubles)
inline int64_t solve_block_rows(int64_t nb, int KB) {
    const int64_t cap = KB <= 16 ? 512 : 256;
    return std::min<int64_t>(nb, cap);
}

Plan make_plan(int64_t n, int64_t nb, int R, int r, int k, bool tma_groups) {
    Plan p;
    p.n = n;
    p.nb = nb;
    p.R = R;
    p.r = r;
    p.k = k;
    p.KB = k <= 4 ? 4 : k <= 8 ? 8 : k <= 16 ? 16 : 32;
    p.nloc = local_cols(n, nb, R, r);
    p.NB64 = (int)((n + kD - 1) / kD);
    p.NBc = (int)((n + nb - 1) / nb);
    p.nsl = (int)((p.nloc + kD - 1) / kD);
    p.gstrip.resize(p.nsl);
    p.chkoff.resize(p.nsl);
    for (int sl = 0; sl < p.nsl; ++sl) {
        p.gstrip[sl] = (int)(global_col(nb, R, r, (int64_t)sl * kD) / kD);
        p.chkoff[sl] = p.nchk;
        p.nchk += p.gstrip[sl];  // tiles (b, s), b < s
    }
    for (int sl = 0; sl < p.nsl; ++sl) {  // a strip's diagonal block b = its global strip
        p.dl_b.push_back(p.gstrip[sl]);
        p.dl_lc.push_back((int64_t)sl * kD);
    }
    p.sb = solve_block_rows(nb, p.KB);
    p.NSB = (int)((n + p.sb - 1) / p.sb);
    p.first_strip_after.resize(p.NSB);
    for (int g = 0; g < p.NSB; ++g) {
        const int64_t end = std::min<int64_t>(n, (int64_t)(g + 1) * p.sb);
        int sl = 0;
        while (sl < p.nsl && (int64_t)p.gstrip[sl] * kD < end) ++sl;
        p.first_strip_after[g] = sl;
    }
    // Apply items: groups of 4 local strips inside one local column block (globally
    // contiguous when nb is a multiple of 256): a TMA item while all 4 are right of row
    // block b, else per-strip tiles for the strips that are
    const int spb = (int)(nb / kD);  // strips per column block
    const bool grp = tma_groups && nb % 256 == 0;
    for (int lb0 = 0; lb0 < p.nsl; lb0 += spb) {
        const int lb_end = std::min(p.nsl, lb0 + spb);
        for (int sl0 = lb0; sl0 < lb_end; sl0 += 4) {
            const int cnt = std::min(4, lb_end - sl0);
            const int last = p.gstrip[sl0 + cnt - 1];
            for (int b = 0; b < last; ++b) {
                if (grp && p.gstrip[sl0] > b) {
                    p.full.push_back(make_int2(b, sl0));
                } else {
                    for (int q = 0; q < cnt; ++q)
                        if (p.gstrip[sl0 + q] > b) p.tiles.push_back(make_int2(b, sl0 + q));
                }
            }
        }
    }
    if (R == 1) {  // the persistent chain's overlapped Apply takes the items row block by row block
        auto by_b = [](const int2 &x, const int2 &y) { return x.x < y.x || (x.x == y.x && x.y < y.y); };
        std::sort(p.full.begin(), p.full.end(), by_b);
        std::sort(p.tiles.begin(), p.tiles.end(), by_b);
        auto offsets = [&](const std::vector<int2> &v, std::vector<int> &off) {
            off.assign(p.NB64 + 1, 0);
            for (const int2 &x : v) ++off[x.x + 1];
            for (int b = 0; b < p.NB64; ++b) off[b + 1] += off[b];
        };
        offsets(p.full, p.full_off);
        offsets(p.tiles, p.tiles_off);
    }
    return p;
}

// workspace carve-up of one rank (byte offsets)
// GCM_HOST_TRACE=1: host timestamps of the panel path's enqueue steps (stderr, one line per call)
struct HostTrace {
    bool on = std::getenv("GCM_HOST_TRACE") != nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    char line[512];
    int len = 0;
    void mark(const char *what) {
        if (!on || len > 440) return;
        const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
        len += std::snprintf(line + len, sizeof(line) - len, " %s %.1f", what, us);
    }
    ~HostTrace() {
        if (on) std::fprintf(stderr, "host_trace:%s\n", line);
    }
};
thread_local HostTrace *g_ht = nullptr;
inline void ht_mark(const char *what) {
    if (g_ht) g_ht->mark(what);
}

// per-device one-time host setup (function attributes, occupancy queries): each of those calls
// costs microseconds of host time on every modify call otherwise, before the first kernel
struct DevOnce {
    std::atomic<unsigned long long> mask{0};
    bool first(int dev) const { return !(mask.load(std::memory_order_acquire) & (1ull << (dev & 63))); }
    void done(int dev) { mask.fetch_or(1ull << (dev & 63), std::memory_order_release); }
};
inline int cur_device() {
    int dev = 0;
    return cudaGetDevice(&dev) == cudaSuccess ? dev : 0;
}

struct Carve {
    size_t P, res, chk, Winv, Q, G, U, panels, key, flags, ctr, sflag, rowcnt, gstrip, chkoff, dlb, dllc, full, tiles,
        total;
};
Carve carve(const Plan &p) {
    Carve c{};
    size_t o = 0;
    auto take = [&](size_t bytes) {
        const size_t at = o;
        o += (bytes + 255) / 256 * 256;
        return at;
    };
    const int KB = p.KB;
    c.P = take((size_t)p.NBc * p.nb * p.k * 8);
    c.res = take((size_t)std::max(p.nsl, 1) * kD * p.k * 8);
    c.chk = take((size_t)std::max<int64_t>(p.nchk, 1) * kD * p.k * 8);
    c.Winv = take((size_t)std::max(p.nsl, 1) * kD * kD * 8);
    c.Q = take((size_t)p.NB64 * KB * KB * 8);
    c.G = take((size_t)p.NB64 * KB * KB * 8);
    c.U = take((size_t)p.NB64 * KB * KB * 8);
    c.panels = take((size_t)p.NB64 * panel_doubles(KB) * 8);
    c.key = take(8);
    c.flags = take((size_t)(p.NSB + 1) * 4);
    c.ctr = take(16);
    c.sflag = take((size_t)p.NB64 * kD * p.k * 8);  // persistent chain: strip hand-offs (self-validating)
    c.rowcnt = take((size_t)p.NB64 * 4);              // persistent chain: tiles of row block b checkpointed
    c.gstrip = take((size_t)std::max(p.nsl, 1) * 4);
    c.chkoff = take((size_t)std::max(p.nsl, 1) * 8);
    c.dlb = take((size_t)std::max<size_t>(p.dl_b.size(), 1) * 4);
    c.dllc = take((size_t)std::max<size_t>(p.dl_lc.size(), 1) * 8);
    c.full = take((size_t)std::max<size_t>(p.full.size(), 1) * 8);
    c.tiles = take((size_t)std::max<size_t>(p.tiles.size(), 1) * 8);
    c.total = o;
    return c;
}

// where a kernel writes replicated data: one pointer per rank (device-initiated puts)
struct Peers {
    double *dst[kMaxRanks];
    double *dst2[kMaxRanks];
    unsigned *flag[kMaxRanks];  // nullptr: no flag (stream order suffices)
    int R;
};

__device__ __forceinline__ void st_release_sys(unsigned *p, unsigned v) {
    chaos_delay();
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void wait_flag_sys(const unsigned *f, unsigned epoch) {
    chaos_delay();
    if (threadIdx.x == 0)
        while (ld_acquire_sys(f) != epoch) __nanosleep(200);
    __syncthreads();
}

// -------------------------------------------------------------------------- kernels
// residual of every local strip = its V rows; checkpoint of tile (0, s) likewise
// (persistent chain: also arms P and the hand-offs with all-ones and zeroes rowcnt -- three
// memsets' worth of host calls before the chain's launch)
__global__ void pinit_kernel(const double *__restrict__ V, int64_t ldv, int64_t nloc, int k, const int *gstrip,
                             const int64_t *chkoff, double *res, double *chk, unsigned long long *arm_p = nullptr,
                             int64_t n_p = 0, unsigned long long *arm_h = nullptr, int64_t n_h = 0,
                             unsigned *zero = nullptr, int n_z = 0) {
    const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gs = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = gt; i < n_p; i += gs) arm_p[i] = kEmpty;
    for (int64_t i = gt; i < n_h; i += gs) arm_h[i] = kEmpty;
    for (int64_t i = gt; i < n_z; i += gs) zero[i] = 0u;
    const int sl = blockIdx.x;
    const int64_t lc0 = (int64_t)sl * kD;
    double *r = res + (int64_t)sl * kD * k;
    double *c0 = gstrip[sl] >= 1 ? chk + chkoff[sl] * kD * k : nullptr;
    for (int o = threadIdx.x; o < kD * k; o += blockDim.x) {
        const int c = o / k, e = o % k;
        const double v = lc0 + c < nloc ? V[lc0 + c + (int64_t)e * ldv] : 0.0;
        r[o] = v;
        if (c0) c0[o] = v;
    }
}

// register-block shape of the residual update (pupdate_kernel, dsolve_kernel): kPT threads,
// CPT adjacent strip columns x EPT update columns each
template <int KB>
struct PuShape {
    // a warp covers LC lanes x CPT strip columns by LE lanes x EPT update columns, so one
    // 16-byte L load serves LE lanes (broadcast) and one P load LC lanes: per row 3 shared
    // wavefronts feed 8 FMAs at KB = 32 (a warp spanning all 64 columns needed 6)
    static constexpr int CPT = KB >= 8 ? 2 : 1;
    static constexpr int LE = KB >= 8 ? 4 : 2;     // lanes along update columns
    static constexpr int LC = 32 / LE;             // lanes along strip columns
    static constexpr int EPT = KB / (2 * LE);      // two warps along update columns
    static constexpr int WC = kD / (LC * CPT);     // warps along strip columns
    static constexpr int LDT = kD + 2;             // row stride of the L tile (16-byte aligned)
    static_assert(WC * 2 * 32 == kPT && EPT >= 1, "kPT threads cover 64 columns x KB");
    __device__ static int c0(int t) { return ((t >> 5) % WC * LC + (t & 31) % LC) * CPT; }
    __device__ static int e0(int t) { return ((t >> 5) / WC * LE + (t & 31) / LC) * EPT; }
};
constexpr int kDsMaxRows = 512;  // solve-block height the kernel's shared memory is sized for (KB <= 16)
__device__ __forceinline__ void cp8(double *dst, const double *src, bool ok) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(ok ? src : nullptr),
                 "r"(ok ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp16(double *dst, const double *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

// Inverse of every local strip's 64x64 diagonal block (upper triangular U, U(i, j) =
// L(r0 + i, lc + j), i <= j; PAPER.md's factor is the upper-triangular L of A = L^T L),
// stored by rows: W[j * 64 + m] = (U^{-1})(j, m), zero for j > m and for m >= D.  It turns
// dsolve's serial 64-step substitution q = U^{-T} r into the data-parallel product
// q_m = sum_{j <= m} W(j, m) r_j (the inverted-diagonal-block TRSV of GPU BLAS libraries;
// DESIGN.md R22), and it runs once per pass over all strips at once, off the solve chain.
// Thread m computes column m by back substitution (U w = e_m), its 64 running sums in
// registers at compile-time indices, every U entry a shared-memory broadcast.  The partial
// sums of rows j > m are never formed, so a NaN in U reaches exactly the q_m that
// substitution would reach.
__global__ void __launch_bounds__(kD) pinv_kernel(const double *__restrict__ L, int64_t ldl, int64_t n,
                                                  const int *gstrip, double *W) {
    __shared__ __align__(16) double Us[kD][kD];
    __shared__ double rd[kD];
    const int sl = blockIdx.x;
    const int64_t r0 = (int64_t)gstrip[sl] * kD, lc = (int64_t)sl * kD;
    const int D = (int)imin64(kD, n - r0);
    pinv_block(L + r0 + lc * ldl, ldl, D, W + (int64_t)sl * kD * kD, Us, rd);
}

// Every rank: residuals of its strips right of solve block g -= L_{rows of g, strip}^T P,
// checkpointing the residual at the start of every 64-row tile.  Thread (column group, e
// group) owns CPT adjacent columns x EPT update columns of the strip (a CPT x EPT register
// block: per row one 16-byte load of the L pair and EPT/2 16-byte loads of P feed CPT*EPT
// FMAs); the L tile (row-major in shared memory) and the P rows of the next 64-row
// sub-block stream in (cp.async, double buffered) under the current one.
// KB here is the update columns ONE CTA handles: the lookahead launch splits a strip's
// columns over gridDim.y CTAs (update columns blockIdx.y * KB ..) to cut its latency.
template <int KB>
__global__ void __launch_bounds__(kPT, 2) pupdate_kernel(const double *__restrict__ L, int64_t ldl, int64_t n,
                                                        int64_t nloc, int k, int64_t row0, int nrows, int sl_first,
                                                        double *res, double *chk, const int64_t *chkoff,
                                                        const double *__restrict__ P, const unsigned *flag,
                                                        unsigned epoch) {
    using S = PuShape<KB>;
    const int eb = blockIdx.y * KB;  // first update column of this CTA
    constexpr int CPT = S::CPT, EPT = S::EPT, LDT = S::LDT;
    extern __shared__ __align__(16) double sm_pu[];
    double *Lt = sm_pu;                // [2][kD rows m][LDT]: Lt[m][c] = L(r0 + m, strip column c)
    double *Ps = sm_pu + 2 * kD * LDT;  // [2][kD][KB]
    const int t = threadIdx.x;
    const int c0 = S::c0(t), e0 = S::e0(t);
    const int sl = sl_first + blockIdx.x;
    const int64_t lc = (int64_t)sl * kD;
    const int nc = (int)imin64(kD, nloc - lc);
    const int na = (nrows + kD - 1) / kD;
    if (flag) wait_flag_sys(flag, epoch);
    double *rs = res + (int64_t)sl * kD * k + eb;
    double acc[CPT][EPT];
#pragma unroll
    for (int u = 0; u < CPT; ++u)
#pragma unroll
        for (int i = 0; i < EPT; ++i) acc[u][i] = (c0 + u < nc && eb + e0 + i < k) ? rs[(c0 + u) * k + e0 + i] : 0.0;
    auto issue = [&](int a) {
        const int64_t r0 = row0 + (int64_t)a * kD;
        const int Da = (int)imin64(kD, n - r0);
        double *lt = Lt + (a & 1) * kD * LDT;
        double *ps = Ps + (a & 1) * kD * KB;
        for (int idx = t; idx < kD * kD; idx += kPT) {
            const int cc = idx / kD, m = idx % kD;  // consecutive threads: consecutive rows (coalesced)
            const bool ok = cc < nc && m < Da;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(lt + m * LDT + cc)),
                         "l"(ok ? L + (r0 + m) + (lc + cc) * ldl : L), "r"(ok ? 8 : 0)
                         : "memory");
        }
        for (int idx = t; idx < kD * KB; idx += kPT) {
            const int m = idx / KB, e = idx % KB;
            const bool ok = m < Da && eb + e < k;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(ps + idx)),
                         "l"(ok ? P + (r0 + m) * k + eb + e : P), "r"(ok ? 8 : 0)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    issue(0);
    for (int a = 0; a < na; ++a) {
        const int64_t r0 = row0 + (int64_t)a * kD;
        if (a + 1 < na) {
            issue(a + 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        {
            double *ck = chk + (chkoff[sl] + r0 / kD) * kD * k + eb;
#pragma unroll
            for (int u = 0; u < CPT; ++u)
#pragma unroll
                for (int i = 0; i < EPT; ++i)
                    if (c0 + u < nc && eb + e0 + i < k) ck[(c0 + u) * k + e0 + i] = acc[u][i];
        }
        const double *lt = Lt + (a & 1) * kD * LDT + c0;
        const double *ps = Ps + (a & 1) * kD * KB + e0;
#pragma unroll 4
        for (int m = 0; m < kD; ++m) {
            double l[CPT], pv[EPT];
            if constexpr (CPT == 2) {
                const double2 l2 = *reinterpret_cast<const double2 *>(lt + m * LDT);
                l[0] = l2.x;
                l[1] = l2.y;
            } else {
                l[0] = lt[m * LDT];
            }
            if constexpr (EPT % 2 == 0) {
#pragma unroll
                for (int i = 0; i < EPT; i += 2) {
                    const double2 p2 = *reinterpret_cast<const double2 *>(ps + m * KB + i);
                    pv[i] = p2.x;
                    pv[i + 1] = p2.y;
                }
            } else {
#pragma unroll
                for (int i = 0; i < EPT; ++i) pv[i] = ps[m * KB + i];
            }
#pragma unroll
            for (int u = 0; u < CPT; ++u)
#pragma unroll
                for (int i = 0; i < EPT; ++i) acc[u][i] = fma(-l[u], pv[i], acc[u][i]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < CPT; ++u)
#pragma unroll
        for (int i = 0; i < EPT; ++i)
            if (c0 + u < nc && eb + e0 + i < k) rs[(c0 + u) * k + e0 + i] = acc[u][i];
}

// The same update on the FP64 tensor cores (DMMA, mma.sync m8n8k4 .f64: D(8x8) += A(8x4) B(4x8)
// with M = strip columns c, N = update columns e, K = rows m).  Warp tile TC x TE MMA tiles;
// the L tile is staged column-major (Lc[c][m], 16-byte cp.async straight from L's columns)
// with a 68-double column stride and the P tile with a KB + 4 row stride, so every fragment
// load is one conflict-free shared wavefront per half warp.  Per 4 rows a warp issues TC + TE
// fragment loads and TC * TE MMAs (256 FMAs each) where the DFMA form issued 4 * 3 loads and
// 4 * 8 DFMAs; the accumulators hold the NEGATED residual (so each MMA adds L^T P).
template <int KB>
struct PmShape {
    static constexpr int TC = KB >= 16 ? 2 : 1;   // 8-column MMA tiles per warp along strip columns
    static constexpr int TE = KB >= 32 ? 2 : 1;   // ... along update columns
    static constexpr int WC = kD / (8 * TC);      // warps along strip columns
    static_assert(WC * (KB / (8 * TE)) * 32 == kPT, "kPT threads cover 64 columns x KB");
    static constexpr int LDC = kD + 4;            // column stride of the L tile
    static constexpr int LDP = KB + 4;            // row stride of the P tile
};
template <int KB>
size_t pupdate_mma_smem() {
    return (size_t)(2 * kD * PmShape<KB>::LDC + 2 * kD * PmShape<KB>::LDP) * 8;
}
template <int KB>
__global__ void __launch_bounds__(kPT, 2) pupdate_mma_kernel(const double *__restrict__ L, int64_t ldl, int64_t n,
                                                            int64_t nloc, int k, int64_t row0, int nrows,
                                                            int sl_first, double *res, double *chk,
                                                            const int64_t *chkoff, const double *__restrict__ P,
                                                            const unsigned *flag, unsigned epoch) {
    using S = PmShape<KB>;
    constexpr int TC = S::TC, TE = S::TE, LDC = S::LDC, LDP = S::LDP;
    const int eb = blockIdx.y * KB;  // first update column of this CTA
    extern __shared__ __align__(16) double sm_pm[];
    double *Lc = sm_pm;                   // [2][kD strip columns c][LDC]: Lc[c][m] = L(r0 + m, lc + c)
    double *Ps = sm_pm + 2 * kD * LDC;    // [2][kD rows m][LDP]
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int gi = lane >> 2, tg = lane & 3;
    const int cw = (warp % S::WC) * 8 * TC, ew = (warp / S::WC) * 8 * TE;
    const int sl = sl_first + blockIdx.x;
    const int64_t lc = (int64_t)sl * kD;
    const int nc = (int)imin64(kD, nloc - lc);
    const int na = (nrows + kD - 1) / kD;
    const int ke = k - eb;  // update columns of this CTA that exist
    // 16-byte copies need 16-byte aligned columns (an even ldl and an aligned L)
    const bool v16 = (ldl % 2 == 0) && ((reinterpret_cast<uintptr_t>(L) & 15) == 0);
    // P rows by 16-byte copies when every (row, column pair) is 16-byte aligned
    const bool p16 = (k % 2 == 0) && (eb % 2 == 0) && ((reinterpret_cast<uintptr_t>(P) & 15) == 0);
    if (flag) wait_flag_sys(flag, epoch);
    double *rs = res + (int64_t)sl * kD * k + eb;
    auto issue = [&](int a) {
        const int64_t r0 = row0 + (int64_t)a * kD;
        const int Da = (int)imin64(kD, n - r0);
        double *lcb = Lc + (a & 1) * kD * LDC;
        double *ps = Ps + (a & 1) * kD * LDP;
        if (v16) {
            for (int idx = t; idx < kD * kD / 2; idx += kPT) {
                const int c = idx >> 5, m = 2 * (idx & 31);  // a column's 64 rows: 32 consecutive threads
                const int bytes = (c < nc && m < Da) ? (Da - m >= 2 ? 16 : 8) : 0;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(lcb + c * LDC + m)),
                             "l"(bytes ? L + (r0 + m) + (lc + c) * ldl : L), "r"(bytes)
                             : "memory");
            }
        } else {
            for (int idx = t; idx < kD * kD; idx += kPT) {
                const int c = idx >> 6, m = idx & 63;
                const bool ok = c < nc && m < Da;
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(lcb + c * LDC + m)),
                             "l"(ok ? L + (r0 + m) + (lc + c) * ldl : L), "r"(ok ? 8 : 0)
                             : "memory");
            }
        }
        if (p16) {
            for (int idx = t; idx < kD * KB / 2; idx += kPT) {
                const int m = idx / (KB / 2), e = 2 * (idx % (KB / 2));
                const int bytes = (m < Da && e < ke) ? (ke - e >= 2 ? 16 : 8) : 0;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(ps + m * LDP + e)),
                             "l"(bytes ? P + (r0 + m) * k + eb + e : P), "r"(bytes)
                             : "memory");
            }
        } else {
            for (int idx = t; idx < kD * KB; idx += kPT) {
                const int m = idx / KB, e = idx % KB;
                const bool ok = m < Da && e < ke;
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(ps + m * LDP + e)),
                             "l"(ok ? P + (r0 + m) * k + eb + e : P), "r"(ok ? 8 : 0)
                             : "memory");
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    issue(0);  // before the residual loads: their first use would stall the issue of the copies
    const int64_t ckbase = chkoff[sl];
    double acc[TC][TE][2];
#pragma unroll
    for (int u = 0; u < TC; ++u)
#pragma unroll
        for (int v = 0; v < TE; ++v)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c = cw + 8 * u + gi, e = ew + 8 * v + 2 * tg + h;
                acc[u][v][h] = (c < nc && e < ke) ? -rs[c * k + e] : 0.0;
            }
    for (int a = 0; a < na; ++a) {
        const int64_t r0 = row0 + (int64_t)a * kD;
        if (a + 1 < na) {
            issue(a + 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        {
            double *ck = chk + (ckbase + r0 / kD) * kD * k + eb;
#pragma unroll
            for (int u = 0; u < TC; ++u)
#pragma unroll
                for (int v = 0; v < TE; ++v)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int c = cw + 8 * u + gi, e = ew + 8 * v + 2 * tg + h;
                        if (c < nc && e < ke) ck[c * k + e] = -acc[u][v][h];
                    }
        }
        const double *la = Lc + (a & 1) * kD * LDC + (cw + gi) * LDC + tg;
        const double *pb = Ps + (a & 1) * kD * LDP + tg * LDP + ew + gi;
#pragma unroll 4
        for (int m0 = 0; m0 < kD; m0 += 4) {
            double af[TC], bf[TE];
#pragma unroll
            for (int u = 0; u < TC; ++u) af[u] = la[8 * u * LDC + m0];
#pragma unroll
            for (int v = 0; v < TE; ++v) bf[v] = pb[m0 * LDP + 8 * v];
#pragma unroll
            for (int u = 0; u < TC; ++u)
#pragma unroll
                for (int v = 0; v < TE; ++v) dmma_884(acc[u][v], af[u], bf[v]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < TC; ++u)
#pragma unroll
        for (int v = 0; v < TE; ++v)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c = cw + 8 * u + gi, e = ew + 8 * v + 2 * tg + h;
                if (c < nc && e < ke) rs[c * k + e] = -acc[u][v][h];
            }
}

// The owner's diagonal solve of column block g: P rows [row0, row0 + nrows) = L_gg^{-T} r_g,
// 64-row sub-block a after sub-block a: q_a = W_a^T r_a (W_a the inverted diagonal block of
// pinv_kernel), the rows written to every rank's P, then the residuals (and Apply
// checkpoints) of the block's later sub-blocks updated with them; both products on the FP64
// tensor cores (DMMA m8n8k4), the diagonal 8x8 blocks of the first by DFMA so that a product
// 0 * r_j with j > m is never formed (a NaN in r_j reaches q_m only for m >= j, as in
// substitution).  One CTA; the block's residuals stay in shared memory for the whole kernel
// (they are dead after it: the block's strips have no tiles below it), and every W and L
// tile is prefetched a step ahead (cp.async), so the only exposed latency is the first load.
template <int KB>
struct DsShape {
    static constexpr int NE = KB >= 8 ? KB : 8;  // update columns held (MMA N = 8: KB = 4 pads)
    static constexpr int LDR = NE + 4;           // row stride of R and q (conflict-free B fragments)
    static constexpr int LDW = kD + 4;           // row stride of W, column stride of the L tiles
    static constexpr int ET = NE / 8;            // 8-column MMA tiles along update columns
    static constexpr int TPW = (8 * ET + 15) / 16;  // of them per warp (16 warps, 8 row / column tiles)
};
template <int KB>
__global__ void __launch_bounds__(kDsT, 1) dsolve_kernel(const double *__restrict__ L, int64_t ldl, int64_t n, int k,
                                                       int64_t row0, int nrows, int sl0, double *res, double *chk,
                                                       const int64_t *chkoff, const double *__restrict__ Winv,
                                                       Peers peers, unsigned epoch) {
    using S = DsShape<KB>;
    constexpr int NE = S::NE, LDR = S::LDR, LDW = S::LDW, ET = S::ET, TPW = S::TPW;
    extern __shared__ __align__(16) double sm_ds[];
    double *Ws = sm_ds;                // [kD rows j][LDW]: W(j, m) of the current sub-block
    double *Lc = Ws + kD * LDW;        // [2][kD columns c][LDW]: Lc[c][m] = L(r0 + m, column c of sub-block a2)
    double *qv = Lc + 2 * kD * LDW;    // [kD][LDR]: q of the current sub-block
    double *R = qv + kD * LDR;         // [rows][LDR]: the block's residuals
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31, gi = lane >> 2, tg = lane & 3;
    const int na = (nrows + kD - 1) / kD;
    const bool v16 = (ldl % 2 == 0) && ((reinterpret_cast<uintptr_t>(L) & 15) == 0);
    // the whole block's residuals (one round trip) and the first W
    for (int o = t; o < na * kD * NE; o += kDsT) {
        const int row = o / NE, e = o % NE;
        const int a = row / kD, m = row % kD;
        cp8(R + row * LDR + e, res + (int64_t)(sl0 + a) * kD * k + m * k + e, e < k && row < nrows);
    }
    auto load_w = [&](int a) {  // W of sub-block a: 32 KB, contiguous
        const double *src = Winv + (int64_t)(sl0 + a) * kD * kD;
        for (int idx = t; idx < kD * kD / 2; idx += kDsT) {
            const int j = idx >> 5, m = 2 * (idx & 31);
            cp16(Ws + j * LDW + m, src + j * kD + m);
        }
    };
    // tile (a, a2): rows of sub-block a, columns of sub-block a2, column-major into Lc[buf]
    auto load_tile = [&](int a, int a2, int buf) {
        const int64_t r0 = row0 + (int64_t)a * kD;
        const int Da = (int)imin64(kD, n - r0);
        const int64_t lc2 = (int64_t)(sl0 + a2) * kD;
        const int D2 = (int)imin64(kD, n - (row0 + (int64_t)a2 * kD));
        double *lt = Lc + buf * kD * LDW;
        if (v16) {
            for (int idx = t; idx < kD * kD / 2; idx += kDsT) {
                const int c = idx >> 5, m = 2 * (idx & 31);  // a column's 64 rows: 32 consecutive threads
                const int bytes = (c < D2 && m < Da) ? (Da - m >= 2 ? 16 : 8) : 0;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(lt + c * LDW + m)),
                             "l"(bytes ? L + (r0 + m) + (lc2 + c) * ldl : L), "r"(bytes)
                             : "memory");
            }
        } else {
            for (int idx = t; idx < kD * kD; idx += kDsT) {
                const int c = idx >> 6, m = idx & 63;
                cp8(lt + c * LDW + m, L + (r0 + m) + (lc2 + c) * ldl, c < D2 && m < Da);
            }
        }
    };
    load_w(0);
    asm volatile("cp.async.commit_group;" ::: "memory");
    for (int a = 0; a < na; ++a) {
        const int64_t r0 = row0 + (int64_t)a * kD;
        const int Da = (int)imin64(kD, n - r0);
        if (a + 1 < na) load_tile(a, a + 1, 0);  // first update tile of this step, under the solve
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 1;" ::: "memory");  // R, W(a) landed
        __syncthreads();
        // q = W^T r_a: M = rows m, N = update columns e, K = rows j; warp -> row tile, TPW column tiles
        {
            const int mt = warp % 8, eg = warp / 8;
            if (eg * TPW < ET) {
                const int m0 = mt * 8;
                const double *Ra = R + a * kD * LDR;
                double acc[TPW][2];
#pragma unroll
                for (int v = 0; v < TPW; ++v) acc[v][0] = acc[v][1] = 0.0;
                for (int j0 = 0; j0 < m0; j0 += 4) {  // blocks strictly above the tile's rows: j < m
                    const double af = Ws[(j0 + tg) * LDW + m0 + gi];
#pragma unroll
                    for (int v = 0; v < TPW; ++v) dmma_884(acc[v], af, Ra[(j0 + tg) * LDR + (eg * TPW + v) * 8 + gi]);
                }
                const int m = m0 + gi;
#pragma unroll
                for (int v = 0; v < TPW; ++v)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int e = (eg * TPW + v) * 8 + 2 * tg + h;
                        double s = acc[v][h];
                        for (int j = m0; j <= m; ++j) s = fma(Ws[j * LDW + m], Ra[j * LDR + e], s);
                        qv[m * LDR + e] = m < Da ? s : 0.0;  // rows past the block stay zero
                    }
            }
        }
        __syncthreads();
        for (int o = t; o < Da * k; o += kDsT) {
            const int m = o / k, e = o % k;
            const double v = qv[m * LDR + e];
            for (int r = 0; r < peers.R; ++r) peers.dst[r][(r0 + m) * k + e] = v;
        }
        if (a + 1 < na) load_w(a + 1);  // Ws is free (the P stores and updates read qv)
        asm volatile("cp.async.commit_group;" ::: "memory");
        for (int a2 = a + 1; a2 < na; ++a2) {
            const int buf = (a2 - a - 1) & 1;
            if (a2 + 1 < na) load_tile(a, a2 + 1, buf ^ 1);
            asm volatile("cp.async.commit_group;" ::: "memory");
            // tile (a, a2) landed: at a2 = a + 1 W(a + 1) and tile (a, a + 2) may still be in
            // flight, later only the tile just issued
            if (a2 == a + 1) asm volatile("cp.async.wait_group 2;" ::: "memory");
            else asm volatile("cp.async.wait_group 1;" ::: "memory");
            __syncthreads();
            const int D2 = (int)imin64(kD, n - (row0 + (int64_t)a2 * kD));
            double *ck = chk + (chkoff[sl0 + a2] + r0 / kD) * kD * k;  // tile (r0/64, strip a2)
            // r_a2 -= L_tile^T q: M = strip columns c, N = update columns e, K = rows m
            const int ct = warp % 8, eg = warp / 8;
            if (eg * TPW < ET) {
                const int c = ct * 8 + gi;
                double *Rc = R + (a2 * kD + c) * LDR;
                double acc[TPW][2];
#pragma unroll
                for (int v = 0; v < TPW; ++v)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int e = (eg * TPW + v) * 8 + 2 * tg + h;
                        const double r = Rc[e];
                        if (c < D2 && e < k) ck[c * k + e] = r;
                        acc[v][h] = -r;
                    }
                const double *la = Lc + buf * kD * LDW + c * LDW + tg;
                const double *qb = qv + tg * LDR + eg * TPW * 8 + gi;
#pragma unroll 4
                for (int m0 = 0; m0 < kD; m0 += 4) {
                    const double af = la[m0];
#pragma unroll
                    for (int v = 0; v < TPW; ++v) dmma_884(acc[v], af, qb[m0 * LDR + v * 8]);
                }
#pragma unroll
                for (int v = 0; v < TPW; ++v)
#pragma unroll
                    for (int h = 0; h < 2; ++h) Rc[(eg * TPW + v) * 8 + 2 * tg + h] = -acc[v][h];
            }
            __syncthreads();  // Lc[buf] is refilled two steps on
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();
    }
    if (peers.flag[0]) {  // PEER mode: the P rows are visible to every rank before the flag
        __threadfence_system();
        __syncthreads();
        if (t == 0)
            for (int r = 0; r < peers.R; ++r) st_release_sys(peers.flag[r], epoch);
    }
}

// ------------------------------------------------------------------ persistent chain (one rank)
// GCM_ALGO_PANEL with one rank replaces the per-solve-block launches (dsolve, lookahead and
// rest pupdate) by ONE cooperative kernel working in 64-row steps:
//   CTAs 0 .. NS-1 (solvers, 8 update columns each: the right-hand sides of P = L^{-T} V are
//     independent, so each solver's DMMA work per step is an 8-column slice), step b:
//     r_b = the hand-off of strip b (its residual after P_{<= b-2}, from
//     its helper; V itself for b < 2) = the checkpoint of tile (b-1, b), minus L_{b-1,b}^T q_{b-1}
//     (its own one-block lookahead), then q_b = W_b^T r_b (W_b = L_bb^{-1}, pinv_kernel) -- both
//     on DMMA -- published as P's rows; W_{b+1}, L_{b,b+1} and strip b+1's hand-off are loaded
//     under the step (a two-block lookahead measured slower: the solver's SM is the bottleneck);
//   CTAs NS.. (helpers): strip s >= 2 belongs to helper (s - 2) mod H; tiles (b, s), b <= s - 2,
//     in b-major order: poll P_b (prefetched a row ahead), checkpoint, r_s -= L_{b,s}^T P_b
//     (DMMA), and after b = s - 2 hand r_s to the solver.  The next tile is staged under the
//     current one; residuals of the first OWN owned strips stay in shared memory between tiles
//     (the rest round-trip res[]).
// P and the hand-offs are self-validating values (st_value / ld_value: the pass arms both with
// all-ones), so a consumer needs one L2 round trip and no flag.  No CTA waits on a later one
// (the solver on hand-offs of earlier tiles, helpers on P blocks the solver publishes without
// waiting for them), so the cooperative grid cannot deadlock.
constexpr int kPcT = 512;
#ifndef GCM_PC_REL
#define GCM_PC_REL 8
#endif
constexpr int kPcRel = GCM_PC_REL;  // helper tiles per rowcnt release
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
#ifdef GCM_PC_TRACE  // solver step timeline (globaltimer ns): tools/pchain_trace.py
__device__ long long g_pc_trace[4096 * 4];
__device__ __forceinline__ long long pc_now() {
    long long v;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
    return v;
}
#define PC_MARK(b, slot) \
    do {                 \
        if (t == 0 && blockIdx.x == 0 && (b) < 4096) g_pc_trace[(b) * 4 + (slot)] = pc_now(); \
    } while (0)
// helper blockIdx.x == 40: per tile (sequence number q) 0 top, 1 P in smem, 2 tile landed, 3 MMA done
#define PH_MARK(q, slot) \
    do {                 \
        if (t == 0 && blockIdx.x == 40 && (q) < 1024) g_pc_trace[(3072 + (q)) * 4 + (slot)] = pc_now(); \
    } while (0)
#else
#define PC_MARK(b, slot) ((void)0)
#define PH_MARK(q, slot) ((void)0)
#endif
template <int KB>
struct PcShape {
    static constexpr int NE = KB >= 8 ? KB : 8;
    static constexpr int LDR = NE + 4;
    static constexpr int LDW = kD + 4;
    static constexpr int ET = NE / 8;
    static constexpr int TPW = (8 * ET + 15) / 16;
    static constexpr int OWN = KB >= 32 ? 5 : 10;  // helper strips whose residual stays in shared memory
    static constexpr int NS = NE / 8;  // solver CTAs
    static constexpr size_t solver_doubles = 4 * kD * LDW + 5 * kD * 12;  // 2 W, 2 lookahead tiles, 2 q, r, 2 hand-off
    static constexpr size_t helper_doubles = 2 * kD * LDW + kD * LDR + (OWN + 2) * kD * LDR;  // + spill slots
    static constexpr size_t doubles = solver_doubles > helper_doubles ? solver_doubles : helper_doubles;
};
template <int KB>
size_t pchain_smem() {
    return PcShape<KB>::doubles * 8;
}
// self-validating values (the pass arms P and the hand-off buffer with all-ones, a NaN pattern no
// producer stores: NaNs are canonicalised): a consumer polls the value itself -- one L2 round
// trip, no flag, no fence
__device__ __forceinline__ void st_value(double *p, double v) {
    chaos_delay();
    const double w = v == v ? v : __longlong_as_double(0x7ff8000000000000ll);
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(w) : "memory");
}
template <int KB>
__global__ void __launch_bounds__(kPcT, 1) pchain_kernel(const double *__restrict__ L, int64_t ldl, int64_t n, int k,
                                                        int NB, double *res, double *chk, const int64_t *chkoff,
                                                        const double *__restrict__ Winv, double *P, double *hand,
                                                        unsigned *rowcnt) {
    using S = PcShape<KB>;
    constexpr int NE = S::NE, LDR = S::LDR, LDW = S::LDW, ET = S::ET, TPW = S::TPW;
    extern __shared__ __align__(16) double sm_pc[];
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31, gi = lane >> 2, tg = lane & 3;
    const bool v16 = (ldl % 2 == 0) && ((reinterpret_cast<uintptr_t>(L) & 15) == 0);
    // the warp's output tiles: strip columns c = ct*8 + gi, update columns e = (eg*TPW + v)*8 + 2tg + h
    const int ct = warp % 8, eg = warp / 8;
    const bool mma_warp = eg * TPW < ET;
    const int c = ct * 8 + gi;
    auto ecol = [&](int v, int h) { return (eg * TPW + v) * 8 + 2 * tg + h; };
    // L(rows of block rb, columns of block cb) -> dst[c][m] (column-major, stride LDW), zero outside
    auto load_tile = [&](double *dst, int rb, int cb, int tid = -1, int nthr = kPcT) {
        if (tid < 0) tid = t;
        const int64_t r0 = (int64_t)rb * kD, c0 = (int64_t)cb * kD;
        const int Dr = (int)imin64(kD, n - r0), Dc = (int)imin64(kD, n - c0);
        if (v16) {
            for (int idx = tid; idx < kD * kD / 2; idx += nthr) {
                const int cc = idx >> 5, m = 2 * (idx & 31);
                const int bytes = (cc < Dc && m < Dr) ? (Dr - m >= 2 ? 16 : 8) : 0;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst + cc * LDW + m)),
                             "l"(bytes ? L + (r0 + m) + (c0 + cc) * ldl : L), "r"(bytes)
                             : "memory");
            }
        } else {
            for (int idx = tid; idx < kD * kD; idx += nthr) {
                const int cc = idx >> 6, m = idx & 63;
                cp8(dst + cc * LDW + m, L + (r0 + m) + (c0 + cc) * ldl, cc < Dc && m < Dr);
            }
        }
    };
    // rows [0, nrows) x k of a row-major (ld k) global block -> dst[m][LDR], zero outside
    auto load_rows = [&](double *dst, const double *src, int nrows) {
        for (int o = t; o < kD * NE; o += kPcT) {
            const int m = o / NE, e = o % NE;
            cp8(dst + m * LDR + e, src + (int64_t)m * k + e, m < nrows && e < k);
        }
    };
    // acc += A^T B: A = tile dst[c][m] (stride LDW), B = rows [m][LDR]; K = 64
    auto mma_tile = [&](double (&acc)[TPW][2], const double *A, const double *B) {
        const double *la = A + c * LDW + tg;
        const double *qb = B + tg * LDR + eg * TPW * 8 + gi;
        double acc2[TPW][2];  // two accumulator chains (k-steps m0 = 0, 8, .. and 4, 12, ..): half the
                              // dependent DMMA latency on the chain's critical path
#pragma unroll
        for (int v = 0; v < TPW; ++v) acc2[v][0] = acc2[v][1] = 0.0;
#pragma unroll 2
        for (int m0 = 0; m0 < kD; m0 += 8) {
            const double af = la[m0], ag = la[m0 + 4];
#pragma unroll
            for (int v = 0; v < TPW; ++v) {
                dmma_884(acc[v], af, qb[m0 * LDR + v * 8]);
                dmma_884(acc2[v], ag, qb[(m0 + 4) * LDR + v * 8]);
            }
        }
#pragma unroll
        for (int v = 0; v < TPW; ++v) {
            acc[v][0] += acc2[v][0];
            acc[v][1] += acc2[v][1];
        }
    };

    constexpr int NS = S::NS;  // solver CTAs: 8 update columns each (the right-hand sides are independent)
    if ((int)blockIdx.x < NS) {
        // ------------------------------------------------------------ solver for columns es .. es+7
        constexpr int LDQ = 12;              // row stride of the solver's q / r (8 columns + pad)
        const int es = blockIdx.x * 8;
        double *Ws = sm_pc;                 // [2][kD][LDW]: W_b at b % 2
        double *Lt = Ws + 2 * kD * LDW;     // [2][kD][LDW]: L_{b-1,b} at b % 2
        double *qh = Lt + 2 * kD * LDW;     // [2][kD][LDQ]: q_b at b % 2
        double *rb = qh + 2 * kD * LDQ;     // [kD][LDQ]
        const bool sw = warp < 8;           // warp = 8-row tile (MMA warps)
        const int sc = warp * 8 + gi;       // this lane's strip column / output row
        auto load_w = [&](int b) {
            const double *src = Winv + (int64_t)b * kD * kD;
            double *dst = Ws + (b & 1) * kD * LDW;
            for (int idx = t - 256; idx < kD * kD / 2; idx += 256) {  // issued by the poller warps
                const int j = idx >> 5, m = 2 * (idx & 31);
                cp16(dst + j * LDW + m, src + j * kD + m);
            }
        };
        // acc (8 x 8 tile per warp, lane: row sc, columns 2tg, 2tg+1) += A^T B, K = 64
        auto mma8 = [&](double (&a2)[2], const double *A, const double *B) {
            const double *la = A + sc * LDW + tg;
            const double *qb = B + tg * LDQ + gi;
            double b2[2] = {0.0, 0.0};  // second accumulator chain (as mma_tile)
#pragma unroll 2
            for (int m0 = 0; m0 < kD; m0 += 8) {
                dmma_884(a2, la[m0], qb[m0 * LDQ]);
                dmma_884(b2, la[m0 + 4], qb[(m0 + 4) * LDQ]);
            }
            a2[0] += b2[0];
            a2[1] += b2[1];
        };
        // warps 8..15 poll strip b+1's hand-off (V for b + 1 < 2) from the top of step b into hs[(b+1) % 2]
        // and store it as checkpoint (b, b+1): the poll runs under step b's MMA work, so at step b+1
        // the value is in shared memory instead of one exposed L2 round trip away
        double *hs = rb + kD * LDQ;         // [2][kD][LDQ]
        const int pr = (t - 256) >> 2, pe = 2 * ((t - 256) & 3);  // poller: row, column pair
        auto poll_hand = [&](int b) {
            const int64_t r0 = (int64_t)b * kD;
            const int Db = (int)imin64(kD, n - r0);
            const double *src = (b < 2 ? res : hand) + r0 * k + (int64_t)pr * k + es;
            double *ck = b >= 1 ? chk + (chkoff[b] + b - 1) * kD * k + (int64_t)pr * k + es : nullptr;
            unsigned long long u[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int e = pe + h;
                u[h] = (pr < Db && es + e < k) ? ld_relaxed_u64(src + e) : 0ull;
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int e = pe + h;
                if (b >= 2 && pr < Db && es + e < k && u[h] == kEmpty) u[h] = __double_as_longlong(ld_value(src + e));
                const double r = __longlong_as_double((long long)u[h]);
                hs[(b & 1) * kD * LDQ + pr * LDQ + e] = r;
                if (ck && pr < Db && es + e < k) ck[e] = r;
            }
        };
        if (!sw) {
            load_w(0);
            asm volatile("cp.async.commit_group;" ::: "memory");
            poll_hand(0);
        }
        for (int b = 0; b < NB; ++b) {
            const int64_t r0 = (int64_t)b * kD;
            const int Db = (int)imin64(kD, n - r0);
            // W_b and L_{b-1,b} were issued at the top of step b - 1; r_b was polled under step b - 1
            PC_MARK(b, 0);
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            __syncthreads();  // also: step b - 1's reads of the buffers refilled next are done
            PC_MARK(b, 1);
            if (!sw) {
                if (b + 1 < NB) {  // the next step's W and lookahead tile fly under this whole step (the
                                   // poller warps issue them: the MMA warps never stall on copy issue)
                    load_w(b + 1);
                    load_tile(Lt + ((b + 1) & 1) * kD * LDW, b, b + 1, t - 256, 256);
                    asm volatile("cp.async.commit_group;" ::: "memory");
                }
                if (b >= 2 && t == 256) {  // tile (b-2, b-1): checkpoint written, L_{b-2,b-1} consumed
                    fence_acq_rel_gpu();
                    atomicAdd(rowcnt + (b - 2), 1u);
                }
                if (b + 1 < NB) poll_hand(b + 1);
                continue;
            }
            // r_b = strip b's hand-off (its residual after P_{<= b-2}), minus L_{b-1,b}^T q_{b-1}
            double acc[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) acc[h] = -hs[(b & 1) * kD * LDQ + sc * LDQ + 2 * tg + h];
            PC_MARK(b, 2);
            if (b >= 1) mma8(acc, Lt + (b & 1) * kD * LDW, qh + ((b - 1) & 1) * kD * LDQ);
#pragma unroll
            for (int h = 0; h < 2; ++h) rb[sc * LDQ + 2 * tg + h] = -acc[h];  // r^{(b)}
            named_bar(1, 256);
            // q_b = W^T r^{(b)} (DMMA above the 8-row diagonal tiles, masked DFMA on them, so a
            // product 0 * r_j with j > m is never formed)
            const double *Wb = Ws + (b & 1) * kD * LDW;
            double *qv = qh + (b & 1) * kD * LDQ;
            {
                const int m0 = warp * 8;
                double qa[2] = {0.0, 0.0};
                for (int j0 = 0; j0 < m0; j0 += 4) dmma_884(qa, Wb[(j0 + tg) * LDW + m0 + gi], rb[(j0 + tg) * LDQ + gi]);
                const int m = m0 + gi;
                double wd[8];  // W(m0 .. m0+7, m): loaded up front, the FMA chain then runs on registers
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) wd[jj] = Wb[(m0 + jj) * LDW + m];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int e = 2 * tg + h;
                    double rd[8];
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj) rd[jj] = rb[(m0 + jj) * LDQ + e];
                    double s = qa[h];
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj)
                        if (jj <= gi) s = fma(wd[jj], rd[jj], s);  // j <= m only
                    s = m < Db ? s : 0.0;  // rows past the block stay zero
                    qv[m * LDQ + e] = s;
                    if (m < Db && es + e < k) st_value(P + (r0 + m) * k + es + e, s);  // published
                }
            }
            PC_MARK(b, 3);
        }
        __syncthreads();
        if (NB >= 2 && t == 256) {  // tile (NB-2, NB-1)
            fence_acq_rel_gpu();
            atomicAdd(rowcnt + (NB - 2), 1u);
        }
        return;
    }
    // ---------------------------------------------------------------- helpers
    const int h = blockIdx.x - NS, H = gridDim.x - NS;
    double *Lh = sm_pc;                 // [2][kD][LDW]: this tile and the next
    double *Ph = Lh + 2 * kD * LDW;     // [kD][LDR]
    double *Rs = Ph + kD * LDR;         // [OWN + 2][kD][LDR]: residuals of the first OWN owned strips,
                                        //   then one spill slot per tile buffer
    int nown = 0;
    for (int s = 2 + h; s < NB; s += H) ++nown;
    if (nown == 0) return;
    auto rload = [&](double *dst, int s) {
        load_rows(dst, res + (int64_t)s * kD * k, (int)imin64(kD, n - (int64_t)s * kD));
    };
    for (int i = 0; i < nown && i < S::OWN; ++i) rload(Rs + i * kD * LDR, 2 + h + i * H);
    // tiles (b, strip #i) in b-major order, b <= s_i - 2; the next tile's copies fly under this one
    struct It {
        int b, i;
    };
    const int last_b = 2 + h + (nown - 1) * H - 2;  // the last tile row any owned strip needs
    auto imin = [&](int b) { return b <= h ? 0 : (b - h + H - 1) / H; };
    auto valid = [&](const It &x) { return x.b <= last_b && x.i < nown; };
    auto adv = [&](It &x) {
        if (++x.i >= nown) {
            ++x.b;
            x.i = imin(x.b);
        }
    };
    // (a spilled residual is copied with its tile unless the tile just before is the same strip's:
    // that tile's result is not stored yet, it hands its registers over instead)
    auto stage = [&](const It &x, int buf, bool same_strip) {
        const int s = 2 + h + x.i * H;
        load_tile(Lh + buf * kD * LDW, x.b, s);
        if (x.i >= S::OWN && !same_strip) rload(Rs + (S::OWN + buf) * kD * LDR, s);
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    It cur{0, 0};
    stage(cur, 0, false);  // (the residual slots' copies are in this first group)
    int buf = 0, pb = -1, seq = 0;
    int rel_b[kPcRel], nrel = 0;  // thread 0: tile rows whose rowcnt release is pending
    // P values of the next tile row, loaded ahead (self-validating: a non-empty value is final;
    // the rest are polled when that row's first tile starts)
    constexpr int PPT = (kD * NE + kPcT - 1) / kPcT;
    unsigned long long pn[PPT];
    int pn_b = -1;
    auto issue_p = [&](int bn) {
        const int64_t rn0 = (int64_t)bn * kD;
        const int Dn = (int)imin64(kD, n - rn0);
#pragma unroll
        for (int q = 0; q < PPT; ++q) {
            const int o = t + q * kPcT, m = o / NE, e = o % NE;
            pn[q] = (o < kD * NE && m < Dn && e < k) ? ld_relaxed_u64(P + (rn0 + m) * k + e) : 0ull;
        }
        pn_b = bn;
    };
    while (valid(cur)) {
        It nx = cur;
        adv(nx);
        const bool chained = valid(nx) && nx.i == cur.i;
        if (valid(nx)) stage(nx, buf ^ 1, chained);
        const int b = cur.b, i = cur.i, s = 2 + h + i * H;
        const int64_t r0 = (int64_t)b * kD;
        const int Db = (int)imin64(kD, n - r0);
        const int64_t cks = chkoff[s];  // issued before the P poll: its latency hides there
        PH_MARK(seq, 0);
        if (b != pb) {  // P_b, polled per value (every load in flight before the first wait)
            if (pn_b != b) issue_p(b);
            unsigned long long u[PPT];
#pragma unroll
            for (int q = 0; q < PPT; ++q) u[q] = pn[q];
#pragma unroll
            for (int q = 0; q < PPT; ++q) {
                const int o = t + q * kPcT, m = o / NE, e = o % NE;
                if (o < kD * NE) {
                    if (u[q] == kEmpty) u[q] = __double_as_longlong(ld_value(P + (r0 + m) * k + e));
                    Ph[m * LDR + e] = __longlong_as_double((long long)u[q]);
                }
            }
            pb = b;
        }
        PH_MARK(seq, 1);
        if (valid(nx)) asm volatile("cp.async.wait_group 1;" ::: "memory");
        else asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        PH_MARK(seq, 2);
        double *Rt = Rs + (i < S::OWN ? i : S::OWN + buf) * kD * LDR;
        const int Dc = (int)imin64(kD, n - (int64_t)s * kD);
        if (mma_warp) {
            double acc[TPW][2], r_in[TPW][2];
#pragma unroll
            for (int v = 0; v < TPW; ++v)
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    r_in[v][hh] = Rt[c * LDR + ecol(v, hh)];
                    acc[v][hh] = -r_in[v][hh];
                }
            mma_tile(acc, Lh + buf * kD * LDW, Ph);
            PH_MARK(seq, 3);
            const bool hoff = b == s - 2;
            double *rg = res + (int64_t)s * kD * k + (int64_t)c * k;
            double *hg = hand + (int64_t)s * kD * k + (int64_t)c * k;
#pragma unroll
            for (int v = 0; v < TPW; ++v)
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const int e = ecol(v, hh);
                    Rt[c * LDR + e] = -acc[v][hh];
                    if (chained && i >= S::OWN) Rs[(S::OWN + (buf ^ 1)) * kD * LDR + c * LDR + e] = -acc[v][hh];
                    if (c < Dc && e < k) {
                        if (i >= S::OWN) rg[e] = -acc[v][hh];
                        if (hoff) st_value(hg + e, -acc[v][hh]);  // strip s's hand-off to the solver
                    }
                }
            if (b >= 1) {  // checkpoint (b, s): the residual before this tile (after the hand-off stores)
                double *ck = chk + (cks + b) * kD * k + (int64_t)c * k;
#pragma unroll
                for (int v = 0; v < TPW; ++v)
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        const int e = ecol(v, hh);
                        if (c < Dc && e < k) ck[e] = r_in[v][hh];
                    }
            }
        }
        // the next row's P, issued after this tile's MMA (issued at the tile's top it came back
        // empty whenever the helpers trail the solver by less than a step, and was polled again)
        if (valid(nx) && nx.b != b && pn_b != nx.b) issue_p(nx.b);
        asm volatile("fence.acq_rel.cta;" ::: "memory");  // spilled residuals: stores before a later tile's copies read them
        __syncthreads();
        if (t == 0) {  // tile (b, s): checkpoint written, L tile consumed (the overlapped Apply's cue),
                       // released every kPcRel tiles: one fence (an L2 round trip on this CTA's
                       // critical path) per kPcRel tiles, the counts are fire-and-forget
            rel_b[nrel++] = b;
            if (nrel == kPcRel || !valid(nx)) {
                fence_acq_rel_gpu();
                for (int q = 0; q < nrel; ++q) atomicAdd(rowcnt + rel_b[q], 1u);
                nrel = 0;
            }
        }
        cur = nx;
        buf ^= 1;
        ++seq;
    }
}

// Q_b = P_b^T P_b per 64-row block (KB x KB, zero padded)
// (the block's P rows are staged in shared memory by coalesced loads, all in flight at once: the
// per-entry loop over global rows was a chain of 64 L2 latencies on the tail's critical path)
template <int KB>
__global__ void pgram_kernel(const double *__restrict__ P, int64_t n, int k, double *Q, int b0 = 0) {
    __shared__ double Ps[kD][KB + 1];
    const int b = b0 + blockIdx.x;
    const int64_t r0 = (int64_t)b * kD;
    const int Db = (int)imin64(kD, n - r0);
    for (int o = threadIdx.x; o < kD * KB; o += blockDim.x) {
        const int m = o / KB, e = o % KB;
        Ps[m][e] = (m < Db && e < k) ? P[(r0 + m) * k + e] : 0.0;
    }
    __syncthreads();
    for (int o = threadIdx.x; o < KB * KB; o += blockDim.x) {
        const int i = o / KB, j = o % KB;
        double s = 0.0;
        for (int m = 0; m < Db; ++m) s = fma(Ps[m][i], Ps[m][j], s);
        Q[(int64_t)b * KB * KB + o] = s;
    }
}
// G_b = sum_{b' < b} Q_b' (exclusive prefix; one thread per entry)
template <int KB>
__global__ void pscan_kernel(const double *__restrict__ Q, int NB, double *G) {
    const int o = threadIdx.x;
    if (o >= KB * KB) return;
    double run = 0.0;
    for (int b = 0; b < NB; ++b) {
        const double q = Q[(int64_t)b * KB * KB + o];
        G[(int64_t)b * KB * KB + o] = run;
        run += q;
    }
}

// G_b for b in [b0, b1), continuing the prefix of the blocks before b0 (row-block chunks of the
// persistent chain's overlapped tail, in order on one stream)
template <int KB>
__global__ void pscan_range_kernel(const double *__restrict__ Q, int b0, int b1, double *G) {
    const int o = threadIdx.x;
    if (o >= KB * KB) return;
    double run = b0 == 0 ? 0.0 : G[(int64_t)(b0 - 1) * KB * KB + o] + Q[(int64_t)(b0 - 1) * KB * KB + o];
    for (int b = b0; b < b1; ++b) {
        const double q = Q[(int64_t)b * KB * KB + o];
        G[(int64_t)b * KB * KB + o] = run;
        run += q;
    }
}
// waits until every tile (b, s), s > b, of row blocks b0 .. b1-1 is checkpointed and its L tile
// consumed (rowcnt[b] = tiles of row b: NB - 2 - b helper tiles + one per solver CTA)
__global__ void pwait_rows_kernel(const unsigned *rowcnt, int b0, int b1, int NB, int NS) {
    for (int b = b0 + (int)threadIdx.x; b < b1; b += blockDim.x) {
        const unsigned want = (unsigned)(NB - 2 - b + NS);
        if (b > NB - 2) continue;
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(rowcnt + b) : "memory");
            if (v != want) __nanosleep(256);
        } while (v != want);
    }
}

// the diagonal sweeps of this rank's 64-row diagonal blocks (bdiag_body, global indexing of
// L and V shifted onto the local columns)
template <int KB>
__global__ void __launch_bounds__(kDiagThreads) pdiag_kernel(double *L, int64_t ldl, int64_t n, double *V, int64_t ldv,
                                                           int k, int sigma, const double *P, double *Ui,
                                                           const double *G, double *panels, unsigned long long *key,
                                                           int64_t ebase, const int *dl_b, const int64_t *dl_lc) {
    extern __shared__ double smem_pd[];
    const int b = dl_b[blockIdx.x];
    const int64_t shift = dl_lc[blockIdx.x] - (int64_t)b * kD;  // local column - global column
    bdiag_body<KB>(L + shift * ldl, n, ldl, V + shift, ldv, k, sigma, P, false, Ui, G, panels, key, ebase, b, smem_pd);
}

// this rank's panels and U_b^{-1} to every other rank (device-initiated puts), then the
// flags of PEER mode
template <int KB>
__global__ void pbcast_kernel(const int *dl_b, int ndl, const double *panels, const double *Ui, Peers peers, int self,
                              unsigned epoch) {
    constexpr int PD = panel_doubles(KB), UD = KB * KB;
    for (int i = blockIdx.x; i < ndl; i += gridDim.x) {
        const int b = dl_b[i];
        for (int r = 0; r < peers.R; ++r) {
            if (r == self) continue;
            for (int o = threadIdx.x; o < PD; o += blockDim.x)
                peers.dst[r][(int64_t)b * PD + o] = panels[(int64_t)b * PD + o];
            for (int o = threadIdx.x; o < UD; o += blockDim.x)
                peers.dst2[r][(int64_t)b * UD + o] = Ui[(int64_t)b * UD + o];
        }
    }
    if (peers.flag[0]) {  // PEER mode: count this rank in on every peer's panel barrier
        __threadfence_system();
        __syncthreads();
        if (threadIdx.x == 0)
            for (int r = 0; r < peers.R; ++r) atomicAdd_system(peers.flag[r], 1u);
    }
}
// PEER mode: wait until all R ranks have published their panels for this call
__global__ void pwait_kernel(const unsigned *ctr, unsigned target) {
    if (threadIdx.x == 0)
        while ((int)(ld_acquire_sys(ctr) - target) < 0) __nanosleep(200);
}

template <int KB>
__global__ void __launch_bounds__(kT2Threads, 2) papply_kernel(const __grid_constant__ CUtensorMap tm, int64_t n,
                                                              int k, const double *__restrict__ chk,
                                                              const double *__restrict__ Ui,
                                                              const double *__restrict__ panels, int NB,
                                                              const int2 *items, ApplyMap map) {
    extern __shared__ __align__(16) unsigned char smem_pa[];
    const int2 it = items[blockIdx.x];
    btma_body<KB>(tm, n, k, chk, Ui, panels, NB, it.x, it.y, smem_pa, 0, map);
}

// one 64 x 64 tile (b, local strip sl) of the diagonal column block (or any tile when L is
// not TMA-addressable): thread = column, V state U_b^{-1} r from the checkpoint, 8-row chunks
// through registers; only the tile's own columns are read and written.
template <int KB>
__global__ void __launch_bounds__(kD) ptile_kernel(double *L, int64_t ldl, int64_t nloc, int k,
                                                  const double *__restrict__ chk, const double *__restrict__ Ui,
                                                  const double *__restrict__ panels, const int2 *items,
                                                  const int64_t *chkoff) {
    __shared__ double2 cs[kD * KB];
    __shared__ double rho[kD], nu[KB], Us[KB * KB];
    const int2 it = items[blockIdx.x];
    const int b = it.x, sl = it.y, c = threadIdx.x;
    const double *pan = panels + (int64_t)b * panel_doubles(KB);
    for (int i = c; i < kD * KB; i += kD) cs[i] = make_double2(pan[2 * i], pan[2 * i + 1]);
    for (int i = c; i < kD; i += kD) rho[i] = pan[2 * kD * KB + i];
    for (int i = c; i < KB; i += kD) nu[i] = pan[2 * kD * KB + kD + i];
    for (int i = c; i < KB * KB; i += kD) Us[i] = Ui[(int64_t)b * KB * KB + i];
    __syncthreads();
    const int64_t lc = (int64_t)sl * kD + c;
    if (lc >= nloc) return;
    const double *r = chk + (chkoff[sl] + b) * kD * k + (int64_t)c * k;
    double rr[KB], v[KB];
#pragma unroll
    for (int e = 0; e < KB; ++e) rr[e] = e < k ? r[e] : 0.0;
#pragma unroll
    for (int e = 0; e < KB; ++e) {
        double acc = 0.0;
#pragma unroll
        for (int ep = 0; ep <= e; ++ep) acc = fma(Us[e * KB + ep], rr[ep], acc);
        v[e] = acc;
    }
    double *col = L + (int64_t)b * kD + lc * ldl;
    for (int j0 = 0; j0 < kD; j0 += 8) {
        double l[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) l[u] = col[j0 + u];
#pragma unroll
        for (int u = 0; u < 8; ++u) l[u] = apply_row<KB>(l[u], v, cs + (j0 + u) * KB, rho[j0 + u], KB);
#pragma unroll
        for (int u = 0; u < 8; ++u) col[j0 + u] = l[u];
    }
}

// min over the virtual ranks' failure keys into key[0]
struct KeyList {
    unsigned long long *k[kMaxRanks];
    int R;
};
__global__ void keymin_kernel(unsigned long long *key0, KeyList keys) {
    unsigned long long m = ~0ull;
    for (int r = 0; r < keys.R; ++r) m = min(m, *keys.k[r]);
    *key0 = m;
}

// -------------------------------------------------------------------------- host driver
enum class Mode { Virtual, Nccl, Peer };

struct Rank {
    double *L;
    int64_t ldl;
    double *V;  // local V rows (ld nloc)
    Plan plan;
    Carve cv;
    char *ws;
    CUtensorMap tm;
    bool tma;
    // PEER mode: the replicated buffers live in the comm's IPC window (peers write into them)
    double *Pw = nullptr, *panw = nullptr, *Uw = nullptr;
    template <typename T>
    T *at(size_t off) const {
        return reinterpret_cast<T *>(ws + off);
    }
    double *Pbuf() const { return Pw ? Pw : at<double>(cv.P); }
    double *panbuf() const { return panw ? panw : at<double>(cv.panels); }
    double *Ubuf() const { return Uw ? Uw : at<double>(cv.U); }
};

template <int KB>
size_t dsolve_smem() {
    using S = DsShape<KB>;
    return (size_t)(3 * kD * S::LDW + kD * S::LDR + (KB <= 16 ? kDsMaxRows : kDsMaxRows / 2) * S::LDR) * 8;
}
template <int KB>
size_t pupdate_smem() {
    return (size_t)(2 * kD * PuShape<KB>::LDT + 2 * kD * KB) * 8;
}
template <int KB>
size_t pdiag_smem() {
    return (size_t)bdiag_smem_doubles(KB) * sizeof(double);
}

struct Exchange {
    Mode mode;
    unsigned *epoch;   // Peer mode: the comm's call counter (identical on every rank); else the workspace's
    void *nccl;        // ncclComm_t (Nccl / Peer modes)
    int self;          // this process's rank (Nccl / Peer); 0 in Virtual mode
    double **peerP;    // Peer mode: every rank's P, panels, Ui buffers and flag words (IPC-mapped)
    double **peerPan;
    double **peerU;
    unsigned **peerFlag;
    unsigned **peerCtr;
};

// The library's auxiliary stream on the current device (the residual updates that overlap the
// next diagonal solve) and two event pairs for the hand-offs between it and the call's stream.
std::mutex g_aux_mutex;
constexpr int kTailStreams = 8;
constexpr size_t kTailGraphs = 4;  // e.g. one per sigma for a caller alternating update/downdate
struct Aux {
    cudaStream_t s = nullptr;
    cudaEvent_t ready[2] = {nullptr, nullptr}, done[2] = {nullptr, nullptr};
    // the persistent chain's overlapped tail: one stream per chunk, its prefix-Gram and done events
    cudaStream_t par[kTailStreams] = {};
    cudaEvent_t scan[kTailStreams] = {}, pdone[kTailStreams] = {}, wdone[kTailStreams] = {};
    // the tail as a CUDA graph (pchain_tail), replayed while its arguments are unchanged
    struct TailGraph {
        std::vector<unsigned char> key;
        cudaGraphExec_t exec = nullptr;
        int launches = 0;
    };
    std::vector<TailGraph> tails;                   // most recent first, at most kTailGraphs
    std::vector<std::vector<unsigned char>> seen;   // argument sets seen without a graph (same cap)
    cudaEvent_t tfork = nullptr, tdone = nullptr;
};
// keyed by (device, call stream) like the workspaces: calls on different streams (host threads)
// never share the auxiliary stream or its events
std::map<std::pair<int, cudaStream_t>, Aux> g_aux;
gcm_status_t aux_stream(cudaStream_t call, cudaStream_t *s, cudaEvent_t **ready, cudaEvent_t **done) {
    int dev = 0;
    gcm_status_t st = check_cuda(cudaGetDevice(&dev));
    if (st != GCM_OK) return st;
    std::lock_guard<std::mutex> lock(g_aux_mutex);
    Aux &a = g_aux[{dev, call}];
    if (!a.s) {
        st = check_cuda(cudaStreamCreateWithFlags(&a.s, cudaStreamNonBlocking));
        for (int i = 0; i < 2 && st == GCM_OK; ++i) {
            st = check_cuda(cudaEventCreateWithFlags(&a.ready[i], cudaEventDisableTiming));
            if (st == GCM_OK) st = check_cuda(cudaEventCreateWithFlags(&a.done[i], cudaEventDisableTiming));
        }
        for (int i = 0; i < kTailStreams && st == GCM_OK; ++i) {
            st = check_cuda(cudaStreamCreateWithFlags(&a.par[i], cudaStreamNonBlocking));
            if (st == GCM_OK) st = check_cuda(cudaEventCreateWithFlags(&a.scan[i], cudaEventDisableTiming));
            if (st == GCM_OK) st = check_cuda(cudaEventCreateWithFlags(&a.pdone[i], cudaEventDisableTiming));
            if (st == GCM_OK) st = check_cuda(cudaEventCreateWithFlags(&a.wdone[i], cudaEventDisableTiming));
        }
        if (st != GCM_OK) return st;
    }
    *s = a.s;
    *ready = a.ready;
    *done = a.done;
    return GCM_OK;
}
// the tail streams and events of (device, call stream) (created by aux_stream)
Aux *aux_of(cudaStream_t call) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) clear_stale_error();
    std::lock_guard<std::mutex> lock(g_aux_mutex);
    return &g_aux[{dev, call}];
}

// GCM_PANEL_TRACE=1 (debug): timing events around every solve block's kernels (solve, lookahead
// on the call stream; the rest on the aux stream) and a per-phase summary on stderr after the
// pass -- how much of the chain is the solve, the lookahead, and waiting for the rest.
struct ChainTrace {
    bool on = false;
    std::vector<cudaEvent_t> ev;  // per block: [solve start, solve end, lookahead end, rest end]
    explicit ChainTrace(int NSB) {
        on = std::getenv("GCM_PANEL_TRACE") != nullptr;
        if (!on) return;
        ev.resize((size_t)NSB * 4);
        for (auto &e : ev) cudaEventCreate(&e);
    }
    void rec(int g, int i, cudaStream_t s) {
        if (on) cudaEventRecord(ev[(size_t)g * 4 + i], s);
    }
    void report(int NSB) {
        if (!on) return;
        cudaEventSynchronize(ev.back());
        cudaDeviceSynchronize();
        double tot[4] = {0, 0, 0, 0};  // solve, lookahead, rest, gap before the next solve
        for (int g = 0; g < NSB; ++g) {
            float a = 0, b = 0, c = 0, d = 0;
            cudaEventElapsedTime(&a, ev[g * 4 + 0], ev[g * 4 + 1]);
            cudaEventElapsedTime(&b, ev[g * 4 + 1], ev[g * 4 + 2]);
            cudaEventElapsedTime(&c, ev[g * 4 + 2], ev[g * 4 + 3]);
            if (g + 1 < NSB) cudaEventElapsedTime(&d, ev[g * 4 + 2], ev[(g + 1) * 4 + 0]);
            tot[0] += a, tot[1] += b, tot[2] += c, tot[3] += d;
        }
        float all = 0;
        cudaEventElapsedTime(&all, ev[0], ev.back());
        std::fprintf(stderr,
                     "gcm panel trace: %d blocks, chain %.3f ms: solve %.3f, lookahead %.3f, gap %.3f; "
                     "rest (aux, overlapped) %.3f ms\n",
                     NSB, all, tot[0], tot[1], tot[3], tot[2]);
        for (auto &e : ev) cudaEventDestroy(e);
    }
};

// One rank: the persistent chain while each helper owns a few strips; at n ~ 1e5 (10+ strips per
// helper) the per-solve-block launches, whose residual updates spread over every SM, are faster
// (68.2 vs 71.9 ms; n = 40000: 14.1 vs 12.3 ms).  GCM_PCHAIN=0 / 1 forces either (A/B, tests).
bool pchain_enabled(int NB64) {
    const char *e = std::getenv("GCM_PCHAIN");
    if (e) return e[0] != '0';
    int dev = 0, nsm = 148;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        clear_stale_error();
    return NB64 - 2 <= 6 * (nsm - 1);
}
template <int KB>
gcm_status_t pchain_launch(Rank &q, int64_t n, int k, int NB64, cudaStream_t stream, cudaEvent_t armed, int reserve) {
    double *hand = q.at<double>(q.cv.sflag);
    unsigned *rowcnt = q.at<unsigned>(q.cv.rowcnt);
    // P and the hand-offs start all-ones (the "not yet written" pattern consumers poll for) and
    // rowcnt zero: armed by this pass's pinit_kernel
    gcm_status_t st = GCM_OK;
    ht_mark("memsets");
    if (armed) st = check_cuda(cudaEventRecord(armed, stream));  // the overlapped tail starts after this
    if (st != GCM_OK) return st;
    const size_t smem = pchain_smem<KB>();
    static DevOnce once;
    static int nsm_c[64], per_sm_c[64];
    const int dev = cur_device();
    if (once.first(dev)) {
        int nsm = 0, per_sm = 0;
        st = check_cuda(cudaFuncSetAttribute(pchain_kernel<KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        if (st == GCM_OK) st = check_cuda(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        if (st == GCM_OK)
            st = check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pchain_kernel<KB>, kPcT, smem));
        if (st != GCM_OK) return st;
        nsm_c[dev & 63] = nsm;
        per_sm_c[dev & 63] = per_sm;
        once.done(dev);
    }
    const int nsm = nsm_c[dev & 63], per_sm = per_sm_c[dev & 63];
    if (per_sm < 1) return GCM_ECUDA;
    // the solver + one helper per strip that needs hand-offs (strips 2 ..), at most one CTA per SM
    constexpr int NS = PcShape<KB>::NS;
    // (reserve: SMs left to the overlapped tail's sweeps and Apply while the chain runs)
    int grid = (int)std::max(NS, std::min(nsm * per_sm - reserve, NS + std::max(0, NB64 - 2)));
    // GCM_PCHAIN_GRID=<g> caps the grid (tests: few helpers own many strips -> the spill slots)
    if (const char *e = std::getenv("GCM_PCHAIN_GRID")) grid = std::max(NS + 1, std::min(grid, std::atoi(e)));
    if (grid <= NS && NB64 > 2) grid = NS + 1;
    const double *L = q.L;
    int64_t ldl = q.ldl;
    double *res = q.at<double>(q.cv.res), *chk = q.at<double>(q.cv.chk), *P = q.Pbuf();
    const int64_t *chkoff = q.at<int64_t>(q.cv.chkoff);
    const double *W = q.at<double>(q.cv.Winv);
    void *args[] = {(void *)&L, &ldl, &n, &k, &NB64, &res, &chk, (void *)&chkoff, (void *)&W, &P, &hand, &rowcnt};
    st = check_cuda(cudaLaunchCooperativeKernel((const void *)pchain_kernel<KB>, dim3(grid), dim3(kPcT), args, smem,
                                                stream));
    count_launch();
    return st;
}

// The persistent chain's tail -- prefix Grams, diagonal sweeps and the Apply -- row block by row
// block while the chain still runs: chunk c's kernels go to the auxiliary stream behind a
// pwait_rows_kernel that waits for the chunk's row counters (every tile of those rows
// checkpointed, its L tile consumed), so they run on the SMs the chain leaves free (or frees
// as its helpers finish); the last chunk runs on the call's stream after the chain.
template <int KB>
gcm_status_t pchain_tail(Rank &q, int64_t n, int k, int sigma, int64_t ebase, int NB64, cudaStream_t stream,
                         cudaStream_t aux, cudaEvent_t armed, cudaEvent_t aux_done) {
    constexpr int NS = PcShape<KB>::NS;
    const size_t smem_t2 = t2_smem_bytes(KB);
    gcm_status_t st = GCM_OK;
    static DevOnce once;
    const int dev = cur_device();
    if (once.first(dev)) {
        st = check_cuda(cudaFuncSetAttribute(papply_kernel<KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_t2));
        if (st != GCM_OK) return st;
        once.done(dev);
    }
    // chunks (GCM_PCHAIN_CHUNKS, default 8): all but the last on their own tail streams, in
    // parallel with each other and the chain (profiles/r02by_tail_chunks.txt)
    const char *ce = std::getenv("GCM_PCHAIN_CHUNKS");
    const int want = std::min(kTailStreams + 1, ce ? std::max(1, std::atoi(ce)) : 8);
    const int cs = std::max(4, (NB64 + want - 1) / want);
    Aux *ax = aux_of(stream);
    ApplyMap map{q.at<int>(q.cv.gstrip), q.at<int64_t>(q.cv.chkoff), q.plan.nloc};
    int nl = 0;  // kernels enqueued (a graph replay counts its captured ones)
    // chunk ci's row wait starts after chunk ci-1's has returned: at most ONE spinning CTA can be
    // resident before the cooperative chain is, and the chain's grid leaves an SM for it (a
    // spinner per chunk could take the SMs a full-width chain grid needs: deadlock)
    auto chunk = [&](int ci, int B0, int B1, cudaStream_t s, bool wait, cudaEvent_t scan_wait,
                     cudaEvent_t scan_rec) -> gcm_status_t {
        if (wait) {
            if (ci > 0) {
                const gcm_status_t s0 = check_cuda(cudaStreamWaitEvent(s, ax->wdone[ci - 1], 0));
                if (s0 != GCM_OK) return s0;
            }
            pwait_rows_kernel<<<1, 64, 0, s>>>(q.at<unsigned>(q.cv.rowcnt), B0, B1, NB64, NS);
            count_launch();
            ++nl;
            if (ci < kTailStreams) {
                const gcm_status_t s1 = check_cuda(cudaEventRecord(ax->wdone[ci], s));
                if (s1 != GCM_OK) return s1;
            }
        }
        pgram_kernel<KB><<<B1 - B0, KB * KB <= 1024 ? KB * KB : 1024, 0, s>>>(q.Pbuf(), n, k, q.at<double>(q.cv.Q), B0);
        if (scan_wait) {  // the previous chunk's prefix (G continues across chunks)
            const gcm_status_t s2 = check_cuda(cudaStreamWaitEvent(s, scan_wait, 0));
            if (s2 != GCM_OK) return s2;
        }
        pscan_range_kernel<KB><<<1, KB * KB, 0, s>>>(q.at<double>(q.cv.Q), B0, B1, q.at<double>(q.cv.G));
        if (scan_rec) {
            const gcm_status_t s2 = check_cuda(cudaEventRecord(scan_rec, s));
            if (s2 != GCM_OK) return s2;
        }
        pdiag_kernel<KB><<<B1 - B0, kDiagThreads, pdiag_smem<KB>(), s>>>(
            q.L, q.ldl, n, q.V, std::max<int64_t>(q.plan.nloc, 1), k, sigma, q.Pbuf(), q.Ubuf(),
            q.at<double>(q.cv.G), q.panbuf(), q.at<unsigned long long>(q.cv.key), ebase, q.at<int>(q.cv.dlb) + B0,
            q.at<int64_t>(q.cv.dllc) + B0);
        count_launch(3);
        nl += 3;
        const int f0 = q.plan.full_off[B0], f1 = q.plan.full_off[B1];
        const int t0 = q.plan.tiles_off[B0], t1 = q.plan.tiles_off[B1];
        if (q.tma && f1 > f0) {
            papply_kernel<KB><<<(unsigned)(f1 - f0), kT2Threads, smem_t2, s>>>(
                q.tm, n, k, q.at<double>(q.cv.chk), q.Ubuf(), q.panbuf(), NB64, q.at<int2>(q.cv.full) + f0, map);
            count_launch();
            ++nl;
        }
        if (t1 > t0) {
            ptile_kernel<KB><<<(unsigned)(t1 - t0), kD, 0, s>>>(q.L, q.ldl, q.plan.nloc, k, q.at<double>(q.cv.chk),
                                                               q.Ubuf(), q.panbuf(), q.at<int2>(q.cv.tiles) + t0,
                                                               q.at<int64_t>(q.cv.chkoff));
            count_launch();
            ++nl;
        }
        return check_cuda(cudaGetLastError());
    };
    // chunk c (all but the last) on tail stream c: its sweeps and Apply run in parallel with the
    // other chunks' (only the prefix-Gram scan is ordered across chunks, by events)
    (void)aux;
    (void)aux_done;
    const int nchunks = (NB64 + cs - 1) / cs;
    // The tail as ONE CUDA graph on the aux stream (GCM_TAIL_GRAPH=0: enqueued directly): its ~90
    // launches and event operations cost ~250 us of host time per call -- longer than the chain
    // runs at n = 5000, so the GPU waited on the host for the last chunks.  Captured once per
    // argument set (buffers, sizes, tensor map) and replayed; every chunk polls its rows (the
    // graph is not stream-ordered after the chain).
    const char *ge = std::getenv("GCM_TAIL_GRAPH");
    if (!(ge && ge[0] == '0') && ax->s) {
        std::vector<unsigned char> key;
        auto add = [&](const void *p, size_t bytes) {
            const unsigned char *b = static_cast<const unsigned char *>(p);
            key.insert(key.end(), b, b + bytes);
        };
        const int kb = KB;
        add(&kb, sizeof kb), add(&n, sizeof n), add(&k, sizeof k), add(&sigma, sizeof sigma), add(&ebase, sizeof ebase);
        add(&NB64, sizeof NB64), add(&nchunks, sizeof nchunks), add(&q.L, sizeof q.L), add(&q.ldl, sizeof q.ldl);
        add(&q.V, sizeof q.V), add(&q.plan.nloc, sizeof q.plan.nloc), add(&q.ws, sizeof q.ws), add(&q.Pw, sizeof q.Pw);
        add(&q.panw, sizeof q.panw), add(&q.Uw, sizeof q.Uw), add(&q.tma, sizeof q.tma), add(&q.tm, sizeof q.tm);
        add(&q.cv, sizeof q.cv), add(&cs, sizeof cs), add(&q.plan.nb, sizeof q.plan.nb);
        int hit = -1;
        for (size_t i = 0; i < ax->tails.size(); ++i)
            if (ax->tails[i].key == key) hit = (int)i;
        // capture on the second call with one argument set (a caller whose buffers change every
        // call keeps the direct path instead of paying a capture per call)
        bool repeat = false;
        if (hit < 0) {
            for (auto it = ax->seen.begin(); it != ax->seen.end(); ++it)
                if (*it == key) {
                    repeat = true;
                    ax->seen.erase(it);
                    break;
                }
            if (!repeat) {
                ax->seen.insert(ax->seen.begin(), key);
                if (ax->seen.size() > kTailGraphs) ax->seen.pop_back();
            }
        }
        if (repeat) {
            if (!ax->tfork) st = check_cuda(cudaEventCreateWithFlags(&ax->tfork, cudaEventDisableTiming));
            if (st == GCM_OK && !ax->tdone) st = check_cuda(cudaEventCreateWithFlags(&ax->tdone, cudaEventDisableTiming));
            if (st != GCM_OK) return st;
            cudaGraph_t g = nullptr;
            cudaGraphExec_t exec = nullptr;
            nl = 0;
            bool cap = cudaStreamBeginCapture(ax->s, cudaStreamCaptureModeRelaxed) == cudaSuccess;
            gcm_status_t cs2 = cap ? check_cuda(cudaEventRecord(ax->tfork, ax->s)) : GCM_ECUDA;
            for (int c = 0; c + 1 < nchunks && cs2 == GCM_OK; ++c) {
                cs2 = check_cuda(cudaStreamWaitEvent(ax->par[c], ax->tfork, 0));
                if (cs2 == GCM_OK)
                    cs2 = chunk(c, c * cs, (c + 1) * cs, ax->par[c], true, c > 0 ? ax->scan[c - 1] : nullptr, ax->scan[c]);
                if (cs2 == GCM_OK) cs2 = check_cuda(cudaEventRecord(ax->pdone[c], ax->par[c]));
            }
            if (cs2 == GCM_OK)
                cs2 = chunk(nchunks - 1, (nchunks - 1) * cs, NB64, ax->s, true, nchunks > 1 ? ax->scan[nchunks - 2] : nullptr, nullptr);
            for (int c = 0; c + 1 < nchunks && cs2 == GCM_OK; ++c)
                cs2 = check_cuda(cudaStreamWaitEvent(ax->s, ax->pdone[c], 0));
            if (cap) {
                const bool ended = cudaStreamEndCapture(ax->s, &g) == cudaSuccess;
                if (!(cs2 == GCM_OK && ended && g && cudaGraphInstantiate(&exec, g, 0) == cudaSuccess)) exec = nullptr;
                if (g) cudaGraphDestroy(g);
            }
            count_launch(-nl);  // the capture's launches never ran; a replay counts them
            if (exec) {
                if (ax->tails.size() >= kTailGraphs) {
                    cudaGraphExecDestroy(ax->tails.back().exec);
                    ax->tails.pop_back();
                }
                Aux::TailGraph tg;
                tg.key = key;
                tg.exec = exec;
                tg.launches = nl;
                ax->tails.insert(ax->tails.begin(), std::move(tg));
                hit = 0;
            } else {  // capture unsupported or failed: enqueue directly (below)
                clear_stale_error();
            }
        }
        const bool ok = hit >= 0;
        if (ok && hit > 0) std::swap(ax->tails[0], ax->tails[hit]);  // most recent first
        if (ok) {
            st = check_cuda(cudaStreamWaitEvent(ax->s, armed, 0));
            if (st == GCM_OK) st = check_cuda(cudaGraphLaunch(ax->tails[0].exec, ax->s));
            if (st == GCM_OK) st = check_cuda(cudaEventRecord(ax->tdone, ax->s));
            if (st == GCM_OK) st = check_cuda(cudaStreamWaitEvent(stream, ax->tdone, 0));
            count_launch(ax->tails[0].launches);
            return st;
        }
    }
    for (int c = 0; c + 1 < nchunks && st == GCM_OK; ++c) {
        cudaStream_t s = ax->par[c];
        st = check_cuda(cudaStreamWaitEvent(s, armed, 0));
        if (st == GCM_OK)
            st = chunk(c, c * cs, (c + 1) * cs, s, true, c > 0 ? ax->scan[c - 1] : nullptr, ax->scan[c]);
        if (st == GCM_OK) st = check_cuda(cudaEventRecord(ax->pdone[c], s));
    }
    if (st != GCM_OK) return st;
    st = chunk(nchunks - 1, (nchunks - 1) * cs, NB64, stream, false, nchunks > 1 ? ax->scan[nchunks - 2] : nullptr, nullptr);
    for (int c = 0; c + 1 < nchunks && st == GCM_OK; ++c) st = check_cuda(cudaStreamWaitEvent(stream, ax->pdone[c], 0));
    return st;
}

// one pass (<= 32 update columns) over all ranks of `rk` (Virtual: all R; else rk has one entry)
template <int KB>
gcm_status_t panel_pass(std::vector<Rank> &rk, int R, int64_t n, int64_t nb, int k, int sigma, int64_t ebase,
                        unsigned epoch, const Exchange &x, cudaStream_t stream) {
    gcm_status_t st = GCM_OK;
    const int nloc_ranks = (int)rk.size();
    // one rank: the persistent chain, with its tail overlapped unless GCM_PCHAIN_TAIL=0
    const int NB64_ = (int)((n + kD - 1) / kD);
    const bool use_pchain = R == 1 && x.mode == Mode::Virtual && pchain_enabled(NB64_);
    const char *tail_env = std::getenv("GCM_PCHAIN_TAIL");
    bool tail_overlap = use_pchain && !(tail_env && tail_env[0] == '0');
    const int NBc = (int)((n + nb - 1) / nb), NB64 = (int)((n + kD - 1) / kD);
    auto peers_P = [&](int owner_local) {
        Peers p{};
        if (x.mode == Mode::Virtual) {
            p.R = R;
            for (int r = 0; r < R; ++r) p.dst[r] = rk[r].Pbuf();
        } else if (x.mode == Mode::Nccl) {
            p.R = 1;
            p.dst[0] = rk[owner_local].Pbuf();
        } else {
            p.R = R;
            for (int r = 0; r < R; ++r) p.dst[r] = x.peerP[r];
        }
        return p;
    };
    static DevOnce attr_once;
    const int dev = cur_device();
    if (attr_once.first(dev))
        st = check_cuda(cudaFuncSetAttribute(dsolve_kernel<KB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)dsolve_smem<KB>()));
    else
        st = GCM_OK;
    const bool set_attrs = attr_once.first(dev);
    if (st == GCM_OK && set_attrs)
        st = check_cuda(cudaFuncSetAttribute(pupdate_kernel<KB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)pupdate_smem<KB>()));
    if (st == GCM_OK && set_attrs)
        st = check_cuda(cudaFuncSetAttribute(pupdate_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)pupdate_smem<8>()));
    if (st == GCM_OK && set_attrs)
        st = check_cuda(cudaFuncSetAttribute(pupdate_mma_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)pupdate_mma_smem<8>()));
    constexpr int KBM = KB >= 8 ? KB : 8;  // (KB = 4 keeps the DFMA kernel)
    if (st == GCM_OK && set_attrs)
        st = check_cuda(cudaFuncSetAttribute(pupdate_mma_kernel<KBM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)pupdate_mma_smem<KBM>()));
    // GCM_PU_DFMA=1: the residual updates on the DFMA kernel (A/B against the tensor-core one)
    const bool pu_mma = KB >= 8 && std::getenv("GCM_PU_DFMA") == nullptr;
    if (st == GCM_OK && set_attrs)
        st = check_cuda(cudaFuncSetAttribute(pdiag_kernel<KB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)pdiag_smem<KB>()));
    if (st != GCM_OK) return st;
    if (set_attrs) attr_once.done(dev);
    // 1. residuals = V, tile (0, s) checkpoints
    for (auto &q : rk) {
        if (q.plan.nsl == 0) continue;
        const bool arm = use_pchain;  // the persistent chain's P / hand-off / rowcnt arming
        pinit_kernel<<<q.plan.nsl, kPT, 0, stream>>>(
            q.V, std::max<int64_t>(q.plan.nloc, 1), q.plan.nloc, k, q.at<int>(q.cv.gstrip), q.at<int64_t>(q.cv.chkoff),
            q.at<double>(q.cv.res), q.at<double>(q.cv.chk),
            arm ? reinterpret_cast<unsigned long long *>(q.Pbuf()) : nullptr, arm ? n * k : 0,
            arm ? q.at<unsigned long long>(q.cv.sflag) : nullptr, arm ? (int64_t)NB64 * kD * k : 0,
            arm ? q.at<unsigned>(q.cv.rowcnt) : nullptr, arm ? NB64 : 0);
        count_launch();
    }
    ht_mark("pinit");
    // 2. the right-looking solve over column blocks
    {
        // (with the overlapped tail the scope holds the whole pass: 'pchain')
        ProfScope ps(tail_overlap ? "pchain" : "ptrsv", stream);
        for (auto &q : rk) {  // inverses of the diagonal blocks the solve chain multiplies by
            if (q.plan.nsl == 0) continue;
            pinv_kernel<<<q.plan.nsl, kD, 0, stream>>>(q.L, q.ldl, n, q.at<int>(q.cv.gstrip),
                                                       q.at<double>(q.cv.Winv));
            count_launch();
        }
        if (use_pchain) {
            cudaStream_t aux = nullptr;
            cudaEvent_t *ev_a = nullptr, *ev_b = nullptr;
            st = aux_stream(stream, &aux, &ev_a, &ev_b);
            if (st != GCM_OK) return st;
            // GCM_PCHAIN_RESERVE=<m>: SMs kept free of chain CTAs for the overlapped tail (default 0)
            const char *re = std::getenv("GCM_PCHAIN_RESERVE");
            // (the overlapped tail: at least one SM for its single spinning row-wait CTA)
            const int reserve = tail_overlap ? std::max(1, re ? std::atoi(re) : 0) : 0;
            ht_mark("pinv");
            st = pchain_launch<KB>(rk[0], n, k, NB64, stream, tail_overlap ? ev_a[0] : nullptr, reserve);
            ht_mark("pchain");
            if (st == GCM_OK && tail_overlap)
                st = pchain_tail<KB>(rk[0], n, k, sigma, ebase, NB64, stream, aux, ev_a[0], ev_b[0]);
            ht_mark("tail");
            if (st != GCM_OK) return st;
        } else {
            cudaStream_t aux = nullptr;
            cudaEvent_t *p_ready = nullptr, *rest_done = nullptr;
            st = aux_stream(stream, &aux, &p_ready, &rest_done);
            if (st != GCM_OK) return st;
            st = check_cuda(cudaEventRecord(p_ready[1], stream));  // the aux stream starts after this call's prologue
            if (st == GCM_OK) st = check_cuda(cudaStreamWaitEvent(aux, p_ready[1], 0));
            if (st != GCM_OK) return st;
            const int64_t sb = rk[0].plan.sb;
            const int NSB = rk[0].plan.NSB;
            ChainTrace tr(NSB);
            for (int g = 0; g < NSB; ++g) {  // solve blocks of sb rows (sb divides nb)
                const int64_t row0 = (int64_t)g * sb;
                tr.rec(g, 0, stream);
                const int owner = (int)((row0 / nb) % R);
                const int nrows = (int)std::min<int64_t>(sb, n - row0);
                const int ol = x.mode == Mode::Virtual ? owner : (owner == x.self ? 0 : -1);
                if (ol >= 0) {
                    Rank &q = rk[ol];
                    // owner's local strip of row0's column: local block (row0/nb)/R, offset row0 % nb
                    const int sl0 = (int)((((row0 / nb) / R) * nb + row0 % nb) / kD);
                    Peers p = peers_P(ol);
                    if (x.mode == Mode::Peer)
                        for (int r = 0; r < R; ++r) p.flag[r] = x.peerFlag[r] + g;
                    dsolve_kernel<KB><<<1, kDsT, dsolve_smem<KB>(), stream>>>(
                        q.L, q.ldl, n, k, row0, nrows, sl0, q.at<double>(q.cv.res), q.at<double>(q.cv.chk),
                        q.at<int64_t>(q.cv.chkoff), q.at<double>(q.cv.Winv), p, epoch);
                    count_launch();
                }
    #ifdef GCM_WITH_NCCL
                if (x.mode == Mode::Nccl) {
                    double *Pg = rk[0].Pbuf() + row0 * k;
                    st = ncclBroadcast(Pg, Pg, (size_t)nrows * k, ncclDouble, owner, (ncclComm_t)x.nccl, stream) ==
                                 ncclSuccess
                             ? GCM_OK
                             : GCM_ENCCL;
                    if (st != GCM_OK) return st;
                }
    #endif
                // lookahead: the strips of the NEXT solve block first, on the call's stream (after the
                // rest of block g-1, which touched the same residuals); the rest on the aux stream,
                // where it overlaps the next diagonal solve
                tr.rec(g, 1, stream);
                if (g >= 1) {
                    st = check_cuda(cudaStreamWaitEvent(stream, rest_done[(g - 1) & 1], 0));
                    if (st != GCM_OK) return st;
                }
                for (int pass = 0; pass < 2; ++pass) {
                    cudaStream_t sp = pass == 0 ? stream : aux;
                    if (pass == 1) {
                        tr.rec(g, 2, stream);
                        st = check_cuda(cudaEventRecord(p_ready[g & 1], stream));
                        if (st == GCM_OK) st = check_cuda(cudaStreamWaitEvent(aux, p_ready[g & 1], 0));
                        if (st != GCM_OK) return st;
                    }
                    for (int ri = 0; ri < nloc_ranks; ++ri) {
                        Rank &q = rk[ri];
                        const int slf = q.plan.first_strip_after[g];
                        const int sla = g + 1 < NSB ? q.plan.first_strip_after[g + 1] : q.plan.nsl;
                        const int s_lo = pass == 0 ? slf : sla, s_hi = pass == 0 ? sla : q.plan.nsl;
                        if (s_lo >= s_hi) continue;
                        const int rank_id = x.mode == Mode::Virtual ? ri : x.self;
                        const unsigned *flag =
                            (x.mode == Mode::Peer && rank_id != owner) ? x.peerFlag[x.self] + g : nullptr;
                        if (pass == 0 && KB > 8 && pu_mma) {  // lookahead: the chain waits on it -- 8 update columns per CTA
                            pupdate_mma_kernel<8><<<dim3(s_hi - s_lo, KB / 8), kPT, pupdate_mma_smem<8>(), sp>>>(
                                q.L, q.ldl, n, q.plan.nloc, k, row0, nrows, s_lo, q.at<double>(q.cv.res),
                                q.at<double>(q.cv.chk), q.at<int64_t>(q.cv.chkoff), q.Pbuf(), flag, epoch);
                        } else if (pu_mma) {
                            pupdate_mma_kernel<KBM><<<s_hi - s_lo, kPT, pupdate_mma_smem<KBM>(), sp>>>(
                                q.L, q.ldl, n, q.plan.nloc, k, row0, nrows, s_lo, q.at<double>(q.cv.res),
                                q.at<double>(q.cv.chk), q.at<int64_t>(q.cv.chkoff), q.Pbuf(), flag, epoch);
                        } else if (pass == 0 && KB > 8) {
                            pupdate_kernel<8><<<dim3(s_hi - s_lo, KB / 8), kPT, pupdate_smem<8>(), sp>>>(
                                q.L, q.ldl, n, q.plan.nloc, k, row0, nrows, s_lo, q.at<double>(q.cv.res),
                                q.at<double>(q.cv.chk), q.at<int64_t>(q.cv.chkoff), q.Pbuf(), flag, epoch);
                        } else {
                            pupdate_kernel<KB><<<s_hi - s_lo, kPT, pupdate_smem<KB>(), sp>>>(
                                q.L, q.ldl, n, q.plan.nloc, k, row0, nrows, s_lo, q.at<double>(q.cv.res),
                                q.at<double>(q.cv.chk), q.at<int64_t>(q.cv.chkoff), q.Pbuf(), flag, epoch);
                        }
                        count_launch();
                    }
                }
                st = check_cuda(cudaEventRecord(rest_done[g & 1], aux));
                tr.rec(g, 3, aux);
                if (st != GCM_OK) return st;
            }
            tr.report(NSB);
            st = check_cuda(cudaStreamWaitEvent(stream, rest_done[(NSB - 1) & 1], 0));  // join the aux stream
            if (st == GCM_OK) st = check_cuda(cudaGetLastError());
            if (st != GCM_OK) return st;
        }
    }
    if (tail_overlap) return check_cuda(cudaGetLastError());  // the tail ran with the chain
    // 3. prefix Grams (replicated), 4. diagonal sweeps of the local diagonal blocks
    {
        ProfScope ps("psweep", stream);
        for (auto &q : rk) {
            pgram_kernel<KB><<<NB64, KB * KB <= 1024 ? KB * KB : 1024, 0, stream>>>(q.Pbuf(), n, k,
                                                                                  q.at<double>(q.cv.Q));
            count_launch();
            pscan_kernel<KB><<<1, KB * KB, 0, stream>>>(q.at<double>(q.cv.Q), NB64, q.at<double>(q.cv.G));
            count_launch();
            if (!q.plan.dl_b.empty()) {
                pdiag_kernel<KB><<<(unsigned)q.plan.dl_b.size(), kDiagThreads, pdiag_smem<KB>(), stream>>>(
                    q.L, q.ldl, n, q.V, std::max<int64_t>(q.plan.nloc, 1), k, sigma, q.Pbuf(),
                    q.Ubuf(), q.at<double>(q.cv.G), q.panbuf(),
                    q.at<unsigned long long>(q.cv.key), ebase, q.at<int>(q.cv.dlb), q.at<int64_t>(q.cv.dllc));
                count_launch();
            }
        }
        // 5. panels and U_b^{-1} to every rank
        if (x.mode == Mode::Virtual || x.mode == Mode::Peer) {
            for (int ri = 0; ri < nloc_ranks; ++ri) {
                Rank &q = rk[ri];
                Peers p{};
                p.R = R;
                for (int r = 0; r < R; ++r) {
                    p.dst[r] = x.mode == Mode::Virtual ? rk[r].panbuf() : x.peerPan[r];
                    p.dst2[r] = x.mode == Mode::Virtual ? rk[r].Ubuf() : x.peerU[r];
                    p.flag[r] = x.mode == Mode::Peer ? x.peerCtr[r] : nullptr;
                }
                const int self = x.mode == Mode::Virtual ? ri : x.self;
                pbcast_kernel<KB><<<std::max<int>(1, std::min<int>(1024, (int)q.plan.dl_b.size())), 256, 0, stream>>>(
                    q.at<int>(q.cv.dlb), (int)q.plan.dl_b.size(), q.panbuf(), q.Ubuf(),
                    p, self, epoch);
                count_launch();
            }
            if (x.mode == Mode::Peer) {
                pwait_kernel<<<1, 32, 0, stream>>>(x.peerCtr[x.self], epoch * (unsigned)R);
                count_launch();
            }
        }
#ifdef GCM_WITH_NCCL
        if (x.mode == Mode::Nccl) {
            ncclGroupStart();
            for (int g = 0; g < NBc; ++g) {
                const int owner = g % R;
                const int b0 = (int)((int64_t)g * nb / kD), b1 = (int)std::min<int64_t>(NB64, ((int64_t)g + 1) * nb / kD);
                double *pan = rk[0].panbuf() + (int64_t)b0 * panel_doubles(KB);
                double *U = rk[0].Ubuf() + (int64_t)b0 * KB * KB;
                ncclBroadcast(pan, pan, (size_t)(b1 - b0) * panel_doubles(KB), ncclDouble, owner,
                              (ncclComm_t)x.nccl, stream);
                ncclBroadcast(U, U, (size_t)(b1 - b0) * KB * KB, ncclDouble, owner, (ncclComm_t)x.nccl, stream);
            }
            if (ncclGroupEnd() != ncclSuccess) return GCM_ENCCL;
        }
#endif
        st = check_cuda(cudaGetLastError());
        if (st != GCM_OK) return st;
    }
    // 6. the Apply of every panel to this rank's tiles
    {
        ProfScope ps("papply", stream);
        const size_t smem_t2 = t2_smem_bytes(KB);
        st = check_cuda(
            cudaFuncSetAttribute(papply_kernel<KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_t2));
        if (st != GCM_OK) return st;
        for (auto &q : rk) {
            ApplyMap map{q.at<int>(q.cv.gstrip), q.at<int64_t>(q.cv.chkoff), q.plan.nloc};
            if (q.tma && !q.plan.full.empty()) {
                papply_kernel<KB><<<(unsigned)q.plan.full.size(), kT2Threads, smem_t2, stream>>>(
                    q.tm, n, k, q.at<double>(q.cv.chk), q.Ubuf(), q.panbuf(), NB64,
                    q.at<int2>(q.cv.full), map);
                count_launch();
            }
            if (!q.plan.tiles.empty()) {
                ptile_kernel<KB><<<(unsigned)q.plan.tiles.size(), kD, 0, stream>>>(
                    q.L, q.ldl, q.plan.nloc, k, q.at<double>(q.cv.chk), q.Ubuf(),
                    q.panbuf(), q.at<int2>(q.cv.tiles), q.at<int64_t>(q.cv.chkoff));
                count_launch();
            }
        }
        st = check_cuda(cudaGetLastError());
    }
    return st;
}

// The host layout arrays live as long as the process (keyed by layout), so the
// asynchronous uploads below never read freed memory.
std::mutex g_plan_mutex;
std::map<std::tuple<int64_t, int64_t, int, int, int, bool>, Plan> g_plans;
const Plan &get_plan(int64_t n, int64_t nb, int R, int r, int k, bool tma) {
    std::lock_guard<std::mutex> lock(g_plan_mutex);
    auto key = std::make_tuple(n, nb, R, r, k, tma);
    auto it = g_plans.find(key);
    if (it == g_plans.end()) {
        it = g_plans.emplace(key, make_plan(n, nb, R, r, k, tma)).first;
        Plan &p = it->second;
        const Carve c = carve(p);
        const size_t bytes = c.total - c.gstrip;
        void *h = nullptr;
        // pageable uploads are staged by the host, one copy at a time (tens of us per call before
        // the first kernel); a failed pinned allocation keeps that path (upload() below)
        if (cudaHostAlloc(&h, bytes, cudaHostAllocDefault) == cudaSuccess) {
            unsigned char *img = static_cast<unsigned char *>(h);
            std::memset(img, 0, bytes);
            auto put = [&](size_t off, const void *src, size_t n_bytes) {
                if (n_bytes) std::memcpy(img + (off - c.gstrip), src, n_bytes);
            };
            put(c.gstrip, p.gstrip.data(), p.gstrip.size() * 4);
            put(c.chkoff, p.chkoff.data(), p.chkoff.size() * 8);
            put(c.dlb, p.dl_b.data(), p.dl_b.size() * 4);
            put(c.dllc, p.dl_lc.data(), p.dl_lc.size() * 8);
            put(c.full, p.full.data(), p.full.size() * 8);
            put(c.tiles, p.tiles.data(), p.tiles.size() * 8);
            p.img = img;
            p.img_bytes = bytes;
        } else {
            (void)cudaGetLastError();
        }
    }
    return it->second;
}

gcm_status_t upload(const Rank &q, cudaStream_t stream) {
    auto up = [&](size_t off, const void *src, size_t bytes) {
        return bytes ? check_cuda(cudaMemcpyAsync(q.ws + off, src, bytes, cudaMemcpyHostToDevice, stream)) : GCM_OK;
    };
    if (q.plan.img) return up(q.cv.gstrip, q.plan.img, q.plan.img_bytes);  // one pinned async copy
    gcm_status_t st = up(q.cv.gstrip, q.plan.gstrip.data(), q.plan.gstrip.size() * 4);
    if (st == GCM_OK) st = up(q.cv.chkoff, q.plan.chkoff.data(), q.plan.chkoff.size() * 8);
    if (st == GCM_OK) st = up(q.cv.dlb, q.plan.dl_b.data(), q.plan.dl_b.size() * 4);
    if (st == GCM_OK) st = up(q.cv.dllc, q.plan.dl_lc.data(), q.plan.dl_lc.size() * 8);
    if (st == GCM_OK) st = up(q.cv.full, q.plan.full.data(), q.plan.full.size() * 8);
    if (st == GCM_OK) st = up(q.cv.tiles, q.plan.tiles.data(), q.plan.tiles.size() * 8);
    return st;
}

// Runs the whole modification for the ranks in `rk` (each with L, ldl, V set).  Virtual
// mode: all R ranks of the job, in this process, on one stream; Nccl / Peer: this process's
// one rank.  d_info receives the global first failure.
gcm_status_t panel_modify(std::vector<Rank> &rk, int R, int64_t n, int64_t nb, int64_t k, int sigma,
                          gcm_info_t *d_info, Exchange x, cudaStream_t stream) {
    HostTrace ht;
    struct HtScope {
        HostTrace *prev;
        explicit HtScope(HostTrace *h) : prev(g_ht) { g_ht = h->on ? h : nullptr; }
        ~HtScope() { g_ht = prev; }
    } ht_scope(&ht);
    gcm_status_t st = GCM_OK;
    const int kc0 = (int)std::min<int64_t>(k, kPassK);
    // workspace: one carve per rank, back to back (sized for the widest pass)
    size_t total = 0;
    std::vector<size_t> base(rk.size());
    for (size_t i = 0; i < rk.size(); ++i) {
        const int r = x.mode == Mode::Virtual ? (int)i : x.self;
        const int64_t nloc = local_cols(n, nb, R, r);
        // the Apply's TMA path needs a tensor map over the local columns (16-byte aligned L,
        // even ldl); otherwise every tile goes through ptile_kernel
        rk[i].tma = nloc > 0 && encode_tmap_f64(&rk[i].tm, rk[i].L, 2, n, nloc, rk[i].ldl, 1, 0, (unsigned)kT2Rows,
                                                 (unsigned)kT2Box, CU_TENSOR_MAP_SWIZZLE_64B);
        rk[i].plan = get_plan(n, nb, R, r, kc0, rk[i].tma);
        rk[i].cv = carve(rk[i].plan);
        base[i] = total;
        total += rk[i].cv.total;
    }
    ht_mark("plan");
    Workspace *ws = nullptr;
    st = get_workspace(stream, total, 1, &ws);
    ht_mark("ws");
    if (st != GCM_OK) return st;
    char *wsb = reinterpret_cast<char *>(ws->panels);
    if (x.mode == Mode::Virtual) {  // one key per rank + the min
        for (size_t i = 0; i < rk.size(); ++i) rk[i].ws = wsb + base[i];
    } else {
        rk[0].ws = wsb;
    }
    for (auto &q : rk) {
        st = upload(q, stream);
        if (st != GCM_OK) return st;
        st = check_cuda(cudaMemsetAsync(q.ws + q.cv.key, 0xff, 8, stream));
        if (st != GCM_OK) return st;
    }
    ht_mark("upload");
    for (int64_t e0 = 0; e0 < k; e0 += kPassK) {
        const int kc = (int)std::min<int64_t>(kPassK, k - e0);
        unsigned *ep = x.epoch ? x.epoch : &ws->epoch;
        if (++*ep == 0xffffffffu || *ep == 0) *ep = 1;
        const unsigned epoch = *ep;
        std::vector<Rank> pass = rk;
        for (auto &q : pass) {
            q.V = q.V + e0 * std::max<int64_t>(q.plan.nloc, 1);
            if (kc != kc0) {  // a narrower last pass: same carve (it is sized for kc0 >= kc)
                Plan p = get_plan(n, nb, R, x.mode == Mode::Virtual ? (int)(&q - pass.data()) : x.self, kc, q.tma);
                p.k = kc;
                q.plan = p;  // identical layout arrays; only k / KB change
            }
        }
#ifdef GCM_WITH_NCCL
        if (x.mode == Mode::Peer) {  // no rank may write into a window another rank still reads
            unsigned long long *kb = rk[0].at<unsigned long long>(rk[0].cv.key);
            if (ncclAllReduce(kb, kb, 1, ncclUint64, ncclMin, (ncclComm_t)x.nccl, stream) != ncclSuccess)
                return GCM_ENCCL;
        }
#endif
        const int KBp = pass[0].plan.KB;
        if (KBp <= 4) st = panel_pass<4>(pass, R, n, nb, kc, sigma, e0, epoch, x, stream);
        else if (KBp <= 8) st = panel_pass<8>(pass, R, n, nb, kc, sigma, e0, epoch, x, stream);
        else if (KBp <= 16) st = panel_pass<16>(pass, R, n, nb, kc, sigma, e0, epoch, x, stream);
        else st = panel_pass<32>(pass, R, n, nb, kc, sigma, e0, epoch, x, stream);
        if (st != GCM_OK) return st;
    }
    // global first failure
    unsigned long long *key0 = rk[0].at<unsigned long long>(rk[0].cv.key);
    if (x.mode == Mode::Virtual && rk.size() > 1) {
        KeyList keys{};
        keys.R = (int)rk.size();
        for (size_t i = 0; i < rk.size(); ++i) keys.k[i] = rk[i].at<unsigned long long>(rk[i].cv.key);
        keymin_kernel<<<1, 1, 0, stream>>>(ws->key, keys);
        count_launch();
        st = check_cuda(cudaGetLastError());
        if (st != GCM_OK) return st;
        return finalize_info(ws->key, d_info, 1, stream);
    }
#ifdef GCM_WITH_NCCL
    if (x.mode != Mode::Virtual) {
        if (ncclAllReduce(key0, key0, 1, ncclUint64, ncclMin, (ncclComm_t)x.nccl, stream) != ncclSuccess)
            return GCM_ENCCL;
    }
#endif
    return finalize_info(key0, d_info, 1, stream);
}

}  // namespace

// GCM_ALGO_PANEL on one GPU: the sharded algorithm with one rank (nb = 512).
gcm_status_t modify_panel(double *L, int64_t n, int64_t ldl, double *V, int64_t k, int sigma, gcm_info_t *d_info,
                          cudaStream_t stream) {
    std::vector<Rank> rk(1);
    rk[0].L = L;
    rk[0].ldl = ldl;
    rk[0].V = V;
    Exchange x{Mode::Virtual, nullptr, nullptr, 0, nullptr, nullptr, nullptr, nullptr, nullptr};
    return panel_modify(rk, 1, n, 512, k, sigma, d_info, x, stream);
}

}  // namespace gcm

using namespace gcm;

extern "C" {

int64_t gcm_dist_local_cols(int64_t n, int64_t nb, int nranks, int rank) { return local_cols(n, nb, nranks, rank); }

int64_t gcm_dist_global_col(int64_t nb, int nranks, int rank, int64_t local_col) {
    if (nb <= 0 || nranks <= 0 || rank < 0 || rank >= nranks || local_col < 0) return -1;
    return global_col(nb, nranks, rank, local_col);
}

int64_t gcm_dist_plan(int64_t n, int64_t nb, int nranks, int rank, int what, int64_t *out, int64_t cap) {
    if (n < 0 || nb <= 0 || nb % kD != 0 || nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks) return -1;
    if (what < 0 || what > 2 || cap < 0 || (cap > 0 && !out)) return -1;
    const Plan &p = get_plan(n, nb, nranks, rank, 1, true);
    int64_t cnt = 0;
    auto put = [&](int64_t v) {
        if (cnt < cap) out[cnt] = v;
        ++cnt;
    };
    if (what == 0) {  // Apply tiles (b, global strip), TMA groups expanded
        for (const int2 &it : p.full)
            for (int q = 0; q < 4 && it.y + q < p.nsl; ++q) {
                const int sl = it.y + q;
                if ((sl * kD) / nb != (it.y * kD) / nb) break;  // groups never leave a column block
                put(it.x);
                put(p.gstrip[sl]);
            }
        for (const int2 &it : p.tiles) {
            put(it.x);
            put(p.gstrip[it.y]);
        }
    } else if (what == 1) {
        for (int b : p.dl_b) put(b);
    } else {
        for (int g = 0; g < p.NBc; ++g)
            if (g % nranks == rank) put(g);
    }
    return cnt;
}

static gcm_status_t dist_args(int64_t n, int64_t nb, int64_t k, int sigma) {
    if (n < 0 || k < 0 || nb <= 0 || nb % kD != 0 || (sigma != 1 && sigma != -1)) return GCM_EINVAL;
    if (n >= (1ll << 31) || k >= (1ll << 22)) return GCM_EINVAL;
    return GCM_OK;
}

gcm_status_t gcm_modify_dist_virtual(int nranks, double *const *L_local, int64_t n, int64_t nb,
                                     const int64_t *ldl_local, double *const *V_local, int64_t k, int sigma,
                                     gcm_info_t *d_info, gcm_stream_t stream_) {
    cudaStream_t stream = (cudaStream_t)stream_;
    if (nranks < 1 || nranks > kMaxRanks || !L_local || !ldl_local || !V_local) return GCM_EINVAL;
    gcm_status_t st = dist_args(n, nb, k, sigma);
    if (st != GCM_OK) return st;
    std::vector<Rank> rk(nranks);
    for (int r = 0; r < nranks; ++r) {
        const int64_t nloc = local_cols(n, nb, nranks, r);
        if (ldl_local[r] < std::max<int64_t>(1, n)) return GCM_EINVAL;
        if (n > 0 && k > 0 && nloc > 0 && (!L_local[r] || !V_local[r])) return GCM_EINVAL;
        rk[r].L = L_local[r];
        rk[r].ldl = ldl_local[r];
        rk[r].V = V_local[r];
    }
    clear_stale_error();
    if (n == 0 || k == 0) return d_info ? check_cuda(cudaMemsetAsync(d_info, 0, sizeof(gcm_info_t), stream)) : GCM_OK;
    Exchange x{Mode::Virtual, nullptr, nullptr, 0, nullptr, nullptr, nullptr, nullptr, nullptr};
    return panel_modify(rk, nranks, n, nb, k, sigma, d_info, x, stream);
}

#ifdef GCM_WITH_NCCL

static gcm_status_t check_nccl(ncclResult_t r) { return r == ncclSuccess ? GCM_OK : GCM_ENCCL; }

gcm_status_t gcm_comm_unique_id(void *host_id_out) {
    if (!host_id_out) return GCM_EINVAL;
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
    ncclUniqueId id;
    gcm_status_t st = check_nccl(ncclGetUniqueId(&id));
    if (st == GCM_OK) std::memcpy(host_id_out, &id, sizeof(id));
    return st;
}

gcm_status_t gcm_comm_init(gcm_comm_t *comm, const void *host_id, int nranks, int rank) {
    if (!comm || !host_id || nranks <= 0 || nranks > kMaxRanks || rank < 0 || rank >= nranks) return GCM_EINVAL;
    clear_stale_error();
    gcm_comm *c = new (std::nothrow) gcm_comm;
    if (!c) return GCM_ENOMEM;
    ncclUniqueId id;
    std::memcpy(&id, host_id, sizeof(id));
    gcm_status_t st = check_nccl(ncclCommInitRank(&c->nc, nranks, id, rank));
    if (st != GCM_OK) {
        delete c;
        return st;
    }
    c->rank = rank;
    c->nranks = nranks;
    *comm = c;
    return GCM_OK;
}

gcm_status_t gcm_comm_destroy(gcm_comm_t comm) {
    if (!comm) return GCM_EINVAL;
    if (comm->win) {
        cudaDeviceSynchronize();
        for (int r = 0; r < comm->nranks; ++r)
            if (r != comm->rank && comm->peers[r]) cudaIpcCloseMemHandle(comm->peers[r]);
        cudaFree(comm->win);
    }
    gcm_status_t st = check_nccl(ncclCommDestroy(comm->nc));
    delete comm;
    return st;
}

gcm_status_t gcm_comm_set_peer(gcm_comm_t comm, int on) {
    if (!comm) return GCM_EINVAL;
    comm->peer = on ? 1 : 0;
    return GCM_OK;
}

// (Re)allocate this rank's IPC window for (n, nb) and map every rank's (collective: all ranks
// call it with the same sizes, in the same order).
static gcm_status_t peer_window(gcm_comm_t c, int64_t n, int64_t nb, cudaStream_t stream) {
    const int64_t NB64 = (n + kD - 1) / kD, NBc = (n + nb - 1) / nb;
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    const size_t sP = al((size_t)NBc * nb * kPassK * 8), sPan = al((size_t)NB64 * panel_doubles(32) * 8),
                 sU = al((size_t)NB64 * 32 * 32 * 8), sF = al((size_t)(NB64 + 1) * 4), sC = 256;
    const size_t need = sP + sPan + sU + sF + sC;
    if (c->win && c->win_bytes >= need) return GCM_OK;
    gcm_status_t st = check_cuda(cudaStreamSynchronize(stream));
    if (st != GCM_OK) return st;
    if (c->win) {
        for (int r = 0; r < c->nranks; ++r)
            if (r != c->rank && c->peers[r]) cudaIpcCloseMemHandle(c->peers[r]);
        cudaFree(c->win);
        c->win = nullptr;
        c->win_bytes = 0;
    }
    void *w = nullptr;
    st = check_cuda(cudaMalloc(&w, need));
    if (st != GCM_OK) return st;
    c->win = static_cast<char *>(w);
    c->win_bytes = need;
    c->epoch = 0;  // flags/counters of a fresh window start at zero on every rank
    st = check_cuda(cudaMemset(w, 0, need));
    if (st != GCM_OK) return st;
    c->offP = 0;
    c->offPan = sP;
    c->offU = sP + sPan;
    c->offFlag = sP + sPan + sU;
    c->offCtr = sP + sPan + sU + sF;
    c->peers[c->rank] = c->win;
    if (c->nranks == 1) return GCM_OK;
    cudaIpcMemHandle_t h;
    st = check_cuda(cudaIpcGetMemHandle(&h, w));
    if (st != GCM_OK) return st;
    const int R = c->nranks;
    char *dh = nullptr;
    st = check_cuda(cudaMalloc(&dh, (size_t)(R + 1) * sizeof(h)));
    if (st != GCM_OK) return st;
    std::vector<cudaIpcMemHandle_t> all(R);
    st = check_cuda(cudaMemcpy(dh, &h, sizeof(h), cudaMemcpyHostToDevice));
    if (st == GCM_OK)
        st = check_nccl(ncclAllGather(dh, dh + sizeof(h), sizeof(h), ncclChar, c->nc, stream));
    if (st == GCM_OK) st = check_cuda(cudaStreamSynchronize(stream));
    if (st == GCM_OK) st = check_cuda(cudaMemcpy(all.data(), dh + sizeof(h), R * sizeof(h), cudaMemcpyDeviceToHost));
    cudaFree(dh);
    for (int r = 0; r < R && st == GCM_OK; ++r) {
        if (r == c->rank) continue;
        void *pw = nullptr;
        st = check_cuda(cudaIpcOpenMemHandle(&pw, all[r], cudaIpcMemLazyEnablePeerAccess));
        c->peers[r] = static_cast<char *>(pw);
    }
    return st;
}

gcm_status_t gcm_modify_dist(gcm_comm_t comm, double *L_local, int64_t n, int64_t nb, int64_t ldl_local,
                             double *V_local, int64_t k, int sigma, gcm_info_t *d_info, gcm_stream_t stream_) {
    cudaStream_t stream = (cudaStream_t)stream_;
    if (!comm) return GCM_EINVAL;
    gcm_status_t st = dist_args(n, nb, k, sigma);
    if (st != GCM_OK) return st;
    if (ldl_local < std::max<int64_t>(1, n)) return GCM_EINVAL;
    const int R = comm->nranks, r = comm->rank;
    const int64_t nloc = local_cols(n, nb, R, r);
    if (n > 0 && k > 0 && nloc > 0 && (L_local == nullptr || V_local == nullptr)) return GCM_EINVAL;
    clear_stale_error();
    if (n == 0 || k == 0) return d_info ? check_cuda(cudaMemsetAsync(d_info, 0, sizeof(gcm_info_t), stream)) : GCM_OK;
    std::vector<Rank> rk(1);
    rk[0].L = L_local;
    rk[0].ldl = ldl_local;
    rk[0].V = V_local;
    if (!comm->peer) {
        Exchange x{Mode::Nccl, nullptr, comm->nc, r, nullptr, nullptr, nullptr, nullptr, nullptr};
        return panel_modify(rk, R, n, nb, k, sigma, d_info, x, stream);
    }
    // device-initiated exchange: the owner's dsolve and every rank's pbcast store straight into
    // the peers' windows (NVLink), with system-scope flags / counters instead of NCCL calls
    st = peer_window(comm, n, nb, stream);
    if (st != GCM_OK) return st;
    double *pP[kMaxRanks], *pPan[kMaxRanks], *pU[kMaxRanks];
    unsigned *pF[kMaxRanks], *pC[kMaxRanks];
    for (int q = 0; q < R; ++q) {
        pP[q] = reinterpret_cast<double *>(comm->peers[q] + comm->offP);
        pPan[q] = reinterpret_cast<double *>(comm->peers[q] + comm->offPan);
        pU[q] = reinterpret_cast<double *>(comm->peers[q] + comm->offU);
        pF[q] = reinterpret_cast<unsigned *>(comm->peers[q] + comm->offFlag);
        pC[q] = reinterpret_cast<unsigned *>(comm->peers[q] + comm->offCtr);
    }
    rk[0].Pw = pP[r];
    rk[0].panw = pPan[r];
    rk[0].Uw = pU[r];
    Exchange x{Mode::Peer, &comm->epoch, comm->nc, r, pP, pPan, pU, pF, pC};
    return panel_modify(rk, R, n, nb, k, sigma, d_info, x, stream);
}

#else  // built without NCCL

gcm_status_t gcm_comm_unique_id(void *) { return GCM_ENOTSUP; }
gcm_status_t gcm_comm_init(gcm_comm_t *, const void *, int, int) { return GCM_ENOTSUP; }
gcm_status_t gcm_comm_destroy(gcm_comm_t) { return GCM_ENOTSUP; }
gcm_status_t gcm_comm_set_peer(gcm_comm_t, int) { return GCM_ENOTSUP; }
gcm_status_t gcm_modify_dist(gcm_comm_t, double *, int64_t, int64_t, int64_t, double *, int64_t, int, gcm_info_t *,
                             gcm_stream_t) {
    return GCM_ENOTSUP;
}

#endif

}  // extern "C"

#ifdef GCM_PC_TRACE
extern "C" int gcm_debug_pc_trace(long long *host, int count) {
    return (int)cudaMemcpyFromSymbol(host, gcm::g_pc_trace, sizeof(long long) * count);
}
#endif
#ifdef GCM_TRACE
// this translation unit's copy of the diagonal-block phase marks (pdiag_kernel): tools/pdiag_phases.py
extern "C" int gcm_debug_dtrace_panel(long long *host, int count) {
    return (int)cudaMemcpyFromSymbol(host, gcm::g_dtrace, sizeof(long long) * count);
}
#endif
