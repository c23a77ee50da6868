// Microbenchmark of the TRSV helper's tile contraction (32 x 32 L tile times a
// 32 x 16 P block, register-blocked 2 x 2 per thread, 128 threads) in isolation:
// cycles per tile on one SM.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tile_bench tools/tile_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kDT = 32, kLdT = 33, KB = 16;

template <int SPLIT>
__global__ void tile(double *out, long long *cyc, int reps, int k) {
    __shared__ double Lt[kDT * kLdT];
    __shared__ __align__(16) double Pt[kDT * KB];
    __shared__ double r[kDT * KB];
    const int t = threadIdx.x;
    for (int i = t; i < kDT * kLdT; i += blockDim.x) Lt[i] = 1.0 + i * 1e-3;
    for (int i = t; i < kDT * KB; i += blockDim.x) Pt[i] = 2.0 - i * 1e-3;
    for (int i = t; i < kDT * KB; i += blockDim.x) r[i] = 0.0;
    __syncthreads();
    constexpr int EG = KB / 2;
    long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
        if (t < 16 * EG) {
            const int cq = t / EG, eg = t % EG;
            const int ca = 2 * cq, e = 2 * eg;
            double acc[SPLIT][4];
#pragma unroll
            for (int q = 0; q < SPLIT; ++q)
#pragma unroll
                for (int o = 0; o < 4; ++o) acc[q][o] = 0.0;
            const double *La = Lt + ca * kLdT, *Lb2 = La + kLdT;
#pragma unroll
            for (int m = 0; m < kDT; ++m) {
                const double2 pv = *reinterpret_cast<const double2 *>(Pt + m * k + e);
                const double la = La[m], lb = Lb2[m];
                acc[m % SPLIT][0] = fma(la, pv.x, acc[m % SPLIT][0]);
                acc[m % SPLIT][1] = fma(la, pv.y, acc[m % SPLIT][1]);
                acc[m % SPLIT][2] = fma(lb, pv.x, acc[m % SPLIT][2]);
                acc[m % SPLIT][3] = fma(lb, pv.y, acc[m % SPLIT][3]);
            }
            double s[4] = {0, 0, 0, 0};
#pragma unroll
            for (int q = 0; q < SPLIT; ++q)
#pragma unroll
                for (int o = 0; o < 4; ++o) s[o] += acc[q][o];
            r[ca * KB + e] -= s[0];
            r[ca * KB + e + 1] -= s[1];
            r[(ca + 1) * KB + e] -= s[2];
            r[(ca + 1) * KB + e + 1] -= s[3];
        }
        __syncthreads();
    }
    long long t1 = clock64();
    if (t == 0) cyc[blockIdx.x] = t1 - t0;
    if (t < kDT * KB) out[blockIdx.x * kDT * KB + t] = r[t];
}


// G groups of 128 threads each take kDT/G rows m; partial 2x2 blocks reduced through smem
template <int G>
__global__ void tile_msplit(double *out, long long *cyc, int reps, int k) {
    __shared__ double Lt[kDT * kLdT];
    __shared__ __align__(16) double Pt[kDT * KB];
    __shared__ double r[kDT * KB];
    __shared__ double part[G][kDT * KB];
    const int t = threadIdx.x;
    for (int i = t; i < kDT * kLdT; i += blockDim.x) Lt[i] = 1.0 + i * 1e-3;
    for (int i = t; i < kDT * KB; i += blockDim.x) Pt[i] = 2.0 - i * 1e-3;
    for (int i = t; i < kDT * KB; i += blockDim.x) r[i] = 0.0;
    __syncthreads();
    constexpr int EG = KB / 2;
    long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
        const int g = t / (16 * EG), tt = t % (16 * EG);
        if (g < G) {
            const int cq = tt / EG, eg = tt % EG;
            const int ca = 2 * cq, e = 2 * eg;
            double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
            const double *La = Lt + ca * kLdT, *Lb2 = La + kLdT;
#pragma unroll
            for (int mm = 0; mm < kDT / G; ++mm) {
                const int m = g * (kDT / G) + mm;
                const double2 pv = *reinterpret_cast<const double2 *>(Pt + m * k + e);
                const double la = La[m], lb = Lb2[m];
                a0 = fma(la, pv.x, a0);
                a1 = fma(la, pv.y, a1);
                a2 = fma(lb, pv.x, a2);
                a3 = fma(lb, pv.y, a3);
            }
            part[g][ca * KB + e] = a0;
            part[g][ca * KB + e + 1] = a1;
            part[g][(ca + 1) * KB + e] = a2;
            part[g][(ca + 1) * KB + e + 1] = a3;
        }
        __syncthreads();
        for (int i = t; i < kDT * KB; i += blockDim.x) {
            double s = 0;
#pragma unroll
            for (int q = 0; q < G; ++q) s += part[q][i];
            r[i] -= s;
        }
        __syncthreads();
    }
    long long t1 = clock64();
    if (t == 0) cyc[blockIdx.x] = t1 - t0;
    if (t < kDT * KB) out[blockIdx.x * kDT * KB + t] = r[t];
}

// FP64 tensor cores: mma.sync m8n8k4; warp w owns output tiles (8 cols x 8 e), 8 tiles total,
// each tile's 8 k-steps split over 2 independent accumulator pairs
__global__ void tile_dmma(double *out, long long *cyc, int reps, int k) {
    __shared__ double Lt[kDT * kLdT];
    __shared__ double Pt[kDT * (KB + 1)];
    __shared__ double r[kDT * KB];
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    for (int i = t; i < kDT * kLdT; i += blockDim.x) Lt[i] = 1.0 + i * 1e-3;
    for (int i = t; i < kDT * (KB + 1); i += blockDim.x) Pt[i] = 2.0 - i * 1e-3;
    for (int i = t; i < kDT * KB; i += blockDim.x) r[i] = 0.0;
    __syncthreads();
    const int nw = blockDim.x / 32;
    long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
        const int g = lane >> 2, t4 = lane & 3;
        for (int tile = warp; tile < 8; tile += nw) {
            const int ct = tile / 2, et = tile % 2;
            double c0 = 0, c1 = 0, d0 = 0, d1 = 0;
            const double *Arow = Lt + (ct * 8 + g) * kLdT + t4;
            const int eb = et * 8 + g;
#pragma unroll
            for (int k0 = 0; k0 < kDT; k0 += 8) {
                const double av = Arow[k0], bv = Pt[(k0 + t4) * (KB + 1) + eb];
                const double av2 = Arow[k0 + 4], bv2 = Pt[(k0 + 4 + t4) * (KB + 1) + eb];
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                             : "+d"(c0), "+d"(c1) : "d"(av), "d"(bv));
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                             : "+d"(d0), "+d"(d1) : "d"(av2), "d"(bv2));
            }
            const int cc = ct * 8 + g, e = et * 8 + 2 * t4;
            r[cc * KB + e] -= c0 + d0;
            r[cc * KB + e + 1] -= c1 + d1;
        }
        __syncthreads();
    }
    long long t1 = clock64();
    if (t == 0) cyc[blockIdx.x] = t1 - t0;
    if (t < kDT * KB) out[blockIdx.x * kDT * KB + t] = r[t];
}


// DMMA with all 8 k-steps of a warp's output tile independent (8 accumulator pairs, summed at the end)
__global__ void tile_dmma_ind(double *out, long long *cyc, int reps, int k) {
    __shared__ double Lt[kDT * kLdT];
    __shared__ double Pt[kDT * (KB + 1)];
    __shared__ double r[kDT * KB];
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    for (int i = t; i < kDT * kLdT; i += blockDim.x) Lt[i] = 1.0 + i * 1e-3;
    for (int i = t; i < kDT * (KB + 1); i += blockDim.x) Pt[i] = 2.0 - i * 1e-3;
    for (int i = t; i < kDT * KB; i += blockDim.x) r[i] = 0.0;
    __syncthreads();
    const int nw = blockDim.x / 32;
    long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
        const int g = lane >> 2, t4 = lane & 3;
        for (int tile = warp; tile < 8; tile += nw) {
            const int ct = tile / 2, et = tile % 2;
            double c[8][2];
            const double *Arow = Lt + (ct * 8 + g) * kLdT + t4;
            const int eb = et * 8 + g;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                c[q][0] = 0; c[q][1] = 0;
                const double av = Arow[4 * q], bv = Pt[(4 * q + t4) * (KB + 1) + eb];
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                             : "+d"(c[q][0]), "+d"(c[q][1]) : "d"(av), "d"(bv));
            }
            double s0 = 0, s1 = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) { s0 += c[q][0]; s1 += c[q][1]; }
            const int cc = ct * 8 + g, e = et * 8 + 2 * t4;
            r[cc * KB + e] -= s0;
            r[cc * KB + e + 1] -= s1;
        }
        __syncthreads();
    }
    long long t1 = clock64();
    if (t == 0) cyc[blockIdx.x] = t1 - t0;
    if (t < kDT * KB) out[blockIdx.x * kDT * KB + t] = r[t];
}

// empty loop: cost of the rep loop + __syncthreads alone
__global__ void tile_empty(double *out, long long *cyc, int reps, int k) {
    __shared__ double r[kDT * KB];
    const int t = threadIdx.x;
    for (int i = t; i < kDT * KB; i += blockDim.x) r[i] = 0.0;
    __syncthreads();
    long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
        if (t < kDT * KB) r[t] -= 1.0;
        __syncthreads();
    }
    long long t1 = clock64();
    if (t == 0) cyc[blockIdx.x] = t1 - t0;
    if (t < kDT * KB) out[blockIdx.x * kDT * KB + t] = r[t];
}


// the helper's new contraction (lane = column pair x m-half, warp = e-set); POLL != 0 adds a warp
// spinning on ld.acquire.gpu + nanosleep(20) like the feeder (POLL 2: ld.relaxed)
template <int POLL>
__global__ void tile_new(double *out, long long *cyc, int reps, int k, unsigned long long *flag) {
    constexpr int kLdTT = 34, EW = KB / 4;
    __shared__ __align__(16) double Lt[kDT * kLdTT];
    __shared__ __align__(16) double Pt[kDT * KB];
    __shared__ double r[kDT * KB];
    __shared__ volatile int stop;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    for (int i = t; i < kDT * kLdTT; i += blockDim.x) Lt[i] = 1.0 + i * 1e-3;
    for (int i = t; i < kDT * KB; i += blockDim.x) Pt[i] = 2.0 - i * 1e-3;
    for (int i = t; i < kDT * KB; i += blockDim.x) r[i] = 0.0;
    if (t == 0) stop = 0;
    __syncthreads();
    if (warp == 4) {
        if (POLL) {
            unsigned long long v = 0;
            while (!stop) {
                if (POLL == 1) asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(flag + lane) : "memory");
                else asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(flag + lane) : "memory");
                __nanosleep(20);
            }
            if (v == 12345) out[0] = 1;
        }
        return;
    }
    long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
        const int q = lane & 15, hm = lane >> 4;
        const int eb = warp * EW;
        double acc0[EW], acc1[EW];
#pragma unroll
        for (int j = 0; j < EW; ++j) acc0[j] = acc1[j] = 0.0;
        const double *Lrow = Lt + (hm * 16) * kLdTT + 2 * q;
        const double *Prow = Pt + (hm * 16) * k + eb;
#pragma unroll
        for (int mm = 0; mm < 16; ++mm) {
            const double2 l = *reinterpret_cast<const double2 *>(Lrow + mm * kLdTT);
#pragma unroll
            for (int j = 0; j < EW; ++j) {
                const double pv = eb + j < k ? Prow[mm * k + j] : 0.0;
                acc0[j] = fma(l.x, pv, acc0[j]);
                acc1[j] = fma(l.y, pv, acc1[j]);
            }
        }
#pragma unroll
        for (int j = 0; j < EW; ++j) {
            acc0[j] += __shfl_xor_sync(0xffffffffu, acc0[j], 16);
            acc1[j] += __shfl_xor_sync(0xffffffffu, acc1[j], 16);
        }
        if (hm == 0) {
#pragma unroll
            for (int j = 0; j < EW; ++j) {
                r[(2 * q) * KB + eb + j] -= acc0[j];
                r[(2 * q + 1) * KB + eb + j] -= acc1[j];
            }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
    }
    long long t1 = clock64();
    if (t == 0) { cyc[blockIdx.x] = t1 - t0; stop = 1; }
    if (t < kDT * KB) out[blockIdx.x * kDT * KB + t] = r[t];
}


// v3: 4 warps = 4 m-quarters; lane (cb = lane & 7, eb = lane >> 3) owns a 4 x 4 output block
// (columns 4cb.., update columns 4eb..); L tile transposed [m][34]; quarters reduced through smem
template <bool RED>
__global__ void tile_v3(double *out, long long *cyc, int reps, int k) {
    constexpr int kLdTT = 34;
    __shared__ __align__(16) double Lt[kDT * kLdTT];
    __shared__ __align__(16) double Pt[kDT * KB];
    __shared__ __align__(16) double part[4][kDT * KB];
    __shared__ double r[kDT * KB];
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    for (int i = t; i < kDT * kLdTT; i += blockDim.x) Lt[i] = 1.0 + i * 1e-3;
    for (int i = t; i < kDT * KB; i += blockDim.x) Pt[i] = 2.0 - i * 1e-3;
    for (int i = t; i < kDT * KB; i += blockDim.x) r[i] = 0.0;
    __syncthreads();
    long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
        const int cb = lane & 7, eb = lane >> 3;
        double acc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
#pragma unroll
        for (int mm = 0; mm < 8; ++mm) {
            const int m = warp * 8 + mm;
            double lv[4], pv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) lv[i] = Lt[m * kLdTT + 4 * cb + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) pv[j] = Pt[m * k + 4 * eb + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(lv[i], pv[j], acc[i][j]);
        }
        if (RED) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                double *pp = &part[warp][(4 * cb + i) * KB + 4 * eb];
                reinterpret_cast<double2 *>(pp)[0] = make_double2(acc[i][0], acc[i][1]);
                reinterpret_cast<double2 *>(pp)[1] = make_double2(acc[i][2], acc[i][3]);
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
            for (int o = t; o < kDT * KB; o += 128)
                r[o] -= (part[0][o] + part[1][o]) + (part[2][o] + part[3][o]);
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) r[(4 * cb + i) * KB + 4 * eb + j] -= acc[i][j];
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
    }
    long long t1 = clock64();
    if (t == 0) cyc[blockIdx.x] = t1 - t0;
    if (t < kDT * KB) out[blockIdx.x * kDT * KB + t] = r[t];
}


// v4: NW warps = m-slices of 32/NW rows; all operand loads of the slice issued before the FMAs
template <int NW>
__global__ void tile_v4(double *out, long long *cyc, int reps, int k) {
    constexpr int kLdTT = 36, MS = kDT / NW;
    __shared__ __align__(16) double Lt[kDT * kLdTT];
    __shared__ __align__(16) double Pt[kDT * KB];
    __shared__ __align__(16) double part[NW > 4 ? 4 : NW][kDT * KB];
    __shared__ double r[kDT * KB];
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    for (int i = t; i < kDT * kLdTT; i += blockDim.x) Lt[i] = 1.0 + i * 1e-3;
    for (int i = t; i < kDT * KB; i += blockDim.x) Pt[i] = 2.0 - i * 1e-3;
    for (int i = t; i < kDT * KB; i += blockDim.x) r[i] = 0.0;
    __syncthreads();
    long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
        const int cb = lane & 7, eb = lane >> 3;
        double lv[MS][4], pv[MS][4];
#pragma unroll
        for (int mm = 0; mm < MS; ++mm) {
            const int m = warp * MS + mm;
            const double2 l01 = *reinterpret_cast<const double2 *>(&Lt[m * kLdTT + 4 * cb]);
            const double2 l23 = *reinterpret_cast<const double2 *>(&Lt[m * kLdTT + 4 * cb + 2]);
            const double2 p01 = *reinterpret_cast<const double2 *>(&Pt[m * KB + 4 * eb]);
            const double2 p23 = *reinterpret_cast<const double2 *>(&Pt[m * KB + 4 * eb + 2]);
            lv[mm][0] = l01.x; lv[mm][1] = l01.y; lv[mm][2] = l23.x; lv[mm][3] = l23.y;
            pv[mm][0] = p01.x; pv[mm][1] = p01.y; pv[mm][2] = p23.x; pv[mm][3] = p23.y;
        }
        double acc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
#pragma unroll
        for (int mm = 0; mm < MS; ++mm)
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(lv[mm][i], pv[mm][j], acc[i][j]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            double *pp = &part[warp & 3][(4 * cb + i) * KB + 4 * eb];
            if (warp < 4) {
                reinterpret_cast<double2 *>(pp)[0] = make_double2(acc[i][0], acc[i][1]);
                reinterpret_cast<double2 *>(pp)[1] = make_double2(acc[i][2], acc[i][3]);
            }
        }
        __syncthreads();
        if (NW > 4) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                double *pp = &part[warp & 3][(4 * cb + i) * KB + 4 * eb];
                if (warp >= 4) {
                    pp[0] += acc[i][0]; pp[1] += acc[i][1]; pp[2] += acc[i][2]; pp[3] += acc[i][3];
                }
            }
            __syncthreads();
        }
        for (int o = t; o < kDT * KB; o += NW * 32) {
            double sum = 0.0;
#pragma unroll
            for (int w = 0; w < (NW > 4 ? 4 : NW); ++w) sum += part[w][o];
            r[o] -= sum;
        }
        __syncthreads();
    }
    long long t1 = clock64();
    if (t == 0) cyc[blockIdx.x] = t1 - t0;
    if (t < kDT * KB) out[blockIdx.x * kDT * KB + t] = r[t];
}

int main2() {
    double *out;
    long long *cyc;
    cudaMalloc(&out, 148 * kDT * KB * 8);
    cudaMalloc(&cyc, 148 * 8);
    const int reps = 1000;
    long long h = 0;
    tile_msplit<2><<<1, 256>>>(out, cyc, reps, KB); cudaDeviceSynchronize(); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("msplit2 256 thr: %.0f cycles per tile\n", (double)h / reps);
    tile_msplit<4><<<1, 512>>>(out, cyc, reps, KB); cudaDeviceSynchronize(); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("msplit4 512 thr: %.0f cycles per tile\n", (double)h / reps);
    tile_msplit<2><<<1, 256>>>(out, cyc, reps, KB); cudaDeviceSynchronize(); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("msplit2 again 256 thr: %.0f cycles per tile\n", (double)h / reps);
    for (int th : {256, 128, 64}) {
        tile_dmma<<<1, th>>>(out, cyc, reps, KB); cudaDeviceSynchronize(); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("dmma %d thr: %.0f cycles per tile\n", th, (double)h / reps);
    }
    for (int th : {256, 128}) {
        tile_dmma_ind<<<1, th>>>(out, cyc, reps, KB); cudaDeviceSynchronize(); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("dmma independent %d thr: %.0f cycles per tile\n", th, (double)h / reps);
    }
    unsigned long long *flag;
    cudaMalloc(&flag, 4096);
    cudaMemset(flag, 0, 4096);
    tile_new<0><<<1, 160>>>(out, cyc, reps, KB, flag); cudaDeviceSynchronize(); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("new contraction, no poller: %.0f cycles per tile\n", (double)h / reps);
    tile_new<1><<<1, 160>>>(out, cyc, reps, KB, flag); cudaDeviceSynchronize(); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("new contraction, acquire poller: %.0f cycles per tile\n", (double)h / reps);
    tile_new<2><<<1, 160>>>(out, cyc, reps, KB, flag); cudaDeviceSynchronize(); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("new contraction, relaxed poller: %.0f cycles per tile\n", (double)h / reps);
    tile_v3<true><<<1, 128>>>(out, cyc, reps, KB); cudaDeviceSynchronize(); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("v3 4x4 blocks, m-quarters + smem reduction: %.0f cycles per tile\n", (double)h / reps);
    tile_v3<false><<<1, 128>>>(out, cyc, reps, KB); cudaDeviceSynchronize(); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("v3 without reduction (timing only): %.0f cycles per tile\n", (double)h / reps);
    tile_v4<4><<<1, 128>>>(out, cyc, reps, KB); cudaDeviceSynchronize(); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("v4 4 warps (8 m each, loads first): %.0f cycles per tile\n", (double)h / reps);
    tile_v4<8><<<1, 256>>>(out, cyc, reps, KB); cudaDeviceSynchronize(); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("v4 8 warps (4 m each, loads first): %.0f cycles per tile\n", (double)h / reps);
    tile_empty<<<1, 256>>>(out, cyc, reps, KB); cudaDeviceSynchronize(); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("empty 256 thr: %.0f cycles per rep\n", (double)h / reps);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

int main() {
    main2();
    double *out;
    long long *cyc;
    cudaMalloc(&out, 148 * kDT * KB * 8);
    cudaMalloc(&cyc, 148 * 8);
    const int reps = 1000;
    for (int blocks : {1, 148}) {
        for (int threads : {128, 288}) {
            tile<4><<<blocks, threads>>>(out, cyc, reps, KB);
            long long h = 0;
            cudaDeviceSynchronize();
            cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
            printf("split4 blocks %3d threads %3d: %.0f cycles per tile (incl. __syncthreads)\n", blocks, threads,
                   (double)h / reps);
            tile<1><<<blocks, threads>>>(out, cyc, reps, KB);
            cudaDeviceSynchronize();
            cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
            printf("split1 blocks %3d threads %3d: %.0f cycles per tile (incl. __syncthreads)\n", blocks, threads,
                   (double)h / reps);
        }
    }
    return 0;
}
