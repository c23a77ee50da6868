// FP64 tensor-core (DMMA, mma.sync .f64) throughput vs DFMA on this GPU: decides whether the
// panel path's residual GEMM (pupdate) should move to mma.sync.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_peak dmma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int SHAPE>
__global__ void dmma_tput(double *out, int iters) {
    // SHAPE 0: m8n8k4 (256 FMA / warp-instr), 1: m16n8k4 (512), 2: m16n8k8 (1024), 3: m16n8k16 (2048)
    double a[8], b[4], c0[4] = {0, 0, 0, 0}, c1[4] = {0, 0, 0, 0}, c2[4] = {0, 0, 0, 0}, c3[4] = {0, 0, 0, 0};
    for (int i = 0; i < 8; ++i) a[i] = 1e-3 * (threadIdx.x + i);
    for (int i = 0; i < 4; ++i) b[i] = 1e-3 * (threadIdx.x - i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if constexpr (SHAPE == 0) {
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(c0[0]), "+d"(c0[1]) : "d"(a[0]), "d"(b[0]));
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(c1[0]), "+d"(c1[1]) : "d"(a[1]), "d"(b[1]));
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(c2[0]), "+d"(c2[1]) : "d"(a[2]), "d"(b[2]));
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(c3[0]), "+d"(c3[1]) : "d"(a[3]), "d"(b[3]));
            } else if constexpr (SHAPE == 1) {
                asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                             : "+d"(c0[0]), "+d"(c0[1]), "+d"(c0[2]), "+d"(c0[3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
                asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                             : "+d"(c1[0]), "+d"(c1[1]), "+d"(c1[2]), "+d"(c1[3]) : "d"(a[2]), "d"(a[3]), "d"(b[1]));
                asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                             : "+d"(c2[0]), "+d"(c2[1]), "+d"(c2[2]), "+d"(c2[3]) : "d"(a[4]), "d"(a[5]), "d"(b[2]));
                asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                             : "+d"(c3[0]), "+d"(c3[1]), "+d"(c3[2]), "+d"(c3[3]) : "d"(a[6]), "d"(a[7]), "d"(b[3]));
            } else if constexpr (SHAPE == 2) {
                asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+d"(c0[0]), "+d"(c0[1]), "+d"(c0[2]), "+d"(c0[3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
                asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+d"(c1[0]), "+d"(c1[1]), "+d"(c1[2]), "+d"(c1[3]) : "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[2]), "d"(b[3]));
            } else {
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                             : "+d"(c0[0]), "+d"(c0[1]), "+d"(c0[2]), "+d"(c0[3])
                             : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                               "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                             : "+d"(c1[0]), "+d"(c1[1]), "+d"(c1[2]), "+d"(c1[3])
                             : "d"(a[7]), "d"(a[6]), "d"(a[5]), "d"(a[4]), "d"(a[3]), "d"(a[2]), "d"(a[1]), "d"(a[0]),
                               "d"(b[3]), "d"(b[2]), "d"(b[1]), "d"(b[0]));
            }
        }
    }
    double s = 0;
    for (int i = 0; i < 4; ++i) s += c0[i] + c1[i] + c2[i] + c3[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// NCH independent accumulator chains per warp, fragments from shared memory (the pchain tile pattern)
template <int NCH>
__global__ void dmma_chains(double *out, int iters) {
    __shared__ double sa[64 * 68], sb[64 * 20];
    for (int i = threadIdx.x; i < 64 * 68; i += blockDim.x) sa[i] = 1e-3 * i;
    for (int i = threadIdx.x; i < 64 * 20; i += blockDim.x) sb[i] = 1e-3 * i;
    __syncthreads();
    const int lane = threadIdx.x & 31, gi = lane >> 2, tg = lane & 3, w = threadIdx.x >> 5;
    double c[NCH][2] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll 4
        for (int m0 = 0; m0 < 64; m0 += 4) {
            const double a = sa[((w & 7) * 8 + gi) * 68 + m0 + tg];
#pragma unroll
            for (int q = 0; q < NCH; ++q) {
                const double b = sb[(m0 + tg) * 20 + q * 8 + gi];
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(c[q][0]), "+d"(c[q][1]) : "d"(a), "d"(b));
            }
        }
    }
    double s = 0;
    for (int q = 0; q < NCH; ++q) s += c[q][0] + c[q][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int NCH>
void run_chains(int warps) {
    double *out;
    cudaMalloc(&out, 148 * 1024 * 8);
    dmma_chains<NCH><<<148, warps * 32>>>(out, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 2048;
    cudaEventRecord(e0);
    dmma_chains<NCH><<<148, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fmas = 148.0 * warps * iters * 16 * NCH * 256;
    std::printf("{\"chains_per_warp\": %d, \"warps_per_cta\": %d, \"ctas\": 148, \"tflops\": %.2f}\n", NCH, warps,
                2 * fmas / (ms * 1e-3) / 1e12);
    cudaFree(out);
}

// dependent-chain latency of one DMMA.8x8x4 (one warp)
__global__ void dmma_lat(double *out, long long *cyc, int iters) {
    double a = 1e-3 * threadIdx.x, b = 1e-3, c[2] = {0, 0};
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
    }
    long long t1 = clock64();
    out[threadIdx.x] = c[0] + c[1];
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int SHAPE>
void run(const char *name, double fma_per_instr, int instr_per_iter) {
    double *out;
    cudaMalloc(&out, 148 * 8 * 1024 * 8);
    const int iters = 4096;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int warps : {4, 8, 16}) {
        dmma_tput<SHAPE><<<sms * 2, warps * 32>>>(out, 16);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        dmma_tput<SHAPE><<<sms * 2, warps * 32>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double fmas = (double)sms * 2 * warps * iters * instr_per_iter * fma_per_instr;
        std::printf("{\"shape\": \"%s\", \"warps_per_cta\": %d, \"ctas\": %d, \"tflops\": %.2f, \"err\": \"%s\"}\n", name,
                    warps, sms * 2, 2 * fmas / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
    cudaFree(out);
}

int main() {
    run<0>("m8n8k4", 256, 16);
    run<1>("m16n8k4", 512, 16);
    run<2>("m16n8k8", 1024, 8);
    run<3>("m16n8k16", 2048, 8);
    {
        double *out;
        long long *cyc, h = 0;
        cudaMalloc(&out, 32 * 8);
        cudaMalloc(&cyc, 8);
        dmma_lat<<<1, 32>>>(out, cyc, 64);
        dmma_lat<<<1, 32>>>(out, cyc, 1024);
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        std::printf("{\"dmma_884_dependent_latency_cycles\": %.2f}\n", (double)h / (1024.0 * 16));
    }
    run_chains<1>(16);
    run_chains<2>(16);
    run_chains<2>(8);
    run_chains<4>(8);
    return 0;
}
