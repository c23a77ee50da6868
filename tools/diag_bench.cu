// Latency of the closed-form diagonal-block pieces (diag.cuh) on an otherwise idle SM:
// one CTA of 256 threads, KB = 8, a 64 x 64 well-conditioned block; clock64 per piece.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o /tmp/diag_bench tools/diag_bench.cu
#include <cstdio>
#include <vector>
#include "../paper_1011_1173_b200/csrc/diag.cuh"

using namespace gcm;
constexpr int KB = 8;

__global__ void __launch_bounds__(256, 2) bench(const double *Lg, const double *Yg, long long *cyc, double *out,
                                                 unsigned long long *key) {
    extern __shared__ double sm[];
    double(*Ls)[kD + 1] = reinterpret_cast<double(*)[kD + 1]>(sm);
    double *qv = sm + kD * (kD + 1);
    double *scr = qv + kD * (KB + 1);
    double *pan = scr + diag_closed_scratch(KB);
    double *rinv = pan + 2 * kD * KB + kD + KB;
    const int t = threadIdx.x;
    long long c0 = 0, c1 = 0, c2 = 0;
    for (int rep = 0; rep < 4; ++rep) {
        for (int i = t; i < kD * kD; i += blockDim.x) Ls[i / kD][i % kD] = Lg[i];
        for (int i = t; i < kD * KB; i += blockDim.x) qv[(i / KB) * (KB + 1) + i % KB] = Yg[i];
        __syncthreads();
        long long a = clock64();
        block_trsv<KB>(Ls, qv, KB + 1, kD, rinv);
        long long b = clock64();
        diag_closed<KB>(Ls, qv, KB + 1, kD, KB, 1, 0, pan, out, kD, key, 0, scr);
        long long c = clock64();
        if (rep == 3) { c0 = b - a; c1 = c - b; }
    }
    if (t == 0) { cyc[0] = c0; cyc[1] = c1; cyc[2] = c2; }
}

int main() {
    std::vector<double> L(kD * kD), Y(kD * KB);
    for (int m = 0; m < kD; ++m)
        for (int j = 0; j < kD; ++j) L[m * kD + j] = j == m ? 2.0 + 0.01 * m : (j < m ? 0.01 * ((m * 7 + j * 3) % 11) : 0.0);
    for (int i = 0; i < kD * KB; ++i) Y[i] = 0.001 * (i % 13);
    double *dL, *dY, *out; long long *cyc; unsigned long long *key;
    cudaMalloc(&dL, 8 * kD * kD); cudaMalloc(&dY, 8 * kD * KB); cudaMalloc(&out, 8 * kD * KB); cudaMalloc(&cyc, 64); cudaMalloc(&key, 8);
    cudaMemcpy(dL, L.data(), 8 * kD * kD, cudaMemcpyHostToDevice);
    cudaMemcpy(dY, Y.data(), 8 * kD * KB, cudaMemcpyHostToDevice);
    const int smem = 8 * (kD * (kD + 1) + kD * (KB + 1) + diag_closed_scratch(KB) + 2 * kD * KB + kD + KB + kD);
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    bench<<<1, 256, smem>>>(dL, dY, cyc, out, key);
    long long h[3];
    cudaMemcpy(h, cyc, 24, cudaMemcpyDeviceToHost);
    printf("idle SM, KB=8: block_trsv %lld cycles, diag_closed %lld cycles (%s)\n", h[0], h[1], cudaGetErrorString(cudaGetLastError()));
    return 0;
}
