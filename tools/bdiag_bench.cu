// Latency of one diagonal-block sweep (bparts.cuh bdiag_body, KB = 16, 288 threads) on an
// otherwise idle SM, closed form vs wave; phases by globaltimer with -DGCM_TRACE.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -DGCM_TRACE -o tools/bdiag_bench tools/bdiag_bench.cu
#include <cstdio>
#include <vector>
#include "../paper_1011_1173_b200/csrc/bparts.cuh"

using namespace gcm;
constexpr int KB = 16;

__global__ void __launch_bounds__(kDiagThreads, 1) bench(double *L, int64_t n, double *V, const double *P, double *Ui,
                                                        const double *G, double *panels, unsigned long long *key,
                                                        long long *cyc) {
    extern __shared__ double smem_b[];
    long long t0 = clock64();
    bdiag_body<KB>(L, n, n, V, n, KB, 1, P, false, Ui, G, panels, key, 0, 1, smem_b);
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
    const int n = 128, k = KB;
    std::vector<double> L(n * n, 0.0), V(n * k), P(n * k), G(2 * KB * KB, 0.0);
    for (int c = 0; c < n; ++c)
        for (int r = 0; r <= c; ++r) L[r + c * n] = r == c ? 2.0 : 0.01 * ((r * 7 + c * 3) % 11);
    for (int i = 0; i < n * k; ++i) { V[i] = 0.01 * (i % 13); P[i] = 0.001 * (i % 7); }
    double *dL, *dV, *dP, *dU, *dG, *dpan; long long *cyc; unsigned long long *key;
    cudaMalloc(&dL, 8 * n * n); cudaMalloc(&dV, 8 * n * k); cudaMalloc(&dP, 8 * n * k); cudaMalloc(&dU, 8 * 2 * KB * KB);
    cudaMalloc(&dG, 8 * 2 * KB * KB); cudaMalloc(&dpan, 8 * 2 * panel_doubles(KB)); cudaMalloc(&cyc, 64); cudaMalloc(&key, 8);
    cudaMemcpy(dL, L.data(), 8 * n * n, cudaMemcpyHostToDevice);
    cudaMemcpy(dV, V.data(), 8 * n * k, cudaMemcpyHostToDevice);
    cudaMemcpy(dP, P.data(), 8 * n * k, cudaMemcpyHostToDevice);
    cudaMemcpy(dG, G.data(), 8 * 2 * KB * KB, cudaMemcpyHostToDevice);
    const int smem = bdiag_smem_doubles(KB) * 8;
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int rep = 0; rep < 3; ++rep) bench<<<1, kDiagThreads, smem>>>(dL, n, dV, dP, dU, dG, dpan, key, cyc);
    long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    long long tr[256 * 8]; cudaMemcpyFromSymbol(tr, g_dtrace, sizeof(tr));
#ifdef GCM_BT_TRACE
    long long dc[16 * 8]; cudaMemcpyFromSymbol(dc, g_dc_trace, sizeof(dc));
    printf("diag_closed sub-steps (cycles): A+prefix %lld, B %lld, C %lld, mu %lld, D %lld\n", dc[9] - dc[8], dc[10] - dc[9],
           dc[11] - dc[10], dc[12] - dc[11], dc[13] - dc[12]);
#endif
    printf("bdiag_body<16> idle SM: %lld cycles; phases (ns): loads %lld, w+U %lld, V,q %lld, closed %lld, tri %lld (%s)\n", h,
           tr[9] - tr[8], tr[10] - tr[9], tr[11] - tr[10], tr[12] - tr[11], tr[13] - tr[12], cudaGetErrorString(cudaGetLastError()));
    return 0;
}
