// DFMA issue rate on one SM vs warps per SM (8 independent chains per thread).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dfma_warps tools/dfma_warps.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(double *out, long long *cyc, int iters, double a, double b) {
    double x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = threadIdx.x + c;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
    double *out; long long *cyc; cudaMalloc(&out, 8 * 1024); cudaMalloc(&cyc, 8);
    const int iters = 4096;
    for (int w : {4, 8, 16, 32}) {
        long long h;
        k<8><<<1, w * 32>>>(out, cyc, iters, 1.0000001, 1e-9); cudaDeviceSynchronize();
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        const double instr_per_smsp = (double)w / 4 * iters * 8;
        printf("8 chains, %2d warps/SM: %.2f cycles per warp-DFMA per SMSP, %.1f DFMA lanes/clk/SM\n", w, h / instr_per_smsp,
               32.0 * w * iters * 8 / h);
        k<2><<<1, w * 32>>>(out, cyc, iters, 1.0000001, 1e-9); cudaDeviceSynchronize();
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("2 chains, %2d warps/SM: %.2f cycles per warp-DFMA per SMSP, %.1f DFMA lanes/clk/SM\n", w,
               h / ((double)w / 4 * iters * 2), 32.0 * w * iters * 2 / h);
    }
    return 0;
}
