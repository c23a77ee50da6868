// Shared-memory load throughput on one SM: uniform-address (broadcast) vs
// per-lane-distinct addresses, 64- and 128-bit.  Cycles per warp-instruction
// with 16 warps issuing independent loads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lds_bench tools/lds_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void lds(double *out, long long *cyc, int iters) {
    __shared__ __align__(16) double sm[4096];
    const int t = threadIdx.x, lane = t & 31;
    for (int i = t; i < 4096; i += blockDim.x) sm[i] = i * 1e-3;
    __syncthreads();
    double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const int base = (it * 64) & 2047;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (MODE == 0) {  // LDS.64 uniform address
                acc0 += sm[base + u * 8];
            } else if (MODE == 1) {  // LDS.64 distinct (32 consecutive doubles)
                acc0 += sm[base + u * 32 + lane];
            } else if (MODE == 2) {  // LDS.128 uniform
                const double2 v = *reinterpret_cast<const double2 *>(sm + base + u * 8);
                acc0 += v.x;
                acc1 += v.y;
            } else if (MODE == 3) {  // LDS.128 distinct
                const double2 v = *reinterpret_cast<const double2 *>(sm + base + u * 64 + 2 * lane);
                acc0 += v.x;
                acc1 += v.y;
            } else if (MODE == 4) {  // LDS.64, 4 distinct addresses per warp (8 lanes each)
                acc0 += sm[base + u * 8 + (lane >> 3) * 33];
            } else if (MODE == 5) {  // LDS.128, 8 distinct 16-B addresses (4 lanes each)
                const double2 v = *reinterpret_cast<const double2 *>(sm + base + u * 16 + 2 * (lane & 7));
                acc0 += v.x;
                acc1 += v.y;
            }
        }
    }
    long long t1 = clock64();
    if (t == 0) cyc[0] = t1 - t0;
    out[t] = acc0 + acc1 + acc2 + acc3;
}

int main() {
    double *out;
    long long *cyc;
    cudaMalloc(&out, 1024 * 8);
    cudaMalloc(&cyc, 8);
    const int iters = 2000, warps = 16;
    const char *names[] = {"LDS.64 uniform", "LDS.64 distinct", "LDS.128 uniform", "LDS.128 distinct",
                           "LDS.64 4-distinct", "LDS.128 8-distinct"};
    for (int mode = 0; mode < 6; ++mode) {
        long long h = 0;
        switch (mode) {
            case 0: lds<0><<<1, warps * 32>>>(out, cyc, iters); break;
            case 1: lds<1><<<1, warps * 32>>>(out, cyc, iters); break;
            case 2: lds<2><<<1, warps * 32>>>(out, cyc, iters); break;
            case 3: lds<3><<<1, warps * 32>>>(out, cyc, iters); break;
            case 4: lds<4><<<1, warps * 32>>>(out, cyc, iters); break;
            case 5: lds<5><<<1, warps * 32>>>(out, cyc, iters); break;
        }
        cudaDeviceSynchronize();
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("%-20s %.2f cycles per warp-load (SM-wide)\n", names[mode], (double)h / (iters * 8.0 * warps));
    }
    return 0;
}
