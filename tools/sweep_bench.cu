// Microbenchmark of the diagonal-block chain: block_sweep vs wave_sweep on one
// 64 x 64 block per CTA (numbers only; parity is covered by the GPU tests).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../include -o sweep_bench sweep_bench.cu
#include <cstdio>
#include <vector>
#include "../paper_1011_1173_b200/csrc/rot.cuh"

using namespace gcm;

template <int KB, bool WAVE, int NQ>
__global__ void bench_kernel(const double *Lin, const double *Vin, int k, double *panels, double *vexit,
                             unsigned long long *key, long long *cyc) {
    extern __shared__ double sm[];
    double(*Ls)[kD + 1] = reinterpret_cast<double(*)[kD + 1]>(sm);
    double *pan = sm + kD * (kD + 1);
    double *vx = pan + wave_panel_doubles(KB) + 1;
    double *dinv = vx + kD * KB;
    double *vt = dinv + kD;
    double *imx = vt + kD * KB;
    double *Vs = imx + kD * KB;
    double *vrow = Vs + kD * KB;
    double *IM = vrow + KB;
    double2 *cs = reinterpret_cast<double2 *>(IM + KB + (((uintptr_t)(IM + KB) & 15) ? 1 : 0));
    double *rho_s = reinterpret_cast<double *>(cs + KB);
    const int t = threadIdx.x;
    for (int i = t; i < kD * kD; i += blockDim.x) {
        const int m = i / kD, j = i % kD;
        if (j <= m) Ls[m][j] = Lin[j + m * kD];
    }
    for (int i = t; i < kD * KB; i += blockDim.x) Vs[i] = (i % KB) < k ? Vin[i / KB + (i % KB) * kD] : 0.0;
    double v[KB];
    for (int e = 0; e < KB; ++e) v[e] = (t < kD && e < k) ? Vin[t + e * kD] : 0.0;
    __syncthreads();
    long long t0 = clock64();
    if (WAVE)
        wave_sweep<KB, NQ, kD + 1>(Ls, Vs, kD, k, 1, 0, pan, vexit + blockIdx.x * kD * k, kD, key, 0, vx, dinv, vt, imx,
                                   0, NQ * kD / 32);
    else
        block_sweep<KB, kD + 1>(Ls, v, kD, k, 1, 0, pan, vexit + blockIdx.x * kD * k, kD, key, 0, vrow, IM, cs, rho_s, 0);
    long long t1 = clock64();
    if (t == 0) cyc[blockIdx.x] = t1 - t0;
    for (int i = t; i < panel_doubles(k); i += blockDim.x) panels[blockIdx.x * panel_doubles(k) + i] = pan[i];
}

template <int KB, bool WAVE, int NQ = 1>
void run(int k, int ctas) {
    std::vector<double> L(kD * kD, 0.0), V(kD * k);
    for (int m = 0; m < kD; ++m)
        for (int j = 0; j <= m; ++j) L[j + m * kD] = (j == m) ? 3.0 + 0.01 * m : 0.01 * ((j * 7 + m * 3) % 11);
    for (int i = 0; i < kD * k; ++i) V[i] = 0.1 * ((i * 13) % 7);
    double *dL, *dV, *dP, *dX;
    unsigned long long *key;
    long long *cyc;
    cudaMalloc(&dL, L.size() * 8);
    cudaMalloc(&dV, V.size() * 8);
    cudaMalloc(&dP, (size_t)ctas * wave_panel_doubles(KB) * 8);
    cudaMalloc(&dX, (size_t)ctas * kD * k * 8);
    cudaMalloc(&key, 8);
    cudaMalloc(&cyc, ctas * 8);
    cudaMemcpy(dL, L.data(), L.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dV, V.data(), V.size() * 8, cudaMemcpyHostToDevice);
    const size_t smem = (kD * (kD + 1) + wave_panel_doubles(KB) + 1 + 4 * kD * KB + kD + 4 * KB + 8) * 8;
    cudaFuncSetAttribute(bench_kernel<KB, WAVE, NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int threads = WAVE ? NQ * kD + 32 : 64;
    for (int it = 0; it < 2; ++it) bench_kernel<KB, WAVE, NQ><<<ctas, threads, smem>>>(dL, dV, k, dP, dX, key, cyc);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    bench_kernel<KB, WAVE, NQ><<<ctas, threads, smem>>>(dL, dV, k, dP, dX, key, cyc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    std::vector<long long> c(ctas);
    cudaMemcpy(c.data(), cyc, ctas * 8, cudaMemcpyDeviceToHost);
    printf("%s NQ=%d k=%2d ctas=%4d: kernel %.1f us, sweep %lld cycles (%.0f per row)  err=%s\n", WAVE ? "wave " : "block",
           NQ, k, ctas, ms * 1e3, c[0], c[0] / 64.0, cudaGetErrorString(cudaGetLastError()));
}

void dump_trace() {
#ifdef GCM_SWEEP_TRACE
    std::vector<long long> tr(4 * 256);
    cudaMemcpyFromSymbol(tr.data(), gcm_sweep_trace, tr.size() * 8);
    double c = 0, b1 = 0, a = 0, tot = 0;
    int nt = 0;
    for (int tau = 5; tau < 60; ++tau, ++nt) {
        c += tr[tau * 4 + 1] - tr[tau * 4 + 0];
        b1 += tr[tau * 4 + 2] - tr[tau * 4 + 0];
        a += tr[tau * 4 + 3] - tr[tau * 4 + 2];
        tot += tr[(tau + 1) * 4 + 0] - tr[tau * 4 + 0];
    }
    printf("  per tick: compute-warp done %.0f, after bar1 %.0f, column phase %.0f, whole tick %.0f cycles\n", c / nt,
           b1 / nt, a / nt, tot / nt);
#endif
}

int main() {
#ifdef GCM_SWEEP_TRACE
    run<8, true, 2>(8, 1); dump_trace();
    run<16, true, 4>(16, 1); dump_trace();
    return 0;
#endif
    for (int ctas : {1, 148}) {
        run<8, false>(8, ctas);
        run<8, true, 1>(8, ctas);
        run<8, true, 2>(8, ctas);
        run<8, true, 4>(8, ctas);
        run<16, false>(16, ctas);
        run<16, true, 2>(16, ctas);
        run<16, true, 4>(16, ctas);
        run<32, false>(32, ctas);
        run<32, true, 4>(32, ctas);
    }
    return 0;
}
