// Inter-SM flag ping-pong: one-way latency of a relaxed/release store seen by a
// polling relaxed/acquire load on another SM (B200).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pingpong tools/pingpong.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// mode 0: relaxed/relaxed, 1: release/acquire, 2: relaxed + __threadfence before store
__global__ void pingpong(unsigned long long *a, unsigned long long *b, int iters, int mode, long long *out) {
    const bool ping = blockIdx.x == 0;
    if (threadIdx.x != 0) return;
    unsigned long long *mine = ping ? a : b, *theirs = ping ? b : a;
    long long t0 = clock64();
    for (int i = 1; i <= iters; ++i) {
        if (ping) {
            if (mode == 1) st_release(mine, i);
            else {
                if (mode == 2) __threadfence();
                st_relaxed(mine, i);
            }
            if (mode == 1) while (ld_acquire(theirs) != (unsigned long long)i) {}
            else while (ld_relaxed(theirs) != (unsigned long long)i) {}
        } else {
            if (mode == 1) while (ld_acquire(theirs) != (unsigned long long)i) {}
            else while (ld_relaxed(theirs) != (unsigned long long)i) {}
            if (mode == 1) st_release(mine, i);
            else {
                if (mode == 2) __threadfence();
                st_relaxed(mine, i);
            }
        }
    }
    long long t1 = clock64();
    if (ping) out[0] = t1 - t0;
}


__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// one-way latency via globaltimer: ping records send time, pong records receive time
__global__ void oneway(unsigned long long *a, long long *ts, int iters) {
    if (threadIdx.x != 0) return;
    for (int i = 1; i <= iters; ++i) {
        if (blockIdx.x == 0) {
            // wait for ack of previous
            while (ld_relaxed(a + 64) != (unsigned long long)(i - 1)) {}
            for (int d = 0; d < 2000; ++d) __nanosleep(1);  // random-ish gap
            ts[2 * i] = gtimer();
            st_relaxed(a, i);
        } else {
            while (ld_relaxed(a) != (unsigned long long)i) {}
            ts[2 * i + 1] = gtimer();
            st_relaxed(a + 64, i);
        }
    }
}

int main() {
    unsigned long long *a, *b;
    long long *out;
    cudaMalloc(&a, 4096);
    cudaMalloc(&b, 4096);
    cudaMalloc(&out, 64);
    const int iters = 2000;
    const char *names[] = {"relaxed/relaxed", "release/acquire", "fence+relaxed"};
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaMemset(a, 0, 4096);
            cudaMemset(b, 0, 4096);
            pingpong<<<2, 32>>>(a, b + 256, iters, mode, out);
            long long h = 0;
            cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
            printf("%-16s round trip %.0f cycles (one-way %.0f)\n", names[mode], (double)h / iters, (double)h / iters / 2);
        }
    }
    long long *ts;
    cudaMalloc(&ts, 8 * 2 * 1100);
    cudaMemset(a, 0, 4096);
    oneway<<<2, 32>>>(a, ts, 1000);
    long long hts[2 * 1001];
    cudaMemcpy(hts, ts, sizeof(hts), cudaMemcpyDeviceToHost);
    double s = 0, mn = 1e18, mx = -1e18;
    for (int i = 2; i <= 1000; ++i) { double d = (double)(hts[2 * i + 1] - hts[2 * i]); s += d; mn = d < mn ? d : mn; mx = d > mx ? d : mx; }
    printf("globaltimer one-way: mean %.0f ns min %.0f max %.0f\n", s / 999, mn, mx);
    return 0;
}
