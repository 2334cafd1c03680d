// Throughput probe (experiment, not product): chained 64-bit Shoup modmuls on
// the integer pipes vs an exact FP64 modmul for q < 2^42 (error-free FMA
// product + magic-constant quotient rounding + exact FMA remainder), and both
// interleaved. Also verifies the FP64 result against the integer one.
#include <cstdio>
#include <cstdint>
#include <cmath>

typedef unsigned long long u64;

__device__ __forceinline__ u64 shoup_lazy(u64 x, u64 w, u64 ws, u64 q) { return x * w - __umul64hi(x, ws) * q; }

// r = x*w mod q in (-q, q), exact for |x| < 2^45, 0 <= w < q < 2^42 (the
// product's rounded high part h also gives the quotient: t = rint(h / q))
__device__ __forceinline__ double fmodmul(double x, double w, double qinv, double q) {
    const double M = 6755399441055744.0;  // 1.5 * 2^52
    double h = x * w;
    double l = fma(x, w, -h);
    double t = fma(h, qinv, M) - M;
    double r = fma(-t, q, h);
    return r + l;
}

__global__ void k_int(int iters, u64 q, u64 w, u64 ws, u64* sink) {
    u64 x[8];
    for (int k = 0; k < 8; ++k) x[k] = (blockIdx.x * 256ull + threadIdx.x) * 8 + k + 1;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = shoup_lazy(x[k], w, ws, q);
    u64 a = 0;
    for (int k = 0; k < 8; ++k) a ^= x[k];
    if (a == 12345) sink[0] = a;
}

__global__ void k_fp(int iters, double q, double w, double wq, double* sink) {
    double x[8];
    for (int k = 0; k < 8; ++k) x[k] = (double)((blockIdx.x * 256ull + threadIdx.x) * 8 + k + 1);
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fmodmul(x[k], w, wq, q);
    double a = 0;
    for (int k = 0; k < 8; ++k) a += x[k];
    if (a == 12345.0) sink[0] = a;
}

__global__ void k_mix(int iters, u64 q, u64 w, u64 ws, double qd, double wd, double wqd, u64* sink) {
    u64 x[4];
    double y[4];
    for (int k = 0; k < 4; ++k) {
        x[k] = (blockIdx.x * 256ull + threadIdx.x) * 8 + k + 1;
        y[k] = (double)(x[k] + 7);
    }
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            x[k] = shoup_lazy(x[k], w, ws, q);
            y[k] = fmodmul(y[k], wd, wqd, qd);
        }
    u64 a = 0;
    for (int k = 0; k < 4; ++k) a ^= x[k] ^ (u64)(long long)y[k];
    if (a == 12345) sink[0] = a;
}

__global__ void k_check(u64 q, u64 w, double wq, int n, int* bad) {
    for (long long t = blockIdx.x * 256ll + threadIdx.x; t < n; t += gridDim.x * 256ll) {
        // x spans (-2^44, 2^44), both signs
        long long xs = (long long)((t * 0x9E3779B97F4A7C15ull) >> 18) - (1ll << 45);  // |x| < 2^45
        double r = fmodmul((double)xs, (double)w, wq, (double)q);
        long long want = (long long)(((__int128)xs * (__int128)w) % (__int128)q);
        long long got = (long long)r;
        long long diff = got - want;
        if (!(r > -(double)q && r < (double)q) || (diff % (long long)q) != 0) atomicAdd(bad, 1);
    }
}

int main() {
    const u64 q = 1099511480321ull;  // 40-bit NTT prime of the nn/net presets
    const u64 w = 123456789012ull % q;
    const u64 ws = (u64)(((unsigned __int128)w << 64) / q);
    const double wq = 1.0 / (double)q;  // qinv
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    u64* sink;
    cudaMalloc(&sink, 64);
    int* bad;
    cudaMalloc(&bad, 4);
    cudaMemset(bad, 0, 4);
    k_check<<<sms * 4, 256>>>(q, w, wq, 1 << 26, bad);
    int hbad = -1;
    cudaMemcpy(&hbad, bad, 4, cudaMemcpyDeviceToHost);
    printf("fp64 modmul exactness: %d mismatches in 2^26 signed inputs |x| < 2^45\n", hbad);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int blocks = sms * 8, iters = 4096;
    const double ops = (double)blocks * 256 * 8 * iters;
    float ms;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        k_int<<<blocks, 256>>>(iters, q, w, ws, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("int  shoup : %.1f Gmodmul/s\n", ops / (ms * 1e6));
        cudaEventRecord(a);
        k_fp<<<blocks, 256>>>(iters, (double)q, (double)w, wq, (double*)sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("fp64 exact : %.1f Gmodmul/s\n", ops / (ms * 1e6));
        cudaEventRecord(a);
        k_mix<<<blocks, 256>>>(iters, q, w, ws, (double)q, (double)w, wq, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("mixed 1:1  : %.1f Gmodmul/s\n", ops / (ms * 1e6));
    }
    return 0;
}
