// Throughput probe for the legacy warp-level integer tensor-core MMA on
// sm_100a: mma.sync.m16n8k32 u8 x u8 -> s32, independent accumulator chains
// in registers. Prints int8 MAC/s. Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o imma_probe tools/imma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CHAINS = 8;

__global__ void k_imma(int iters, int* out) {
    unsigned a[4], b[2];
    for (int i = 0; i < 4; ++i) a[i] = 0x01010101u * (threadIdx.x + i);
    for (int i = 0; i < 2; ++i) b[i] = 0x01010101u * (threadIdx.x + 7 * i);
    int c[CHAINS][4] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int ch = 0; ch < CHAINS; ++ch) {
            asm volatile(
                "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};\n"
                : "+r"(c[ch][0]), "+r"(c[ch][1]), "+r"(c[ch][2]), "+r"(c[ch][3])
                : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
        }
    }
    int s = 0;
    for (int ch = 0; ch < CHAINS; ++ch) s += c[ch][0] + c[ch][1] + c[ch][2] + c[ch][3];
    if (s == 0x12345) out[0] = s;
}

int main() {
    int* out;
    cudaMalloc(&out, 4);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int warps : {4, 8, 16, 32}) {
        const int iters = 4096, blocks = sms * 2;
        k_imma<<<blocks, warps * 16>>>(16, out);
        cudaEventRecord(e0);
        k_imma<<<blocks, warps * 16>>>(iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double macs = double(blocks) * (warps / 2) * iters * CHAINS * 16.0 * 8 * 32;
        printf("warps/SM %2d: %.1f T int8 MAC/s (%.3f ms) %s\n", warps, macs / ms / 1e9, ms,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
