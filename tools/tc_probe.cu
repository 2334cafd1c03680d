// tcgen05 kind::i8 probe (experiment, not product): D[128 x N] (s32, TMEM) =
// sum_a A_a[128 x 32] (u8) x B[N x 32]^T (u8) written at TMEM column offset
// a * OC, i.e. the byte-plane diagonal trick the conv kernel uses. Checks the
// smem descriptor / instruction descriptor encodings against a CPU GEMM.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

constexpr int M = 128, K = 32, OC = 48, NB = 5, N = NB * OC, NA = 5, COLS = (NA + NB - 1) * OC;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// K-major, no swizzle: core matrix = 8 rows x 16 B contiguous; K halves 128 B apart (LBO), row groups 256 B (SBO)
__device__ __forceinline__ uint64_t desc_kmajor(const void* base) {
    const uint64_t addr = smem_u32(base);
    uint64_t d = 0;
    d |= (addr >> 4) & 0x3FFF;                 // start address
    d |= static_cast<uint64_t>(128 >> 4) << 16;  // LBO
    d |= static_cast<uint64_t>(256 >> 4) << 32;  // SBO
    d |= 1ull << 46;                           // version (sm100)
    return d;                                  // layout 0 = SWIZZLE_NONE, base offset 0
}
__host__ __device__ constexpr uint32_t idesc_u8(int m, int n) {
    return (2u << 4)                 // D = s32
         | (0u << 7) | (0u << 10)    // A, B unsigned 8-bit
         | (0u << 15) | (0u << 16)   // K-major both
         | (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}
__device__ __forceinline__ int koff(int row, int k) { return (row / 8) * 256 + (k / 16) * 128 + (row % 8) * 16 + (k % 16); }

__global__ void k_probe(const uint8_t* A, const uint8_t* B, int* D) {
    __shared__ __align__(1024) uint8_t sa[NA][M * K];
    __shared__ __align__(1024) uint8_t sb[N * K];
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid / 32;
    for (int e = tid; e < NA * M * K; e += blockDim.x) {
        const int a = e / (M * K), r = (e / K) % M, k = e % K;
        sa[a][koff(r, k)] = A[e];
    }
    for (int e = tid; e < N * K; e += blockDim.x) sb[koff(e / K, e % K)] = B[e];
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "n"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tbase;
    {   // zero the accumulator columns (plane ranges overlap, so every MMA accumulates)
        const uint32_t z = 0;
        for (int c = 0; c < COLS; c += 16)
            asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};"
                         ::"r"(tm + (static_cast<uint32_t>(warp * 32) << 16) + c), "r"(z));
        asm volatile("tcgen05.wait::st.sync.aligned;");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;");
    }
    if (tid == 0) {
        const uint64_t db = desc_kmajor(sb);
        for (int a = 0; a < NA; ++a) {
            const uint64_t da = desc_kmajor(sa[a]);
            // first MMA into each column range must not read stale TMEM: planes a>0 overlap a-1's range, so
            // zero-init via enable_input_d = 0 only for a == 0 and pre-clear the tail with tcgen05.st instead
            const uint32_t acc = 1u;
            asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;}"
                         ::"r"(tm + a * OC), "l"(da), "l"(db), "r"(idesc_u8(M, N)), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    }
    // wait for the MMAs
    asm volatile("{.reg .pred P1; WAIT: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1; @!P1 bra WAIT;}" ::"r"(smem_u32(&bar)), "r"(0));
    asm volatile("tcgen05.fence::after_thread_sync;");
    // warp w reads lanes 32w..32w+31: row = tid
    for (int c = 0; c < COLS; c += 16) {
        uint32_t v[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(tm + (static_cast<uint32_t>(warp * 32) << 16) + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int q = 0; q < 16; ++q) D[tid * COLS + c + q] = static_cast<int>(v[q]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "n"(512));
}

int main() {
    std::vector<uint8_t> A(NA * M * K), B(N * K);
    srand(1);
    for (auto& v : A) v = rand() & 255;
    for (auto& v : B) v = rand() & 255;
    // CPU: D[r][s*OC + oc] = sum_{a+b=s} sum_k A_a[r][k] B[b*OC+oc][k]; columns >= (a+b) range never written
    // for s>=5 until a>0 -- all columns s in 0..8 are covered by some (a,b)
    std::vector<long long> want(M * COLS, 0);
    for (int a = 0; a < NA; ++a)
        for (int r = 0; r < M; ++r)
            for (int n = 0; n < N; ++n) {
                long long s = 0;
                for (int k = 0; k < K; ++k) s += A[(a * M + r) * K + k] * B[n * K + k];
                want[r * COLS + a * OC + n] += s;
            }
    uint8_t *dA, *dB;
    int* dD;
    cudaMalloc(&dA, A.size());
    cudaMalloc(&dB, B.size());
    cudaMalloc(&dD, M * COLS * 4);
    cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, M * COLS * 4);
    k_probe<<<1, 128>>>(dA, dB, dD);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<int> got(M * COLS);
    cudaMemcpy(got.data(), dD, got.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0, first = -1;
    for (int i = 0; i < M * COLS; ++i)
        if (got[i] != want[i]) { if (first < 0) first = i; ++bad; }
    printf("status %s, mismatches %d / %d", cudaGetErrorString(e), bad, M * COLS);
    if (first >= 0) printf(" (first at row %d col %d: got %d want %lld)", first / COLS, first % COLS, got[first], want[first]);
    printf("\n");
    return bad != 0;
}
