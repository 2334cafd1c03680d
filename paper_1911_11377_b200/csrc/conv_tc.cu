// Plaintext-weight x ciphertext conv layers on the 5th-generation tensor
// cores (tcgen05.mma kind::i8, accumulators in TMEM) for limbs with q < 2^40:
// conv2d_encrypted (layers.hpp:174-211) -> mul_scalar_mac (ckks.hpp:448-465)
// summed over the taps of every output pixel.
//
// Per (component, limb) row, pixel p and a block of 128 coefficients j:
//   Y[j][oc] = sum_k X[k][j] W[k][oc] mod q,  X[k][j] = x[src(p, k)][comp][limb][j]
// Both factors are residues below 2^40: X = sum_a 2^8a X_a, W = sum_b 2^8b W_b
// (bytes), and Y = sum_s 2^8s D_s with D_s = sum_{a+b=s} X_a W_b (s = 0..8),
// each D_s an exact int32 while K <= 6144 (<= 5 * 255^2 * K < 2^31).
//
// The byte-plane diagonals fold into the MMA addressing: the B operand is the
// weight tile with all five byte planes side by side, N = 5 x 48 columns
// (b, oc), and the MMA of ciphertext plane a writes TMEM columns starting at
// a x 48, so column s x 48 + oc accumulates exactly sum_{a+b=s} X_a W_b: five
// 128 x 240 x 32 MMAs per 32-tap step, 9 x 48 = 432 accumulator columns, no
// wasted products. The epilogue reads D_s with tcgen05.ld and reduces
// sum_s D_s (2^8s mod q) with the exact FP64 modmul (ntt_core.cuh).
//
// Roles: warps 0-7 gather the ciphertext words (thread t: coefficient row
// j0 + t % 128, taps of K half t / 128; coalesced across the warp, the next
// step's words in flight while the current step is converted), split them
// into byte planes and write them with the weight tile into a STAGES-deep
// shared-memory ring in the UMMA K-major no-swizzle layout (8 x 16-byte core
// matrices), then run the epilogue of their TMEM lanes (channel half t / 128);
// warp 8 owns TMEM and one elected thread issues the MMAs. mbarriers order the
// ring (full: 256 producer arrivals after a proxy fence; empty:
// tcgen05.commit) and the accumulator (ready: commit; free: 256 epilogue
// arrivals after the lanes are read and re-zeroed).
// The 60-bit limb (WIDE) runs the same kernel with the six balanced signed
// base-256 digits of the weight integers W = round(w * Delta) (one copy for
// every limb) against the eight bytes of the ciphertext words: B = 6 x 32
// columns (signed), eight A planes, 13 x 32 = 416 accumulator columns, and a
// 64-bit Shoup fold of the 13 classes (|D_s| <= 6 * 128 * 255 * K < 2^31).
// Modular sums are order independent, so the words equal the reference's
// sequential accumulation.

#include <stdexcept>

#include "ntt_core.cuh"

namespace hecnn_b200 {

namespace {

#ifndef HECNN_TC_MIN_KSTEPS
#define HECNN_TC_MIN_KSTEPS 8
#endif
#ifndef HECNN_TC_GDEPTH
#define HECNN_TC_GDEPTH 3
#endif

constexpr int TC_M = 128;                   // coefficients per tile (TMEM lanes)
constexpr int TC_PRODUCERS = 256;           // 8 warps: (row j, K half) per thread
constexpr int TC_THREADS = TC_PRODUCERS + 32;
constexpr int TC_MMA_WARP = TC_PRODUCERS / 32;
constexpr int TC_GDEPTH = HECNN_TC_GDEPTH;  // gathered-word staging depth (steps in flight per thread)
constexpr int TC_GSTAGE_BYTES = TC_PRODUCERS * 16 * 8;
constexpr int TC_A_BYTES = TC_M * 32;       // one ciphertext byte plane, 32 taps

template <bool WIDE>
struct TcShape {
    static constexpr int NA = WIDE ? 8 : 5;        // ciphertext byte planes
    static constexpr int NB = WIDE ? 6 : 5;        // weight byte / signed-digit planes
    static constexpr int OC = WIDE ? 32 : 48;      // output channels per tile
    static constexpr int N = NB * OC;              // B columns (b, oc): 192 / 240
    static constexpr int NS = NA + NB - 1;         // shift classes: 13 / 9
    static constexpr int STAGES = WIDE ? 3 : 4;
    static constexpr int B_BYTES = N * 32;
    static constexpr int STAGE_BYTES = NA * TC_A_BYTES + B_BYTES;
    static constexpr int SMEM = STAGES * STAGE_BYTES + TC_GDEPTH * TC_GSTAGE_BYTES + 2048;  // + alignment slack, barriers
    // kind::i8 instruction descriptor: D s32, A unsigned 8-bit, B unsigned (signed
    // digits when WIDE), both K-major, M x N
    static constexpr uint32_t IDESC = (2u << 4) | ((WIDE ? 1u : 0u) << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
                                      (static_cast<uint32_t>(TC_M >> 4) << 24);
    static_assert(NS * OC <= 512, "accumulator exceeds the TMEM columns");
    static_assert(SMEM <= 227 * 1024, "shared memory");
};

__device__ __forceinline__ uint32_t s_addr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// K-major, no swizzle: core matrices of 8 rows x 16 B (128 B contiguous); the
// two 16-byte K halves 128 B apart (LBO), row groups 256 B apart (SBO).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
    uint64_t d = (saddr >> 4) & 0x3FFF;
    d |= static_cast<uint64_t>(128 >> 4) << 16;
    d |= static_cast<uint64_t>(256 >> 4) << 32;
    d |= 1ull << 46;  // descriptor version (sm_100)
    return d;
}

__device__ __forceinline__ int core_off(int row, int k) { return (row >> 3) * 256 + (k >> 4) * 128 + (row & 7) * 16 + (k & 15); }

__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_addr(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("{.reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0];}" ::"r"(s_addr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    asm volatile(
        "{.reg .pred P1;\n"
        "WAIT_%=: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;}" ::"r"(s_addr(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 4x4 byte transpose of four 32-bit words: p[a] = byte a of each word, word u in byte u.
__device__ __forceinline__ void transpose4(unsigned l0, unsigned l1, unsigned l2, unsigned l3, unsigned* p) {
    const unsigned x01 = __byte_perm(l0, l1, 0x5140), x01h = __byte_perm(l0, l1, 0x7362);
    const unsigned x23 = __byte_perm(l2, l3, 0x5140), x23h = __byte_perm(l2, l3, 0x7362);
    p[0] = __byte_perm(x01, x23, 0x5410);
    p[1] = __byte_perm(x01, x23, 0x7632);
    p[2] = __byte_perm(x01h, x23h, 0x5410);
    p[3] = __byte_perm(x01h, x23h, 0x7632);
}

__device__ __forceinline__ void tmem_ld8(uint32_t addr, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(addr));
}
__device__ __forceinline__ void tmem_zero8(uint32_t addr) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(addr), "r"(0u));
}

// blockIdx.x = (column block * pixels + pixel) * tiles + oc tile: the CTAs
// resident at any time cover a few column blocks, whose slice of every input
// cell (cells x 1 KB) stays L2-resident while all pixels and channel tiles
// gather from it. One (pixel, oc tile) per CTA.
template <bool WIDE>
__global__ void __launch_bounds__(TC_THREADS, 1) k_conv_tc(DevRing R, ImmaMac g, const u64* __restrict__ x,
                                                          u64* __restrict__ y, int level, int limb0, int nl) {
    using S = TcShape<WIDE>;
    constexpr int NA = S::NA, NS = S::NS, OC = S::OC, STAGES = S::STAGES;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1 KB-aligned base, by offset so the compiler keeps shared-space stores
    unsigned char* smem = smem_raw + ((1024u - (s_addr(smem_raw) & 1023u)) & 1023u);
    u64* gstage = reinterpret_cast<u64*>(smem + STAGES * S::STAGE_BYTES);  // [GDEPTH][16 words][producers]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * S::STAGE_BYTES + TC_GDEPTH * TC_GSTAGE_BYTES);
    uint64_t* full = bars;               // [STAGES]
    uint64_t* empty = bars + STAGES;     // [STAGES]
    uint64_t* acc_ready = bars + 2 * STAGES;
    uint64_t* acc_free = acc_ready + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_free + 1);

    const int tid = threadIdx.x, warp = tid >> 5;
    const int limbs = level + 1;
    const long long poly_words = static_cast<long long>(limbs) * R.n;
    const long long cell_words = 2 * poly_words;
    const int nj = R.n / TC_M;
    const int tiles = (g.oc + OC - 1) / OC;
    const long long bid = blockIdx.x;
    const int ot = static_cast<int>(bid % tiles);
    const long long pix_cb = bid / tiles;
    const long long cb = pix_cb / g.pixels;
    const int p = static_cast<int>(pix_cb - cb * g.pixels);
    const int jb = static_cast<int>(cb % nj);
    const int row = static_cast<int>(cb / nj);
    const int comp = row / nl, i = limb0 + row % nl;
    const int j0 = jb * TC_M;
    const long long col_base = comp * poly_words + static_cast<long long>(i) * R.n + j0;
    const int ks_n = g.ksteps;

    if (warp == TC_MMA_WARP) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s_addr(tmem_slot)), "n"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full + s, TC_PRODUCERS);
            mbar_init(empty + s, 1);
        }
        mbar_init(acc_ready, 1);
        mbar_init(acc_free, TC_PRODUCERS);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp < TC_MMA_WARP) {
        const int r = tid & (TC_M - 1), kh = tid / TC_M;  // coefficient row, K half / channel half
        const uint32_t lane_base = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16);
        constexpr int HOC = OC / 2;
        static_assert(HOC % 8 == 0, "epilogue chunks of 8 channels");
        // this thread's channel half of every shift class starts at zero (the plane
        // ranges overlap, so every MMA accumulates)
#pragma unroll
        for (int s = 0; s < NS; ++s)
#pragma unroll
            for (int c = 0; c < HOC; c += 8) tmem_zero8(lane_base + s * OC + kh * HOC + c);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        mbar_arrive(acc_free);  // the accumulator is ready for the MMAs

#ifndef HECNN_TC_G16
#define HECNN_TC_G16 0
#endif
        // producer mapping: G16 -> a thread owns two adjacent coefficient rows and
        // 8 taps (16-byte cp.async per tap), else one row and 16 taps (8-byte copies)
        constexpr bool G16 = HECNN_TC_G16;
        constexpr int ROWS = G16 ? 2 : 1, TAPS = G16 ? 8 : 16;
        const int prow = G16 ? 2 * (tid & 63) : r;         // first row of this thread
        const int pk0 = G16 ? 8 * (tid >> 6) : 16 * kh;     // first tap of this thread within a step
        const u64* xcol = x + col_base + prow;
        const uint4* wt = (WIDE ? g.wtc_wide : g.wtc + static_cast<long long>(i) * tiles * ks_n * (S::B_BYTES / 16)) +
                          static_cast<long long>(ot) * ks_n * (S::B_BYTES / 16);
        // this thread's tap words of step ks, gathered with cp.async into the
        // staging ring (padding taps, -1, zero-fill); each thread reads back
        // only its own words, so cp.async.wait_group alone orders the ring.
        // Steps are gathered in order; the tap indices of the next one are
        // loaded one gather ahead so their latency is off the issue path.
        const int* src_p = g.src + static_cast<long long>(p) * g.kpad + pk0;
        int4 taps[TAPS / 4];
        auto load_taps = [&](int ks) {
#pragma unroll
            for (int c = 0; c < TAPS / 4; ++c) taps[c] = __ldg(reinterpret_cast<const int4*>(src_p + ks * 32 + 4 * c));
        };
        load_taps(0);
        auto gather = [&](int ks) {
            // staging slot: [tap][thread] entries of ROWS words
            u64* dst = gstage + (ks % TC_GDEPTH) * (16 * TC_PRODUCERS) + tid * ROWS;
            int tt[TAPS];
#pragma unroll
            for (int c = 0; c < TAPS / 4; ++c) tt[4 * c] = taps[c].x, tt[4 * c + 1] = taps[c].y, tt[4 * c + 2] = taps[c].z, tt[4 * c + 3] = taps[c].w;
            if (ks + 1 < ks_n) load_taps(ks + 1);
#pragma unroll
            for (int u = 0; u < TAPS; ++u) {
                const u64* from = xcol + static_cast<long long>(max(tt[u], 0)) * cell_words;
                if constexpr (G16)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s_addr(dst + u * 2 * TC_PRODUCERS)), "l"(from),
                                 "r"(tt[u] >= 0 ? 16 : 0)
                                 : "memory");
                else
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s_addr(dst + u * TC_PRODUCERS)), "l"(from),
                                 "r"(tt[u] >= 0 ? 8 : 0)
                                 : "memory");
            }
        };
#pragma unroll
        for (int d = 0; d < TC_GDEPTH; ++d) {
            if (d < ks_n) gather(d);
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        for (int ks = 0; ks < ks_n; ++ks) {
            asm volatile("cp.async.wait_group %0;" ::"n"(TC_GDEPTH - 1) : "memory");  // step ks landed
            u64 cur[ROWS][TAPS];
            {
                const u64* from = gstage + (ks % TC_GDEPTH) * (16 * TC_PRODUCERS) + tid * ROWS;
#pragma unroll
                for (int u = 0; u < TAPS; ++u) {
                    if constexpr (G16) {
                        const ulonglong2 v2 = *reinterpret_cast<const ulonglong2*>(from + u * 2 * TC_PRODUCERS);
                        cur[0][u] = v2.x;
                        cur[ROWS - 1][u] = v2.y;
                    } else {
                        cur[0][u] = from[u * TC_PRODUCERS];
                    }
                }
            }
            const int stage = ks % STAGES;
            if (ks >= STAGES) mbar_wait(empty + stage, ((ks / STAGES) - 1) & 1);
            unsigned char* st = smem + stage * S::STAGE_BYTES;
#pragma unroll
            for (int rr = 0; rr < ROWS; ++rr) {
                // byte planes a < NA of row prow + rr, this thread's taps
                unsigned pl[NA][TAPS / 4];
#pragma unroll
                for (int c = 0; c < TAPS / 4; ++c) {
                    const u64* ww = cur[rr] + 4 * c;
                    unsigned p4[4];
                    transpose4(static_cast<unsigned>(ww[0]), static_cast<unsigned>(ww[1]), static_cast<unsigned>(ww[2]),
                               static_cast<unsigned>(ww[3]), p4);
#pragma unroll
                    for (int a = 0; a < 4; ++a) pl[a][c] = p4[a];
                    const unsigned h0 = static_cast<unsigned>(ww[0] >> 32), h1 = static_cast<unsigned>(ww[1] >> 32);
                    const unsigned h2 = static_cast<unsigned>(ww[2] >> 32), h3 = static_cast<unsigned>(ww[3] >> 32);
                    if constexpr (WIDE) {
                        transpose4(h0, h1, h2, h3, p4);
#pragma unroll
                        for (int a = 0; a < 4; ++a) pl[4 + a][c] = p4[a];
                    } else {
                        pl[4][c] = __byte_perm(__byte_perm(h0, h1, 0x0040), __byte_perm(h2, h3, 0x0040), 0x5410);
                    }
                }
#pragma unroll
                for (int a = 0; a < NA; ++a) {
                    unsigned char* dst = st + a * TC_A_BYTES + core_off(prow + rr, pk0);
                    if constexpr (G16) *reinterpret_cast<uint2*>(dst) = make_uint2(pl[a][0], pl[a][1]);
                    else *reinterpret_cast<uint4*>(dst) = make_uint4(pl[a][0], pl[a][1], pl[a][2], pl[a][3]);
                }
            }
            // refill the staging slot just read (its words are consumed: the plane stores used them)
            if (ks + TC_GDEPTH < ks_n) gather(ks + TC_GDEPTH);
            asm volatile("cp.async.commit_group;" ::: "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor-core reads
            if (tid == 0) {
                // the weight tile (already in the core-matrix layout): one bulk copy on
                // the async proxy, counted on the same barrier as transaction bytes
                const uint4* wsrc = wt + static_cast<long long>(ks) * (S::B_BYTES / 16);
                asm volatile("{.reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;}" ::"r"(s_addr(full + stage)),
                             "r"(S::B_BYTES)
                             : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                 s_addr(st + NA * TC_A_BYTES)),
                             "l"(wsrc), "r"(S::B_BYTES), "r"(s_addr(full + stage))
                             : "memory");
            } else {
                mbar_arrive(full + stage);
            }
        }

        // epilogue: D_s from TMEM (lane = this coefficient), this channel half
        mbar_wait(acc_ready, 0);
        tc_fence_after();
        const u64 q = R.mod[i].q;
        const int j = j0 + r;
#pragma unroll 1
        for (int c0 = kh * HOC; c0 < kh * HOC + HOC; c0 += 8) {
            uint32_t d[NS][8];
#pragma unroll
            for (int s = 0; s < NS; ++s) tmem_ld8(lane_base + s * OC + c0, d[s]);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int o = 0; o < 8; ++o) {
                const int oc = ot * OC + c0 + o;
                u64 res;
                if constexpr (WIDE) {
                    // classes in pairs: |D_s + 2^8 D_s+1| < 2^31 * 257 < 2^40 <= q, so one
                    // conditional add of q makes the pair canonical
                    const ulonglong2* cs = g.shift_wide + i * 16;
                    res = 0;
#pragma unroll
                    for (int s = 0; s < NS; s += 2) {
                        long long t = static_cast<int>(d[s][o]);
                        if (s + 1 < NS) t += static_cast<long long>(static_cast<int>(d[s + 1][o])) * 256;
                        const u64 rr = t >= 0 ? static_cast<u64>(t) : q - static_cast<u64>(-t);
                        const ulonglong2 k = __ldg(cs + s);
                        res = add_mod(res, mul_shoup(rr, k.x, k.y, q), q);
                    }
                } else {
                    const double qd = static_cast<double>(q), qinv = R.inv_q[i];
                    const double* cs = g.shift + i * 9;
                    auto D = [&](int s) { return static_cast<double>(d[s][o]); };
                    double v;
                    if (ks_n <= 48) {  // D_s < 2^29: three classes per exact double
                        v = ntt::fmodmul(D(0) + 256.0 * D(1) + 65536.0 * D(2), __ldg(cs + 0), qd, qinv);
                        v += ntt::fmodmul(D(3) + 256.0 * D(4) + 65536.0 * D(5), __ldg(cs + 3), qd, qinv);
                        v += ntt::fmodmul(D(6) + 256.0 * D(7) + 65536.0 * D(8), __ldg(cs + 6), qd, qinv);
                    } else {
                        v = 0.0;
#pragma unroll
                        for (int s = 0; s < 9; ++s) v += ntt::fmodmul(D(s), __ldg(cs + s), qd, qinv);
                    }
                    res = ntt::fcanon(v, qd, qinv);
                }
                if (oc < g.oc) {
                    if (g.bias && comp == 0 && j == 0) res = add_mod(res, g.bias[static_cast<long long>(oc) * limbs + i], q);
                    y[(static_cast<long long>(p) * g.out_stride_pixel + oc) * cell_words + col_base + r] = res;
                }
            }
        }
    } else if ((tid & 31) == 0) {
        // MMA issuer: one elected thread of warp 8
        const uint32_t a0 = s_addr(smem);
        mbar_wait(acc_free, 0);  // the producers zeroed the accumulator
        tc_fence_after();
        for (int ks = 0; ks < ks_n; ++ks) {
            const int stage = ks % STAGES;
            mbar_wait(full + stage, (ks / STAGES) & 1);
            tc_fence_after();
            const uint32_t sa = a0 + stage * S::STAGE_BYTES;
            const uint64_t db = umma_desc(sa + NA * TC_A_BYTES);
#pragma unroll
            for (int a = 0; a < NA; ++a) {
                const uint64_t da = umma_desc(sa + a * TC_A_BYTES);
                asm volatile(
                    "{.reg .pred p; setp.ne.b32 p, %4, 0;\n"
                    "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;}" ::"r"(tmem + a * OC),
                    "l"(da), "l"(db), "r"(S::IDESC), "r"(1u));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             s_addr(empty + stage))
                         : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s_addr(acc_ready))
                     : "memory");
    }
    tc_fence_before();
    __syncthreads();
    if (warp == TC_MMA_WARP) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
    }
}

}  // namespace

int tc_oc_tile(bool wide) { return wide ? TcShape<true>::OC : TcShape<false>::OC; }

bool tc_mac_supported(const DevRing& R, const ImmaMac& g, bool wide) {
    // one exact int32 chunk (K <= 6144); short K stays on mma.sync (the
    // per-tile epilogue would dominate a handful of MMAs)
    return (wide ? g.wtc_wide != nullptr : g.wtc != nullptr) && R.n % TC_M == 0 && g.ksteps >= HECNN_TC_MIN_KSTEPS &&
           g.ksteps <= 192;
}

void tc_mac(const DevRing& R, const ImmaMac& g, const u64* x, u64* y, int level, int limb0, int limb1, bool wide,
            const Launch& L) {
    const int nl = limb1 - limb0;
    if (!g.pixels || !g.oc || nl <= 0) return;
    if (!tc_mac_supported(R, g, wide)) throw std::invalid_argument("tc_mac: unsupported shape");
    auto kern = wide ? k_conv_tc<true> : k_conv_tc<false>;
    const int smem = wide ? TcShape<true>::SMEM : TcShape<false>::SMEM;
    const int oc_tile = tc_oc_tile(wide);
    smem_opt_in(kern, smem);
    const long long rows = 2LL * nl, nj = R.n / TC_M;
    const long long blocks = rows * nj * g.pixels * ((g.oc + oc_tile - 1) / oc_tile);
    if (blocks > 0x7fffffffLL) throw std::runtime_error("tc_mac: grid too large");
    const double ncols = double(rows) * R.n;
    L.begin(wide ? "k_conv_tc_wide" : "k_conv_tc", double(g.pixels) * g.K * g.oc * ncols,
            8.0 * ncols * (double(g.pixels) * g.oc + double(g.pixels) * g.K));
    kern<<<static_cast<unsigned>(blocks), TC_THREADS, smem, L.stream>>>(R, g, x, y, level, limb0, nl);
    L.count();
    check_launch(wide ? "tc_mac_wide" : "tc_mac");
}

}  // namespace hecnn_b200
