// Plaintext-weight x ciphertext layers on the integer tensor cores (K8 in
// SURVEY.md §2.3; conv2d_encrypted layers.hpp:174-211, dense_encrypted
// :269-293), for limbs with q < 2^40.
//
// Per (component, limb, coefficient) column the layer is an exact integer
// GEMM with a gather: y[pixel][oc] = sum_k W[k][oc] x[src(pixel,k)] mod q.
// Both factors are residues below 2^40, so they split into five unsigned
// bytes each (x = sum_a x_a 2^8a, W = sum_b W_b 2^8b) and
//   sum_k W x = sum_s 2^8s D_s,  D_s = sum_{a+b=s} sum_k W_b x_a   (s = 0..8)
// where every D_s is an exact int32 sum of u8 x u8 products while K <= 6144
// (at most five byte pairs per s: 5 * 255^2 * 6144 < 2^31). The D_s are
// mma.sync.m16n8k32 u8.u8.s32 tensor-core products (25 per 32-tap step: the
// weight byte planes are the A operand, stored in global memory already in
// fragment order; the ciphertext byte planes are the B operand, transposed
// out of 64-bit words with byte permutes in registers). The epilogue reduces
// sum_s D_s (2^8s mod q) with the exact FP64 modmul of ntt_core.cuh; longer
// K folds the int32 sums into FP64 residues every 6144 taps. Modular sums
// are order independent, so the words equal the reference's sequential
// mul_scalar_mac accumulation (ckks.hpp:448-465).
//
// Tiling: a warp owns 8 consecutive columns of one (component, limb) row and
// MT x 16 output channels; a CTA is 4 warps = 32 columns of one pixel (a
// group of pixels when K is short). The grid is column-block major (pixels
// fastest), so a column block of every input cell stays L2-resident while all
// pixels consume it. Operands stream through a STAGES-deep cp.async ring in
// shared memory: each thread's gathered ciphertext words, and the CTA's
// weight fragments (one copy shared by the four warps); the pixel's tap
// table is staged once.

#include <stdexcept>

#include "ntt_core.cuh"

namespace hecnn_b200 {

namespace {

constexpr int WARPS = 4;
constexpr int KSTEP = 32;
constexpr int FOLD_STEPS = 192;  // 6144 taps per exact int32 accumulation chunk

__device__ __forceinline__ void imma(int (&c)[4], const uint4& a, unsigned b0, unsigned b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void imma_s8(int (&c)[4], const uint4& a, unsigned b0, unsigned b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
}

constexpr int STAGES = 4;
constexpr int KSRC = 3584;  // taps staged in shared memory (conv K up to 3 x 3 x 384); longer K reads L2

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// 4x4 byte transpose of four 32-bit words: p[a] = byte a of each word, word u in byte u.
__device__ __forceinline__ void transpose4(unsigned l0, unsigned l1, unsigned l2, unsigned l3, unsigned* p) {
    const unsigned x01 = __byte_perm(l0, l1, 0x5140), x01h = __byte_perm(l0, l1, 0x7362);
    const unsigned x23 = __byte_perm(l2, l3, 0x5140), x23h = __byte_perm(l2, l3, 0x7362);
    p[0] = __byte_perm(x01, x23, 0x5410);
    p[1] = __byte_perm(x01, x23, 0x7632);
    p[2] = __byte_perm(x01h, x23h, 0x5410);
    p[3] = __byte_perm(x01h, x23h, 0x7632);
}

// Byte planes of four words (taps k..k+3 of one column), the B-fragment
// order along K: NA = 5 for residues below 2^40, 8 for full words.
template <int NA>
__device__ __forceinline__ void byte_planes(const u64 (&w)[4], unsigned (&p)[NA]) {
    transpose4(static_cast<unsigned>(w[0]), static_cast<unsigned>(w[1]), static_cast<unsigned>(w[2]),
               static_cast<unsigned>(w[3]), p);
    const unsigned h0 = static_cast<unsigned>(w[0] >> 32), h1 = static_cast<unsigned>(w[1] >> 32);
    const unsigned h2 = static_cast<unsigned>(w[2] >> 32), h3 = static_cast<unsigned>(w[3] >> 32);
    if constexpr (NA == 8) {
        transpose4(h0, h1, h2, h3, p + 4);
    } else {
        static_assert(NA == 5, "5 or 8 byte planes");
        p[4] = __byte_perm(__byte_perm(h0, h1, 0x0040), __byte_perm(h2, h3, 0x0040), 0x5410);
    }
}

// SHORT: every accumulation chunk has <= 48 steps (three shift classes per
// exact double in the fold); otherwise classes are folded in pairs.
template <bool WIDE, int MT>
struct ImmaShape {
    static constexpr int NA = WIDE ? 8 : 5;        // ciphertext byte planes
    static constexpr int NB = WIDE ? 6 : 5;        // weight digit planes
    static constexpr int NS = NA + NB - 1;         // shift classes
    static constexpr int XWORDS = STAGES * 8 * WARPS * 32;        // u64
    static constexpr int WCHUNKS = MT * NB * 32;                  // uint4 per stage
    static constexpr int SMEM = XWORDS * 8 + STAGES * WCHUNKS * 16 + KSRC * 4;
};

// WIDE = false: limbs with q < 2^40, weights = the five unsigned bytes of each
// limb's residue (u8 x u8, FP64 fold). WIDE = true: limbs with q >= 2^40 (the
// 60-bit q0): weights = the six balanced signed base-256 digits of the weight
// integer W = round(w * Delta) (|W| < 2^47, one copy for all limbs), the
// ciphertext words as eight unsigned bytes; 48 s8 x u8 products per tap in
// 13 classes, each an exact int32 (|D_s| <= 6 * 128 * 255 * 6144 < 2^31);
// 64-bit Shoup fold. SHORT: every accumulation chunk has <= 48 steps (three
// classes per exact double in the FP64 fold).
template <int MT, bool SHORT, bool WIDE>
__global__ void __launch_bounds__(WARPS * 32) k_conv_imma(DevRing R, ImmaMac g, const u64* __restrict__ x,
                                                         u64* __restrict__ y, int level, int limb0, int nl,
                                                         int groups, int pg) {
    using S = ImmaShape<WIDE, MT>;
    constexpr int NA = S::NA, NB = S::NB, NS = S::NS;
    extern __shared__ __align__(16) unsigned char smem[];
    u64* xr = reinterpret_cast<u64*>(smem);                                  // [STAGES][8][threads]
    uint4* wr = reinterpret_cast<uint4*>(smem + S::XWORDS * 8);             // [STAGES][MT][NB][32]
    int* s_src = reinterpret_cast<int*>(smem + S::XWORDS * 8 + STAGES * S::WCHUNKS * 16);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gq = lane >> 2, tq = lane & 3;
    const int limbs = level + 1;
    const long long poly_words = static_cast<long long>(limbs) * R.n;
    const long long cell_words = 2 * poly_words;
    const int nj = R.n / (WARPS * 8);
    const long long bid = blockIdx.x;
    const long long cb = bid / groups;  // pixel groups fastest
    const int p_begin = static_cast<int>(bid - cb * groups) * pg;
    const int p_end = SHORT ? min(p_begin + pg, g.pixels) : p_begin + 1;  // host: pg == 1 unless SHORT
    const int jb = static_cast<int>(cb % nj);
    const int row = static_cast<int>(cb / nj);  // comp * nl + li
    const int comp = row / nl, i = limb0 + row % nl;
    const int j0 = jb * (WARPS * 8) + warp * 8;
    const long long col_base = comp * poly_words + static_cast<long long>(i) * R.n + j0;
    const u64* xc = x + col_base + gq;  // this lane's B-operand column
    const u64 q = R.mod[i].q;
    const double qd = static_cast<double>(q), qinv = R.inv_q[i];
    const uint4* wbase = WIDE ? g.wfrag_wide : g.wfrag + static_cast<long long>(i) * g.oc_tiles * g.ksteps * 5 * 32;
    const bool staged = g.kpad <= KSRC;

    for (int p = p_begin; p < p_end; ++p) {
        const int* src_g = g.src + static_cast<long long>(p) * g.kpad;
        __syncthreads();  // previous pixel's readers are done with the tap table and rings
        if (staged)
            for (int t = tid; t < g.kpad; t += WARPS * 32) s_src[t] = src_g[t];
        __syncthreads();
        const int* src = staged ? s_src : src_g;

        for (int ot = 0; ot < g.oc_tiles; ot += MT) {
            u64 iacc[WIDE ? MT : 1][4];       // WIDE: canonical partial sums
            double facc[WIDE ? 1 : MT][4];    // else: centred FP64 partial sums
#pragma unroll
            for (int c = 0; c < 4; ++c) {
#pragma unroll
                for (int mt = 0; mt < (WIDE ? MT : 1); ++mt) iacc[mt][c] = 0;
#pragma unroll
                for (int mt = 0; mt < (WIDE ? 1 : MT); ++mt) facc[mt][c] = 0.0;
            }
            for (int ks0 = 0; ks0 < g.ksteps; ks0 += FOLD_STEPS) {
                const int ks1 = min(g.ksteps, ks0 + FOLD_STEPS);
                // copies of step ks into ring slot ks % STAGES: this thread's 8
                // gathered words (taps ks*32 + 4t + {0..3}, +16) and its share of
                // the CTA's weight fragments
                auto issue = [&](int ks) {
                    const int slot = ks % STAGES;
                    const int4 sa = *reinterpret_cast<const int4*>(src + ks * KSTEP + 4 * tq);
                    const int4 sb = *reinterpret_cast<const int4*>(src + ks * KSTEP + 16 + 4 * tq);
                    const int tp[8] = {sa.x, sa.y, sa.z, sa.w, sb.x, sb.y, sb.z, sb.w};
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        u64* dst = xr + (slot * 8 + u) * (WARPS * 32) + tid;
                        if (tp[u] >= 0) cp_async8(dst, xc + tp[u] * cell_words);
                        else *dst = 0;
                    }
                    for (int t = tid; t < S::WCHUNKS; t += WARPS * 32) {
                        const int mt = t / (NB * 32), rem = t - mt * (NB * 32);
                        const int b = rem >> 5, ln = rem & 31;
                        cp_async16(wr + slot * S::WCHUNKS + t,
                                   wbase + ((static_cast<long long>(ot + mt) * g.ksteps + ks) * NB + b) * 32 + ln);
                    }
                };
                int acc[NS][MT][4];
#pragma unroll
                for (int s = 0; s < NS; ++s)
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                        for (int c = 0; c < 4; ++c) acc[s][mt][c] = 0;
                __syncthreads();  // every warp is done with the rings before the prologue refills them
#pragma unroll
                for (int d = 0; d < STAGES - 1; ++d) {
                    if (ks0 + d < ks1) issue(ks0 + d);
                    cp_async_commit();
                }
                for (int ks = ks0; ks < ks1; ++ks) {
                    cp_async_wait<STAGES - 2>();  // step ks landed (this thread's copies) ...
                    __syncthreads();              // ... and everyone's; slot ks - 1 is free
                    if (ks + STAGES - 1 < ks1) issue(ks + STAGES - 1);
                    cp_async_commit();
                    const int slot = ks % STAGES;
                    u64 wa[4], wb[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        wa[u] = xr[(slot * 8 + u) * (WARPS * 32) + tid];
                        wb[u] = xr[(slot * 8 + 4 + u) * (WARPS * 32) + tid];
                    }
                    unsigned pa[NA], pb[NA];
                    byte_planes<NA>(wa, pa);
                    byte_planes<NA>(wb, pb);
                    const uint4* ws = wr + slot * S::WCHUNKS + lane;
#pragma unroll
                    for (int b = 0; b < NB; ++b) {
                        uint4 af[MT];
#pragma unroll
                        for (int mt = 0; mt < MT; ++mt) af[mt] = ws[(mt * NB + b) * 32];
#pragma unroll
                        for (int a = 0; a < NA; ++a)
#pragma unroll
                            for (int mt = 0; mt < MT; ++mt) {
                                if constexpr (WIDE) imma_s8(acc[a + b][mt], af[mt], pa[a], pb[a]);
                                else imma(acc[a + b][mt], af[mt], pa[a], pb[a]);
                            }
                    }
                }
                // fold the class sums into the residue accumulators
#pragma unroll
                for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        if constexpr (WIDE) {
                            // pairs: |D_s + 2^8 D_s+1| < 2^31 * 257 < 2^40 <= q
                            const ulonglong2* cs = g.shift_wide + i * 16;
                            u64 v = iacc[mt][c];
#pragma unroll
                            for (int s = 0; s < NS; s += 2) {
                                long long t = acc[s][mt][c];
                                if (s + 1 < NS) t += static_cast<long long>(acc[s + 1][mt][c]) * 256;
                                const u64 r = t >= 0 ? static_cast<u64>(t) : q - static_cast<u64>(-t);
                                const ulonglong2 k = __ldg(cs + s);
                                v = add_mod(v, mul_shoup(r, k.x, k.y, q), q);
                            }
                            iacc[mt][c] = v;
                        } else {
                            const double* cs = g.shift + i * 9;
                            auto D = [&](int s) { return static_cast<double>(acc[s][mt][c]); };
                            double v = facc[mt][c];
                            if constexpr (SHORT) {
                                // D_s < 5 * 255^2 * 1536 < 2^29: three classes per exact double (< 2^45)
                                v += ntt::fmodmul(D(0) + 256.0 * D(1) + 65536.0 * D(2), __ldg(cs + 0), qd, qinv);
                                v += ntt::fmodmul(D(3) + 256.0 * D(4) + 65536.0 * D(5), __ldg(cs + 3), qd, qinv);
                                v += ntt::fmodmul(D(6) + 256.0 * D(7) + 65536.0 * D(8), __ldg(cs + 6), qd, qinv);
                            } else {
#pragma unroll
                                for (int s = 0; s < 9; ++s) v += ntt::fmodmul(D(s), __ldg(cs + s), qd, qinv);
                            }
                            facc[mt][c] = ntt::fcentre(v, qd, qinv);
                        }
                    }
            }
            // C fragment: c0, c1 -> row g, cols 2t, 2t+1; c2, c3 -> row g + 8
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int oc = (ot + mt) * 16 + gq + (c >= 2 ? 8 : 0);
                    const int j = j0 + 2 * tq + (c & 1);
                    if (oc >= g.oc) continue;
                    u64 v;
                    if constexpr (WIDE) v = iacc[mt][c];
                    else v = ntt::fcanon(facc[mt][c], qd, qinv);
                    if (g.bias && comp == 0 && j == 0) v = add_mod(v, g.bias[static_cast<long long>(oc) * limbs + i], q);
                    y[(static_cast<long long>(p) * g.out_stride_pixel + oc) * cell_words + col_base - j0 + j] = v;
                }
        }
    }
}

// ---- short K (<= 8 steps): the barrier-free variant. Each thread streams its
// own gathered words through a private cp.async ring and the weight fragments
// come straight from L2; with 1-8 steps per output there is nothing to
// amortise CTA-wide staging against.
// occupancy knob for experiments: a minimum-blocks bound changes the register
// allocation even at 1 (the default leaves it to the compiler: 96-128 registers)
#ifdef HECNN_DIRECT_MINB
#define HECNN_DIRECT_LB __launch_bounds__(WARPS * 32, HECNN_DIRECT_MINB)
#else
#define HECNN_DIRECT_LB __launch_bounds__(WARPS * 32)
#endif
namespace direct {
constexpr int WARPS = 4;
constexpr int KSTEP = 32;
constexpr int FOLD_STEPS = 192;  // 6144 taps per exact int32 accumulation chunk

__device__ __forceinline__ void imma(int (&c)[4], const uint4& a, unsigned b0, unsigned b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void imma_s8(int (&c)[4], const uint4& a, unsigned b0, unsigned b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
}

// Gathered input words go through a STAGES-deep cp.async ring in shared
// memory, laid out [stage][word][thread] (conflict-free); every thread
// consumes only the words it copied itself, so cp.async.wait_group alone
// orders the pipeline (no CTA barrier).
constexpr int STAGES = 4;

struct XRing {
    u64* s;  // [STAGES][8][WARPS * 32]
    __device__ __forceinline__ u64* at(int stage, int u) const {
        return s + (stage * 8 + u) * (WARPS * 32) + threadIdx.x;
    }
};

__device__ __forceinline__ void cp_async8(u64* dst, const u64* src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Issue the copies of step ks (taps ks*32 + 4t + {0..3}, +16) into `stage`.
__device__ __forceinline__ void gather_step(const XRing& ring, int stage, const int* src, int ks, int tq,
                                            const u64* xc, long long cell_words) {
    const int4 sa = __ldg(reinterpret_cast<const int4*>(src + ks * KSTEP + 4 * tq));
    const int4 sb = __ldg(reinterpret_cast<const int4*>(src + ks * KSTEP + 16 + 4 * tq));
    const int t[8] = {sa.x, sa.y, sa.z, sa.w, sb.x, sb.y, sb.z, sb.w};
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        if (t[u] >= 0) cp_async8(ring.at(stage, u), xc + t[u] * cell_words);
        else *ring.at(stage, u) = 0;
    }
}

__device__ __forceinline__ void read_step(const XRing& ring, int stage, u64 (&wa)[4], u64 (&wb)[4]) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        wa[u] = *ring.at(stage, u);
        wb[u] = *ring.at(stage, 4 + u);
    }
}

// 4x4 byte transpose of four 32-bit words: p[a] = byte a of each word, word u in byte u.
__device__ __forceinline__ void transpose4(unsigned l0, unsigned l1, unsigned l2, unsigned l3, unsigned* p) {
    const unsigned x01 = __byte_perm(l0, l1, 0x5140), x01h = __byte_perm(l0, l1, 0x7362);
    const unsigned x23 = __byte_perm(l2, l3, 0x5140), x23h = __byte_perm(l2, l3, 0x7362);
    p[0] = __byte_perm(x01, x23, 0x5410);
    p[1] = __byte_perm(x01, x23, 0x7632);
    p[2] = __byte_perm(x01h, x23h, 0x5410);
    p[3] = __byte_perm(x01h, x23h, 0x7632);
}

// Byte planes of four words (taps k..k+3 of one column), the B-fragment
// order along K: NA = 5 for residues below 2^40, 8 for full words.
template <int NA>
__device__ __forceinline__ void byte_planes(const u64 (&w)[4], unsigned (&p)[NA]) {
    transpose4(static_cast<unsigned>(w[0]), static_cast<unsigned>(w[1]), static_cast<unsigned>(w[2]),
               static_cast<unsigned>(w[3]), p);
    const unsigned h0 = static_cast<unsigned>(w[0] >> 32), h1 = static_cast<unsigned>(w[1] >> 32);
    const unsigned h2 = static_cast<unsigned>(w[2] >> 32), h3 = static_cast<unsigned>(w[3] >> 32);
    if constexpr (NA == 8) {
        transpose4(h0, h1, h2, h3, p + 4);
    } else {
        static_assert(NA == 5, "5 or 8 byte planes");
        p[4] = __byte_perm(__byte_perm(h0, h1, 0x0040), __byte_perm(h2, h3, 0x0040), 0x5410);
    }
}

// SHORT: every accumulation chunk has <= 48 steps (three shift classes per
// exact double in the fold); otherwise classes are folded in pairs.
template <int MT, bool SHORT>
__global__ void HECNN_DIRECT_LB k_conv_imma_direct(DevRing R, ImmaMac g, const u64* __restrict__ x,
                                                         u64* __restrict__ y, int level, int limb0, int nl,
                                                         int groups, int pg) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gq = lane >> 2, tq = lane & 3;
    const int limbs = level + 1;
    const long long poly_words = static_cast<long long>(limbs) * R.n;
    const long long cell_words = 2 * poly_words;
    const int nj = R.n / (WARPS * 8);  // column blocks per (component, limb) row
    const long long bid = blockIdx.x;
    const long long cb = bid / groups;  // pixel groups fastest
    const int p_begin = static_cast<int>(bid - cb * groups) * pg;
    const int p_end = SHORT ? min(p_begin + pg, g.pixels) : p_begin + 1;  // host: pg == 1 unless SHORT
    const int jb = static_cast<int>(cb % nj);
    const int row = static_cast<int>(cb / nj);  // comp * nl + li
    const int comp = row / nl, i = limb0 + row % nl;
    const int j0 = jb * (WARPS * 8) + warp * 8;
    const long long col_base = comp * poly_words + static_cast<long long>(i) * R.n + j0;
    const u64* xc = x + col_base + gq;  // this lane's B-operand column
    const double qd = static_cast<double>(R.mod[i].q), qinv = R.inv_q[i];
    const u64 q = R.mod[i].q;
    const double* cs = g.shift + i * 9;  // 2^8s mod q, read at fold time
    const uint4* wf = g.wfrag + static_cast<long long>(i) * g.oc_tiles * g.ksteps * 5 * 32 + lane;
    __shared__ u64 s_ring[STAGES * 8 * WARPS * 32];
    const XRing ring{s_ring};

    for (int p = p_begin; p < p_end; ++p) {
    const int* src = g.src + static_cast<long long>(p) * g.kpad;
    for (int ot = 0; ot < g.oc_tiles; ot += MT) {
        double facc[MT][4];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int c = 0; c < 4; ++c) facc[mt][c] = 0.0;
        for (int ks0 = 0; ks0 < g.ksteps; ks0 += FOLD_STEPS) {
            const int ks1 = min(g.ksteps, ks0 + FOLD_STEPS);
            int acc[9][MT][4];
#pragma unroll
            for (int s = 0; s < 9; ++s)
#pragma unroll
                for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                    for (int c = 0; c < 4; ++c) acc[s][mt][c] = 0;
            // prologue: steps ks0 .. ks0 + STAGES - 2 in flight
#pragma unroll
            for (int d = 0; d < STAGES - 1; ++d) {
                if (ks0 + d < ks1) gather_step(ring, (ks0 + d) % STAGES, src, ks0 + d, tq, xc, cell_words);
                cp_async_commit();
            }
            for (int ks = ks0; ks < ks1; ++ks) {
                // B operand: taps ks*32 + 4t + {0..3} (reg 0) and +16 (reg 1) of column j0 + g
                if (ks + STAGES - 1 < ks1) gather_step(ring, (ks + STAGES - 1) % STAGES, src, ks + STAGES - 1, tq, xc, cell_words);
                cp_async_commit();
                cp_async_wait<STAGES - 1>();
                u64 wa[4], wb[4];
                read_step(ring, ks % STAGES, wa, wb);
                unsigned pa[5], pb[5];
                byte_planes<5>(wa, pa);
                byte_planes<5>(wb, pb);
#pragma unroll
                for (int b = 0; b < 5; ++b) {
                    uint4 af[MT];
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt)
                        af[mt] = __ldg(wf + ((static_cast<long long>(ot + mt) * g.ksteps + ks) * 5 + b) * 32);
#pragma unroll
                    for (int a = 0; a < 5; ++a)
#pragma unroll
                        for (int mt = 0; mt < MT; ++mt) imma(acc[a + b][mt], af[mt], pa[a], pb[a]);
                }
            }
            // fold: sum_s D_s (2^8s mod q), exact FP64 (|D_s| < 2^31, sums < 2^45)
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    double v = facc[mt][c];
                    auto D = [&](int s) { return static_cast<double>(acc[s][mt][c]); };
                    if constexpr (SHORT) {
                        // D_s < 5 * 255^2 * 1536 < 2^29: three classes per exact double (< 2^45)
                        v += ntt::fmodmul(D(0) + 256.0 * D(1) + 65536.0 * D(2), __ldg(cs + 0), qd, qinv);
                        v += ntt::fmodmul(D(3) + 256.0 * D(4) + 65536.0 * D(5), __ldg(cs + 3), qd, qinv);
                        v += ntt::fmodmul(D(6) + 256.0 * D(7) + 65536.0 * D(8), __ldg(cs + 6), qd, qinv);
                    } else {
#pragma unroll
                        for (int s = 0; s < 9; ++s) v += ntt::fmodmul(D(s), __ldg(cs + s), qd, qinv);
                    }
                    facc[mt][c] = ntt::fcentre(v, qd, qinv);
                }
        }
        // C fragment: c0, c1 -> row g, cols 2t, 2t+1; c2, c3 -> row g + 8
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int oc = (ot + mt) * 16 + gq + (c >= 2 ? 8 : 0);
                const int j = j0 + 2 * tq + (c & 1);
                if (oc >= g.oc) continue;
                u64 v = ntt::fcanon(facc[mt][c], qd, qinv);
                if (g.bias && comp == 0 && j == 0) v = add_mod(v, g.bias[static_cast<long long>(oc) * limbs + i], q);
                y[(static_cast<long long>(p) * g.out_stride_pixel + oc) * cell_words + col_base - j0 + j] = v;
            }
    }
    }  // pixel loop
}

// Limbs with q >= 2^40 (the 60-bit q0): the weights enter as the six
// balanced signed base-256 digits of the integer W = round(w * Delta) itself
// (identical for every limb, |W| < 2^47), the ciphertext words as eight
// unsigned bytes; 48 s8 x u8 products per tap in 13 shift classes, each an
// exact int32 sum (|D_s| <= 6 * 128 * 255 * 6144 < 2^31). The epilogue adds
// D_s (2^8s mod q) with 64-bit Shoup multiplies.
__global__ void HECNN_DIRECT_LB k_conv_imma_wide_direct(DevRing R, ImmaMac g, const u64* __restrict__ x,
                                                              u64* __restrict__ y, int level, int limb0, int nl,
                                                              int groups, int pg) {
    constexpr int NA = 8, NB = 6, NS = NA + NB - 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gq = lane >> 2, tq = lane & 3;
    const int limbs = level + 1;
    const long long poly_words = static_cast<long long>(limbs) * R.n;
    const long long cell_words = 2 * poly_words;
    const int nj = R.n / (WARPS * 8);
    const long long bid = blockIdx.x;
    const long long cb = bid / groups;  // pixel groups fastest
    const int p_begin = static_cast<int>(bid - cb * groups) * pg, p_end = min(p_begin + pg, g.pixels);
    const int jb = static_cast<int>(cb % nj);
    const int row = static_cast<int>(cb / nj);
    const int comp = row / nl, i = limb0 + row % nl;
    const int j0 = jb * (WARPS * 8) + warp * 8;
    const long long col_base = comp * poly_words + static_cast<long long>(i) * R.n + j0;
    const u64* xc = x + col_base + gq;
    const u64 q = R.mod[i].q;
    const ulonglong2* cs = g.shift_wide + i * 16;  // (2^8s mod q, shoup)
    const uint4* wf = g.wfrag_wide + lane;
    __shared__ u64 s_ring[STAGES * 8 * WARPS * 32];
    const XRing ring{s_ring};

    for (int p = p_begin; p < p_end; ++p) {
    const int* src = g.src + static_cast<long long>(p) * g.kpad;
    for (int ot = 0; ot < g.oc_tiles; ++ot) {
        u64 facc[4] = {0, 0, 0, 0};
        for (int ks0 = 0; ks0 < g.ksteps; ks0 += FOLD_STEPS) {
            const int ks1 = min(g.ksteps, ks0 + FOLD_STEPS);
            int acc[NS][4];
#pragma unroll
            for (int s = 0; s < NS; ++s)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[s][c] = 0;
#pragma unroll
            for (int d = 0; d < STAGES - 1; ++d) {
                if (ks0 + d < ks1) gather_step(ring, (ks0 + d) % STAGES, src, ks0 + d, tq, xc, cell_words);
                cp_async_commit();
            }
            for (int ks = ks0; ks < ks1; ++ks) {
                if (ks + STAGES - 1 < ks1) gather_step(ring, (ks + STAGES - 1) % STAGES, src, ks + STAGES - 1, tq, xc, cell_words);
                cp_async_commit();
                cp_async_wait<STAGES - 1>();
                u64 wa[4], wb[4];
                read_step(ring, ks % STAGES, wa, wb);
                unsigned pa[NA], pb[NA];
                byte_planes<NA>(wa, pa);
                byte_planes<NA>(wb, pb);
#pragma unroll
                for (int b = 0; b < NB; ++b) {
                    const uint4 af = __ldg(wf + ((static_cast<long long>(ot) * g.ksteps + ks) * NB + b) * 32);
#pragma unroll
                    for (int a = 0; a < NA; ++a) imma_s8(acc[a + b], af, pa[a], pb[a]);
                }
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                u64 v = facc[c];
                // classes in pairs: |D_s + 2^8 D_s+1| < 2^31 * 257 < 2^40 <= q, so one
                // conditional add of q makes the pair canonical
#pragma unroll
                for (int s = 0; s < NS; s += 2) {
                    long long t = acc[s][c];
                    if (s + 1 < NS) t += static_cast<long long>(acc[s + 1][c]) * 256;
                    const u64 r = t >= 0 ? static_cast<u64>(t) : q - static_cast<u64>(-t);
                    const ulonglong2 k = __ldg(cs + s);
                    v = add_mod(v, mul_shoup(r, k.x, k.y, q), q);
                }
                facc[c] = v;
            }
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int oc = ot * 16 + gq + (c >= 2 ? 8 : 0);
            const int j = j0 + 2 * tq + (c & 1);
            if (oc >= g.oc) continue;
            u64 v = facc[c];
            if (g.bias && comp == 0 && j == 0) v = add_mod(v, g.bias[static_cast<long long>(oc) * limbs + i], q);
            y[(static_cast<long long>(p) * g.out_stride_pixel + oc) * cell_words + col_base - j0 + j] = v;
        }
    }
    }  // pixel loop
}

}  // namespace direct

template <int MT, bool SHORT, bool WIDE>
void launch_imma(const DevRing& R, const ImmaMac& g, const u64* x, u64* y, int level, int limb0, int nl, int groups,
                 int pg, long long blocks, cudaStream_t st) {
    auto kern = k_conv_imma<MT, SHORT, WIDE>;
    constexpr int smem = ImmaShape<WIDE, MT>::SMEM;
    smem_opt_in(kern, smem);
    kern<<<static_cast<unsigned>(blocks), WARPS * 32, smem, st>>>(R, g, x, y, level, limb0, nl, groups, pg);
}

}  // namespace

bool imma_mac_supported(const DevRing& R, std::size_t K) {
    return R.n >= WARPS * 8 && K > 0 && K <= (1u << 20);
}

void imma_mac(const DevRing& R, const ImmaMac& g, const u64* x, u64* y, int level, int limb0, int limb1, bool wide,
              const Launch& L) {
    const int nl = limb1 - limb0;
    if (!g.pixels || !g.oc || nl <= 0) return;
    if (R.n < WARPS * 8) throw std::invalid_argument("imma_mac: ring degree below 32");
    const long long rows = 2LL * nl, nj = R.n / (WARPS * 8);
    const int pg = g.ksteps <= 4 ? 8 : 1;  // short K: a CTA runs a group of pixels
    const int groups = (g.pixels + pg - 1) / pg;
    const long long blocks = rows * nj * groups;
    if (blocks > 0x7fffffffLL) throw std::runtime_error("imma_mac: grid too large");
    const double cols = double(rows) * R.n;
    const bool short_k = g.ksteps <= 48;
    L.begin(wide ? "k_conv_imma_wide" : "k_conv_imma", double(g.pixels) * g.K * g.oc * cols,
            8.0 * cols * (double(g.pixels) * g.oc + double(g.pixels) * g.K));
    if (g.ksteps <= 8) {
        const dim3 grid(static_cast<unsigned>(blocks)), block(WARPS * 32);
        if (wide) direct::k_conv_imma_wide_direct<<<grid, block, 0, L.stream>>>(R, g, x, y, level, limb0, nl, groups, pg);
        else if (g.oc_tiles >= 2) direct::k_conv_imma_direct<2, true><<<grid, block, 0, L.stream>>>(R, g, x, y, level, limb0, nl, groups, pg);
        else direct::k_conv_imma_direct<1, true><<<grid, block, 0, L.stream>>>(R, g, x, y, level, limb0, nl, groups, pg);
    } else if (wide) {
        if (short_k) launch_imma<1, true, true>(R, g, x, y, level, limb0, nl, groups, pg, blocks, L.stream);
        else launch_imma<1, false, true>(R, g, x, y, level, limb0, nl, groups, pg, blocks, L.stream);
    } else if (g.oc_tiles >= 2) {
        if (short_k) launch_imma<2, true, false>(R, g, x, y, level, limb0, nl, groups, pg, blocks, L.stream);
        else launch_imma<2, false, false>(R, g, x, y, level, limb0, nl, groups, pg, blocks, L.stream);
    } else {
        if (short_k) launch_imma<1, true, false>(R, g, x, y, level, limb0, nl, groups, pg, blocks, L.stream);
        else launch_imma<1, false, false>(R, g, x, y, level, limb0, nl, groups, pg, blocks, L.stream);
    }
    L.count();
    check_launch(wide ? "imma_mac_wide" : "imma_mac");
}

}  // namespace hecnn_b200
