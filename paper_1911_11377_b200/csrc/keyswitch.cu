// Key switching (K5 + K6 in SURVEY.md §2.3): CkksEngine::key_switch,
// ckks.hpp:601-630.
//
// Step 1 (k_crt_digits): per coefficient of d2, exact CRT reconstruction
//   x = sum_i [a_i (Q/q_i)^-1]_{q_i} (Q/q_i) mod Q (reconstruct_mod_q,
//   ring.hpp:529-538) in multiword registers, the quotient by Q estimated
//   from sum_i w_i/q_i in double and corrected exactly, then the base-2^20
//   digits (BigUInt::bits, bigint.hpp:110-114) are written as u32 [D][n].
// Step 2 (k_keyswitch): one CTA per (ciphertext, limb i, block). For each
//   digit t it lifts digit_t into limb i (v < q_i, else v mod q_i:
//   ckks.hpp:622), runs the forward NTT in shared memory (same rounds and
//   swizzle as ntt.cu) and multiply-accumulates against evk_t (b_t, a_t)
//   (exact FP64 arithmetic for q < 2^42, Shoup for the 60-bit limb); the
//   accumulators stay on chip across all D digits (c0 in registers, c1 in
//   tensor memory), so neither the D lifted digit polynomials nor partial
//   sums ever touch HBM. The epilogue adds (d0, d1) in place. For N > 2^13 a CTA owns
//   a 2^13 block and recomputes the C = log2(N) - 13 column stages for its
//   block directly from the (L2-resident) u32 digits.

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <type_traits>

#include "ntt_core.cuh"

#pragma nv_diag_suppress 177  // KsShape constants unused by some instantiations

namespace hecnn_b200 {

namespace {

template <int W>
__global__ void __launch_bounds__(128) k_crt_digits(DevRing R, const u64* __restrict__ d2, u32* __restrict__ digits,
                                                  int level, int D, long long count) {
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= count * R.n) return;
    const long long ct = t / R.n;
    const int j = static_cast<int>(t % R.n);
    const int limbs = level + 1;
    const u64* a = d2 + ct * limbs * R.n + j;
    u64 acc[W];
#pragma unroll
    for (int w = 0; w < W; ++w) acc[w] = 0;
    double frac = 0.0;
    for (int i = 0; i < limbs; ++i) {
        const u64 q = R.mod[i].q;
        const ulonglong2 pinv = R.punct_inv[level * R.limbs + i];
        const u64 wi = mul_shoup(a[static_cast<long long>(i) * R.n], pinv.x, pinv.y, q);
        frac += static_cast<double>(wi) * R.inv_q[i];
        const u64* P = R.punct + (static_cast<long long>(level) * R.limbs + i) * R.crt_words;
        u64 carry = 0;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const u64 p = P[w];
            u64 lo = wi * p, hi = mulhi(wi, p);
            lo += carry;
            hi += lo < carry;
            acc[w] += lo;
            hi += acc[w] < lo;
            carry = hi;
        }
    }
    // subtract k*Q with k = floor(sum w_i/q_i) (exact up to one unit), then fix up
    const u64 k = static_cast<u64>(frac);
    const u64* Q = R.modulus + static_cast<long long>(level) * R.crt_words;
    {
        u64 carry = 0, borrow = 0;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const u64 p = Q[w];
            u64 lo = k * p, hi = mulhi(k, p);
            lo += carry;
            hi += lo < carry;
            carry = hi;
            const u64 before = acc[w];
            const u64 d = before - lo - borrow;
            borrow = (before < lo) || (before - lo < borrow) ? 1 : 0;
            acc[w] = d;
        }
        if (borrow) {  // went negative: add Q back
            u64 c = 0;
#pragma unroll
            for (int w = 0; w < W; ++w) {
                const u64 s = acc[w] + Q[w];
                const u64 c1 = s < acc[w];
                acc[w] = s + c;
                c = c1 | (acc[w] < s);
            }
        } else {  // at most one Q too many
            bool ge = true, decided = false;
#pragma unroll
            for (int w = W - 1; w >= 0; --w) {
                // lexicographic compare from the top word, first difference decides
                // (no early exit: a fully unrolled scan keeps acc[] in registers)
                const u64 qw = Q[w];
                if (!decided && acc[w] != qw) {
                    ge = acc[w] > qw;
                    decided = true;
                }
            }
            if (ge) {
                u64 b = 0;
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    const u64 before = acc[w];
                    acc[w] = before - Q[w] - b;
                    b = (before < Q[w]) || (before - Q[w] < b) ? 1 : 0;
                }
            }
        }
    }
    // digit layout for the key switch: [ct][D][B][E] with E = N / B column
    // partners (positions r + k B, k < E) adjacent, B = 2^min(logn, 13), so the
    // column stage of a block loads one vector per element (plain [D][N] when
    // N <= 2^13)
    const int lb = R.logn < 13 ? R.logn : 13, le = R.logn - lb;
    const int jj = ((j & ((1 << lb) - 1)) << le) | (j >> lb);
    u32* out = digits + ct * D * R.n + jj;
    // every digit position is a compile-time (word, shift) pair, so acc[]
    // stays in registers (a runtime word index sends it to local memory)
    constexpr int DMAX = (64 * W + 19) / 20;
#pragma unroll
    for (int d = 0; d < DMAX; ++d) {
        if (d >= D) break;
        const int off = 20 * d;
        const int wi = off >> 6, sh = off & 63;
        u64 v = acc[wi] >> sh;
        if (sh > 44 && wi + 1 < W) v |= acc[wi + 1] << (64 - sh);
        out[static_cast<long long>(d) * R.n] = static_cast<u32>(v & 0xFFFFFu);
    }
}

// The same digits through Garner's mixed radix: x = v_0 + q_0 (v_1 + q_1 (v_2 + ...))
// with v_i = ((a_i - v_0) q_0^-1 - v_1) q_1^-1 - ... mod q_i in [0, q_i): the
// O(l^2 / 2) mixed-radix digits run as exact FP64 modmuls (limbs 1..l, q_i < 2^42;
// the 60-bit v_0 enters as two 30-bit halves), then a Horner pass of l
// multiword-by-prime products on the integer pipes, whose length grows with
// the partial product -- half the 64-bit multiply-adds of the sum of
// Q/q_i multiples above, and no quotient estimate: x lands in [0, Q) exactly.
// Only chains whose 60-bit limb is limb 0 alone (the presets).
template <int W>
__global__ void __launch_bounds__(128) k_crt_digits_garner(DevRing R, const u64* __restrict__ d2,
                                                           u32* __restrict__ digits, int level, int D, long long count) {
    extern __shared__ u64 sv[];  // mixed-radix digits [limb][thread]
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= count * R.n) return;
    const long long ct = t / R.n;
    const int j = static_cast<int>(t % R.n);
    const int limbs = level + 1, T = blockDim.x, tid = threadIdx.x;
    const u64* a = d2 + ct * limbs * R.n + j;
    const u64 v0 = a[0];
    const double v0h = ntt::to_fp(v0 >> 30), v0l = ntt::to_fp(v0 & ((1ull << 30) - 1));
    // (a column order -- every t_i stepped once v_k is known, the t_i in shared
    // memory -- was measured slower: the extra shared-memory traffic outweighs the ILP)
    for (int i = 1; i < limbs; ++i) {
        const double q = static_cast<double>(R.mod[i].q), qinv = R.inv_q[i];
        const double* gi = R.garner_inv + i * R.limbs;
        double v = ntt::to_fp(a[static_cast<long long>(i) * R.n]) - (ntt::fmodmul(v0h, R.garner_c30[i], q, qinv) + v0l);
        v = ntt::fmodmul(v, gi[0], q, qinv);
        for (int k = 1; k < i; ++k) v = ntt::fmodmul(v - ntt::to_fp(sv[k * T + tid]), gi[k], q, qinv);
        sv[i * T + tid] = ntt::fcanon(v, q, qinv);
    }
    u64 acc[W];
#pragma unroll
    for (int w = 0; w < W; ++w) acc[w] = 0;
    acc[0] = level ? sv[level * T + tid] : v0;
    int nw = 1;
    for (int i = level - 1; i >= 0; --i) {
        const u64 qi = R.mod[i].q;
        u64 carry = i ? sv[i * T + tid] : v0;
        bool grow = false;
        // compile-time word indices only (a runtime acc[nw] would put acc[] in local memory)
#pragma unroll
        for (int w = 0; w < W; ++w) {
            if (w < nw) {
                u64 lo = acc[w] * qi, hi = mulhi(acc[w], qi);
                lo += carry;
                hi += lo < carry;
                acc[w] = lo;
                carry = hi;
            } else if (w == nw) {
                acc[w] = carry;
                grow = carry != 0;
            }
        }
        nw += grow;
    }
    const int lb = R.logn < 13 ? R.logn : 13, le = R.logn - lb;
    const int jj = ((j & ((1 << lb) - 1)) << le) | (j >> lb);
    u32* out = digits + ct * D * R.n + jj;
    constexpr int DMAX = (64 * W + 19) / 20;
#pragma unroll
    for (int d = 0; d < DMAX; ++d) {
        if (d >= D) break;
        const int off = 20 * d;
        const int wi = off >> 6, sh = off & 63;
        u64 v = acc[wi] >> sh;
        if (sh > 44 && wi + 1 < W) v |= acc[wi + 1] << (64 - sh);
        out[static_cast<long long>(d) * R.n] = static_cast<u32>(v & 0xFFFFFu);
    }
}

__device__ __forceinline__ u64 lift_digit(u32 v, u64 q) { return v < q ? v : v % q; }

// ---- tensor memory / bulk-copy helpers: ks_saddr / ks_mbar_wait / ks_bulk_load (ntt_core.cuh)
// EL doubles of this thread's TMEM lane at column `col` (2 x 32-bit columns each)
template <int EL>
__device__ __forceinline__ void tmem_ld_d(uint32_t addr, double (&v)[EL]) {
    static_assert(EL == 4, "4-word units");
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int k = 0; k < EL; ++k) v[k] = __hiloint2double(static_cast<int>(r[2 * k + 1]), static_cast<int>(r[2 * k]));
}
template <int EL>
__device__ __forceinline__ void tmem_ld_u(uint32_t addr, u64 (&v)[EL]) {
    static_assert(EL == 4, "4-word units");
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int k = 0; k < EL; ++k) v[k] = (static_cast<u64>(r[2 * k + 1]) << 32) | r[2 * k];
}
template <int EL>
__device__ __forceinline__ void tmem_st_u(uint32_t addr, const u64 (&v)[EL]) {
    static_assert(EL == 4, "4-word units");
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(addr),
                 "r"(static_cast<uint32_t>(v[0])), "r"(static_cast<uint32_t>(v[0] >> 32)), "r"(static_cast<uint32_t>(v[1])),
                 "r"(static_cast<uint32_t>(v[1] >> 32)), "r"(static_cast<uint32_t>(v[2])), "r"(static_cast<uint32_t>(v[2] >> 32)),
                 "r"(static_cast<uint32_t>(v[3])), "r"(static_cast<uint32_t>(v[3] >> 32))
                 : "memory");
}
template <int EL>
__device__ __forceinline__ void tmem_st_d(uint32_t addr, const double (&v)[EL]) {
    static_assert(EL == 4, "4-word units");
    uint32_t r[8];
#pragma unroll
    for (int k = 0; k < EL; ++k) {
        r[2 * k] = static_cast<uint32_t>(__double2loint(v[k]));
        r[2 * k + 1] = static_cast<uint32_t>(__double2hiint(v[k]));
    }
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(addr), "r"(r[0]), "r"(r[1]),
                 "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}

// Value at block-local position r after the C column stages (block b): only
// the butterflies on the path to output b are evaluated (2^C - 1 products).
// E column partners of block position r, adjacent in the digit layout
// (k_crt_digits): one 4 / 8 / 16-byte load
template <int E>
__device__ __forceinline__ void load_partners(const u32* __restrict__ dig, int r, u32 (&v)[E]) {
    if constexpr (E == 1) {
        v[0] = __ldg(dig + r);
    } else if constexpr (E == 2) {
        const uint2 w = __ldg(reinterpret_cast<const uint2*>(dig) + r);
        v[0] = w.x, v[1] = w.y;
    } else if constexpr (E == 4) {
        const uint4 w = __ldg(reinterpret_cast<const uint4*>(dig) + r);
        v[0] = w.x, v[1] = w.y, v[2] = w.z, v[3] = w.w;
    } else {
#pragma unroll
        for (int k = 0; k < E; k += 4) {
            const uint4 w = __ldg(reinterpret_cast<const uint4*>(dig + r * E + k));
            v[k] = w.x, v[k + 1] = w.y, v[k + 2] = w.z, v[k + 3] = w.w;
        }
    }
}

template <int LOGN, int C>
__device__ __forceinline__ u64 column_value(const u32* __restrict__ dig, const ulonglong2* __restrict__ tw, u64 q, int r,
                                            int b) {
    if constexpr (C == 0) {
        return lift_digit(dig[r], q);
    } else {
        constexpr int E = 1 << C;
        const u64 two_q = q << 1;
        u64 x[E];
        u32 raw[E];
        load_partners<E>(dig, r, raw);
#pragma unroll
        for (int k = 0; k < E; ++k) x[k] = lift_digit(raw[k], q);
#pragma unroll
        for (int rho = 0; rho < C; ++rho) {
            const int half = E >> (rho + 1);
#pragma unroll
            for (int blk = 0; blk < (1 << rho); ++blk) {
                const ulonglong2 w = tw[(1 << rho) + blk];
#pragma unroll
                for (int kk = 0; kk < half; ++kk) ntt::ct_butterfly(x[blk * 2 * half + kk], x[blk * 2 * half + kk + half], w, q, two_q);
            }
        }
        u64 v = x[0];
#pragma unroll
        for (int k = 1; k < E; ++k)
            if (k == b) v = x[k];
        return v;
    }
}

// The same column stages on the FP64 pipe (limbs with q < 2^42): values stay
// below (C + 1) q < 2^45 in magnitude, so fmodmul stays exact without
// corrections; the block's first round continues from these doubles.
template <int LOGN, int C, bool LIFT>
__device__ __forceinline__ double column_value_fp(const u32* __restrict__ dig, const double* __restrict__ tw, u64 q,
                                                  double qd, double qinv, int r, int b) {
    constexpr int E = 1 << C;
    double x[E];
    u32 raw[E];
    load_partners<E>(dig, r, raw);
#pragma unroll
    for (int k = 0; k < E; ++k) x[k] = ntt::to_fp(LIFT ? lift_digit(raw[k], q) : raw[k]);
#pragma unroll
    for (int rho = 0; rho < C; ++rho) {
        const int half = E >> (rho + 1);
#pragma unroll
        for (int blk = 0; blk < (1 << rho); ++blk) {
            const double w = tw[(1 << rho) + blk];
#pragma unroll
            for (int kk = 0; kk < half; ++kk) {
                double& a = x[blk * 2 * half + kk];
                double& c = x[blk * 2 * half + kk + half];
                const double v = ntt::fmodmul(c, w, qd, qinv);
                const double u = a;
                a = u + v;
                c = u - v;
            }
        }
    }
    double v = x[0];
#pragma unroll
    for (int k = 1; k < E; ++k)
        if (k == b) v = x[k];
    return v;
}

// Per digit t: lift -> forward NTT (shared rounds) -> in the last butterfly
// round each thread multiplies its outputs by (b_t, a_t) and accumulates;
// accumulator positions are the thread's last-round positions, identical for
// every t. The last round's units are EL consecutive words (its stride is 1),
// so the MAC runs once per unit with 16-byte evk loads (KeyAt::unit) instead
// of one 8-byte load per word. A = IntArith (u64 Shoup, evk + evk_sh) or
// FpArith (exact FP64, evk_f = e as doubles). The block's twiddles sit in
// shared memory as a block-local table TL[2^s + m] = tw[2^(s+C) + b 2^s + m]
// (precomputed per (limb, block) in DevRing::ks_tw / ks_tw_f and bulk-copied
// when a CTA moves to another limb or block) and are reused by all D digit
// transforms (round code indexes it with b = c = 0).
// FP64 path (all limbs but the 60-bit q0): the c1 accumulator lives in tensor
// memory (TM below; without it, in a thread-private [slot][thread] shared-
// memory layout), the shared memory the integer path needs for its 16-byte
// twiddles holds the digit's b_t slice, and the registers the accumulator
// frees hold the next digit's first-round inputs, loaded while the current
// digit is transformed.
// LIFT: some prime of the chain is <= 2^20, so digits need v mod q_i
// (ckks.hpp:622); otherwise every digit is already a residue.
//
// The kernel is persistent: a CTA keeps its tensor-memory allocation and
// mbarriers and walks work items (ciphertext, limb, block) with a grid
// stride, so one item's epilogue overlaps the next item's first round on
// other warps and the per-CTA setup is paid once.
template <int LOGN, int LOGB, int LOGE, int T, bool FP, bool AUXK = false>
struct KsShape {
    static constexpr int B = 1 << LOGB, C = LOGN - LOGB;
    static constexpr int SL = ntt::last_round_start(LOGB, LOGE);
    static constexpr int RL = LOGB - SL, EL = 1 << RL, UL = B >> RL, PL = (UL + T - 1) / T;
    // c1 accumulator slots: thread-private [slot][thread] when every thread
    // owns PL whole units (fits the B-word region), else at swizzled positions
    static constexpr bool PRIV = UL % T == 0;
#ifndef HECNN_KS_TMEM
#define HECNN_KS_TMEM 1
#endif
    // TM: the c1 accumulators live in tensor memory (thread-private lane
    // columns, tcgen05.ld/st) and the shared-memory region they used holds
    // the digit's b_t slice, bulk-copied in while the previous digit's
    // transform runs; a_t streams from L2
    static constexpr bool TM = FP && PRIV && HECNN_KS_TMEM && EL == 4;
    // TMI: the integer (60-bit limb) path keeps its c1 accumulators in tensor
    // memory as well (its 16-byte Shoup twiddles leave no shared memory to stage evk)
    static constexpr bool TMI = !FP && PRIV && HECNN_KS_TMEM && EL == 4;
    static constexpr bool USE_TMEM = TM || TMI;
    // tensor-memory columns per thread: c1, plus (AUXK) limb 0's two
    // accumulators mod q_s in the aux limbs 1..3
    static constexpr int TCW = (AUXK ? 6 : 2) * PL * EL;
    static constexpr int TNEED = (T / 128) * TCW;
    static constexpr int TCOLS = TNEED <= 32 ? 32 : (TNEED <= 64 ? 64 : (TNEED <= 128 ? 128 : (TNEED <= 256 ? 256 : 512)));
    static_assert(!USE_TMEM || TNEED <= 512, "key switch: tensor-memory accumulators exceed the 512 TMEM columns");
    static_assert(EL % 2 == 0, "last round units must hold an even number of words");
    static_assert(!ntt::Split<LOGB, LOGE, T>::on || UL % T == 0, "split blocks own whole last-round units");
    // first round (S0 = 0): unit u owns positions u + k * STR0, k < E0
    static constexpr int R0 = ntt::round_size(LOGB, LOGE, 0), E0 = 1 << R0, U0 = B >> R0, P0 = (U0 + T - 1) / T;
    static constexpr int STR0 = U0;
    // FP64 path, N <= 2^LOGB: the next digit's first-round inputs are loaded
    // into registers while the current digit is transformed
    static constexpr bool PREFETCH = FP && C == 0;
};

// Shared-memory map (dynamic): data [B] words | twiddle table [B] TW | FP:
// c1 accumulators or b_t stage [B] doubles | 2 mbarriers (b_t, twiddles).
template <int LOGN, int LOGB, int LOGE, int T, bool LIFT, bool AUXK, class A, class KeyAt>
__device__ __forceinline__ void ks_item(const DevRing& R, const A& ar, const typename A::TW* tw_block,
                                        bool load_tw, const u32* digits, KeyAt key, u64* acc01, int level, int D,
                                        long long ct, int i, int b, u64 q, int mode, const u64* fy, uint32_t tm_lane,
                                        unsigned& bphase, unsigned& tphase, int aux_slot, const double* aux_tab,
                                        u64* aux_out) {
    using V = typename A::V;
    using TW = typename A::TW;
    constexpr bool FP = std::is_same<V, double>::value;
    using S = KsShape<LOGN, LOGB, LOGE, T, FP, AUXK>;
    constexpr int B = S::B, C = S::C, EL = S::EL, PL = S::PL, UL = S::UL, E0 = S::E0, U0 = S::U0, P0 = S::P0;
    constexpr int STR0 = S::STR0;
    constexpr bool PRIV = S::PRIV, TM = S::TM, TMI = S::TMI, USE_TMEM = S::USE_TMEM, PREFETCH = S::PREFETCH;
    extern __shared__ u64 smem[];
    const long long n = 1LL << LOGN;
    const long long blk_off = static_cast<long long>(b) << LOGB;
    const ulonglong2* itw = R.fwd + (static_cast<long long>(i) << LOGN);  // integer twiddles for the column stages
    TW* stw = reinterpret_cast<TW*>(smem + B);
    double* sacc = reinterpret_cast<double*>(smem + 2 * B);  // FP path: c1 accumulators (TM: b_t staging)
    uint64_t* bbar = reinterpret_cast<uint64_t*>(smem + 3 * B);
    uint64_t* tbar = bbar + 1;

    // the previous item's rounds are over (barrier after its last digit):
    // shared memory may be refilled
    if (threadIdx.x == 0) {
        if (load_tw) ntt::bulk_load(stw, tw_block, B * sizeof(TW), tbar);
        if constexpr (TM) ntt::bulk_load(sacc, key.evk_f + key.ioff + blk_off, B * 8, bbar);  // b_0 of this block
    }
    if constexpr (USE_TMEM) {
        const u64 z[EL] = {};
#pragma unroll
        for (int uu = 0; uu < S::TCW / (2 * EL); ++uu) tmem_st_u<EL>(tm_lane + uu * 2 * EL, z);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    auto slot = [&](int idx, int uu, int k) -> int {
        if constexpr (PRIV) { (void)idx; return (uu * EL + k) * T + threadIdx.x; }
        else { (void)uu; (void)k; return ntt::swz(idx); }
    };
    if constexpr (FP && !TM) {
        for (int j = threadIdx.x; j < B; j += T) sacc[j] = 0.0;
    }

    V a0[PL * EL], a1[(FP || TMI) ? 1 : PL * EL];
#pragma unroll
    for (int k = 0; k < PL * EL; ++k) a0[k] = V(0);
#pragma unroll
    for (int k = 0; k < ((FP || TMI) ? 1 : PL * EL); ++k) a1[k] = V(0);

    u32 pf[PREFETCH ? P0 * E0 : 1];
    auto prefetch = [&](int t) {
        if constexpr (PREFETCH) {
            const u32* dig = digits + (ct * D + t) * n;
#pragma unroll
            for (int uu = 0; uu < P0; ++uu) {
                const int u = threadIdx.x + uu * T;
#pragma unroll
                for (int k = 0; k < E0; ++k) pf[uu * E0 + k] = (U0 % T != 0 && u >= U0) ? 0u : __ldg(dig + u + k * STR0);
            }
        }
    };
    prefetch(0);
    if (load_tw) {
        ntt::mbar_wait(tbar, tphase & 1);  // twiddle table landed
        ++tphase;
    }
    if constexpr (!TM) __syncthreads();  // zeroed c1 slots before any thread accumulates

    auto lift = [&](u32 v) -> u64 {
        if constexpr (LIFT) return lift_digit(v, q);
        else return v;
    };
    for (int t = 0; t < D; ++t) {
        const u32* dig = digits + (ct * D + t) * n;
        auto first = [&](int r, int uu, int k) -> V {
            if constexpr (PREFETCH) {
                (void)r;
                return ntt::to_fp(lift(pf[uu * E0 + k]));
            } else if constexpr (FP) {
                (void)uu, (void)k;
                return column_value_fp<LOGN, C, LIFT>(dig, R.fwd_f + (static_cast<long long>(i) << LOGN), q, ar.q, ar.qinv, r, b);
            } else {
                (void)uu, (void)k;
                return column_value<LOGN, C>(dig, itw, q, r, b);
            }
        };
        V stash[EL];
        const unsigned par = bphase & 1;
        ntt::fwd_block<LOGB, LOGE, T>(reinterpret_cast<V*>(smem), ar, stw, 0, 0, first,
                                      [&](int idx, V v, int uu, int k) {
                                          stash[k] = v;
                                          if (k == EL - 1) {
                                              const int base = idx - (EL - 1);
                                              if constexpr (TM) {
                                                  ntt::mbar_wait(bbar, par);  // b_t landed
                                                  if (AUXK && aux_slot >= 0)
                                                      key.template unit_tm_aux<EL>(
                                                          t, blk_off + base, stash, a0 + uu * EL, sacc + base,
                                                          tm_lane + uu * 2 * EL, tm_lane + (2 * PL + 4 * uu) * EL,
                                                          aux_tab + (8LL * t + aux_slot) * n,       // [t][b][slot]
                                                          aux_tab + (8LL * t + 4 + aux_slot) * n);  // [t][a][slot]
                                                  else
                                                      key.template unit_tm<EL>(t, blk_off + base, stash, a0 + uu * EL,
                                                                               sacc + base, tm_lane + uu * 2 * EL);
                                              } else if constexpr (FP) {
                                                  key.template unit<EL>(t, blk_off + base, stash, a0 + uu * EL,
                                                                        [&](int kk) -> double& { return sacc[slot(base + kk, uu, kk)]; });
                                              } else if constexpr (TMI) {
                                                  key.template unit_tm<EL>(t, blk_off + base, stash, a0 + uu * EL, tm_lane + uu * 2 * EL);
                                              } else {
                                                  key.template unit<EL>(t, blk_off + base, stash, a0 + uu * EL,
                                                                        [&](int kk) -> u64& { return a1[uu * EL + kk]; });
                                              }
                                          }
                                      },
                                      [&] {
                                          // the first round has consumed pf: the next digit's
                                          // inputs land while this one is transformed
                                          if (t + 1 < D) prefetch(t + 1);
                                      });
        if constexpr (TM) ++bphase;
        if constexpr (USE_TMEM) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        __syncthreads();  // the next digit's first round overwrites shared memory
        if constexpr (TM) {
            if (threadIdx.x == 0 && t + 1 < D)
                ntt::bulk_load(sacc, key.evk_f + (2LL * (t + 1)) * key.key_stride + key.ioff + blk_off, B * 8, bbar);
        }
    }
    const int limbs = level + 1;
    u64* o0 = acc01 + ((ct * 2) * limbs + i) * n + blk_off;
    u64* o1 = o0 + static_cast<long long>(limbs) * n;
    const u64* y0 = fy ? fy + ((ct * 2) * limbs + i) * n + blk_off : nullptr;
    const u64* y1 = fy ? y0 + static_cast<long long>(limbs) * n : nullptr;
    const ModConst mc = R.mod[i];
    // the tensor product's (d0, d1) from the forward-transformed operands
    // (ckks.hpp:320-327), formed at the positions this thread writes
    auto mulq = [&](u64 a, u64 c) -> u64 {
        if constexpr (FP) return ntt::fcanon(ntt::fmodmul(ntt::to_fp(a), ntt::to_fp(c), ar.q, ar.qinv), ar.q, ar.qinv);
        else return mul_mod(a, c, mc);
    };
    // each unit's EL words are contiguous: 16-byte loads and stores. With
    // whole units per thread, every unit's (x0, x1) words are loaded before
    // the first is used (their HBM latency overlaps instead of serialising)
    constexpr bool EPF = FP && PRIV && T <= 512;  // 1024-thread blocks (64 registers) and the integer path spill with it
    ulonglong2 xpre[EPF ? PL * EL : 1];
    if constexpr (EPF) {
#pragma unroll
        for (int uu = 0; uu < PL; ++uu) {
            const int base = ntt::fwd_last_base<LOGB, LOGE, T>(uu);
#pragma unroll
            for (int k = 0; k < EL; k += 2) {
                xpre[uu * EL + k] = *reinterpret_cast<const ulonglong2*>(o0 + base + k);
                xpre[uu * EL + k + 1] = *reinterpret_cast<const ulonglong2*>(o1 + base + k);
            }
        }
    }
#pragma unroll
    for (int uu = 0; uu < PL; ++uu) {
        const int u = threadIdx.x + uu * T;
        if (UL % T != 0 && u >= UL) break;
        const int base = ntt::fwd_last_base<LOGB, LOGE, T>(uu);
        double c1u[EL];
        u64 c1i[EL];
        if constexpr (TMI) tmem_ld_u<EL>(tm_lane + uu * 2 * EL, c1i);
        if constexpr (TM) tmem_ld_d<EL>(tm_lane + uu * 2 * EL, c1u);
#pragma unroll
        for (int k = 0; k < EL; k += 2) {
            const int idx = base + k;
            u64 r0[2], r1[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if constexpr (FP) {
                    r0[h] = ntt::fcanon(a0[uu * EL + k + h], ar.q, ar.qinv);
                    if constexpr (TM) r1[h] = ntt::fcanon(c1u[k + h], ar.q, ar.qinv);
                    else r1[h] = ntt::fcanon(sacc[slot(idx + h, uu, k + h)], ar.q, ar.qinv);
                } else {
                    r0[h] = reduce_2q(a0[uu * EL + k + h], q);
                    if constexpr (TMI) r1[h] = reduce_2q(c1i[k + h], q);
                    else r1[h] = reduce_2q(a1[uu * EL + k + h], q);
                }
            }
            const ulonglong2 x0 = EPF ? xpre[uu * EL + k] : *reinterpret_cast<const ulonglong2*>(o0 + idx);
            const ulonglong2 x1 = EPF ? xpre[uu * EL + k + 1] : *reinterpret_cast<const ulonglong2*>(o1 + idx);
            u64 b0[2], b1[2];
            const u64 xa[2] = {x0.x, x0.y}, xb[2] = {x1.x, x1.y};
            if (mode == 0) {  // acc01 already holds (d0, d1)
#pragma unroll
                for (int h = 0; h < 2; ++h) b0[h] = xa[h], b1[h] = xb[h];
            } else if (mode == 1) {  // acc01 holds NTT(x): d = x^2
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    b0[h] = mulq(xa[h], xa[h]);
                    const u64 c = mulq(xa[h], xb[h]);
                    b1[h] = add_mod(c, c, q);
                }
            } else {  // d = x * y
                const ulonglong2 v0 = *reinterpret_cast<const ulonglong2*>(y0 + idx);
                const ulonglong2 v1 = *reinterpret_cast<const ulonglong2*>(y1 + idx);
                const u64 va[2] = {v0.x, v0.y}, vb[2] = {v1.x, v1.y};
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    b0[h] = mulq(xa[h], va[h]);
                    b1[h] = add_mod(mulq(xa[h], vb[h]), mulq(xb[h], va[h]), q);
                }
            }
            *reinterpret_cast<ulonglong2*>(o0 + idx) = make_ulonglong2(add_mod(b0[0], r0[0], q), add_mod(b0[1], r0[1], q));
            *reinterpret_cast<ulonglong2*>(o1 + idx) = make_ulonglong2(add_mod(b1[0], r1[0], q), add_mod(b1[1], r1[1], q));
        }
    }
    if constexpr (AUXK && TM && C == 0) {
        if (aux_slot >= 0) {
            // limb 0's accumulators mod q_s, inverse-transformed in this CTA (the
            // whole polynomial is its block): coefficients of E mod q_s straight to
            // aux_out [ct][comp][4][n] slot s
            double* sd = reinterpret_cast<double*>(smem);
            const double ni = R.n_inv_f[i];
            for (int comp = 0; comp < 2; ++comp) {
                __syncthreads();  // the data region is free (digit loop / previous transform done)
#pragma unroll
                for (int uu = 0; uu < PL; ++uu) {
                    const int base = ntt::fwd_last_base<LOGB, LOGE, T>(uu);
                    double e[EL];
                    tmem_ld_d<EL>(tm_lane + (2 * PL + 4 * uu + 2 * comp) * EL, e);
#pragma unroll
                    for (int k = 0; k < EL; ++k) sd[ntt::swz(base + k)] = ntt::fcentre(e[k], ar.q, ar.qinv);
                }
                __syncthreads();
                u64* z = aux_out + ((ct * 2 + comp) * 4 + aux_slot) * n;
                const ntt::FpArith far{ar.q, ar.qinv};
                ntt::inv_block<LOGB, LOGE, T>(
                    sd, far, R.inv_f + (static_cast<long long>(i) << LOGN), 0, 0,
                    [=](int idx) { return sd[ntt::swz(idx)]; },
                    [=](int idx, double v, int, int) { z[idx] = ntt::fcanon(ntt::fmodmul(v, ni, far.q, far.qinv), far.q, far.qinv); });
            }
        }
    } else if constexpr (AUXK && TM) {
        if (aux_slot >= 0) {
            // limb 0's accumulators mod q_s (NTT domain of limb s) -> aux_out
            // [ct][comp][4][n] slot s; ntt_inverse_limbs + k_aux_crt take them from there
#pragma unroll
            for (int uu = 0; uu < PL; ++uu) {
                const int base = ntt::fwd_last_base<LOGB, LOGE, T>(uu);
                double e0[EL], e1[EL];
                tmem_ld_d<EL>(tm_lane + (2 * PL + 4 * uu) * EL, e0);
                tmem_ld_d<EL>(tm_lane + (2 * PL + 4 * uu + 2) * EL, e1);
                u64* z0 = aux_out + ((ct * 2) * 4 + aux_slot) * n + blk_off + base;
                u64* z1 = aux_out + ((ct * 2 + 1) * 4 + aux_slot) * n + blk_off + base;
#pragma unroll
                for (int k = 0; k < EL; k += 2) {
                    *reinterpret_cast<ulonglong2*>(z0 + k) =
                        make_ulonglong2(ntt::fcanon(e0[k], ar.q, ar.qinv), ntt::fcanon(e0[k + 1], ar.q, ar.qinv));
                    *reinterpret_cast<ulonglong2*>(z1 + k) =
                        make_ulonglong2(ntt::fcanon(e1[k], ar.q, ar.qinv), ntt::fcanon(e1[k + 1], ar.q, ar.qinv));
                }
            }
        }
    }
    if constexpr (!USE_TMEM && FP) __syncthreads();  // c1 slots are re-zeroed by the next item
}

// Unit-wise evk MACs: EL consecutive NTT outputs v[] at key positions
// pos..pos+EL-1 of digit t, 16-byte loads of the key words.
struct FpKey {
    const double* evk_f;
    long long key_stride, ioff;
    double q, qinv;
    template <int EL, class S1>
    __device__ __forceinline__ void unit(int t, long long pos, const double* v, double* s0, S1 s1) const {
        const double2* kb = reinterpret_cast<const double2*>(evk_f + (2LL * t) * key_stride + ioff + pos);
        const double2* ka = reinterpret_cast<const double2*>(evk_f + (2LL * t + 1) * key_stride + ioff + pos);
        double2 wb[EL / 2], wa[EL / 2];
#pragma unroll
        for (int k = 0; k < EL / 2; ++k) wb[k] = __ldg(kb + k), wa[k] = __ldg(ka + k);
#pragma unroll
        for (int k = 0; k < EL / 2; ++k) {
            // |s| < D q < 2^48: exact sums
            s0[2 * k] += ntt::fmodmul(v[2 * k], wb[k].x, q, qinv);
            s0[2 * k + 1] += ntt::fmodmul(v[2 * k + 1], wb[k].y, q, qinv);
            s1(2 * k) += ntt::fmodmul(v[2 * k], wa[k].x, q, qinv);
            s1(2 * k + 1) += ntt::fmodmul(v[2 * k + 1], wa[k].y, q, qinv);
        }
    }
    // unit_tm plus limb 0's key switch mod q_s (aux): e0 += v * Tb, e1 += v * Ta
    // with Tb / Ta = NTT_{q_s}(INTT_{q0}(b_t / a_t of limb 0)), in two more
    // tensor-memory column groups
    template <int EL>
    __device__ __forceinline__ void unit_tm_aux(int t, long long pos, const double* v, double* s0, const double* bst,
                                                uint32_t tcol, uint32_t acol, const double* aux_b,
                                                const double* aux_a) const {
        unit_tm<EL>(t, pos, v, s0, bst, tcol);
        const double2* xb = reinterpret_cast<const double2*>(aux_b + pos);
        const double2* xa = reinterpret_cast<const double2*>(aux_a + pos);
        double2 wb[EL / 2], wa[EL / 2];
#pragma unroll
        for (int k = 0; k < EL / 2; ++k) wb[k] = __ldg(xb + k), wa[k] = __ldg(xa + k);
        double e0[EL], e1[EL];
        tmem_ld_d<EL>(acol, e0);
        tmem_ld_d<EL>(acol + 2 * EL, e1);
#pragma unroll
        for (int k = 0; k < EL / 2; ++k) {
            e0[2 * k] += ntt::fmodmul(v[2 * k], wb[k].x, q, qinv);
            e0[2 * k + 1] += ntt::fmodmul(v[2 * k + 1], wb[k].y, q, qinv);
            e1[2 * k] += ntt::fmodmul(v[2 * k], wa[k].x, q, qinv);
            e1[2 * k + 1] += ntt::fmodmul(v[2 * k + 1], wa[k].y, q, qinv);
        }
        tmem_st_d<EL>(acol, e0);
        tmem_st_d<EL>(acol + 2 * EL, e1);
    }
    // b_t from the shared-memory stage, a_t from L2, c1 read-modify-written in
    // this thread's tensor-memory columns
    template <int EL>
    __device__ __forceinline__ void unit_tm(int t, long long pos, const double* v, double* s0, const double* bst,
                                            uint32_t tcol) const {
        const double2* ka = reinterpret_cast<const double2*>(evk_f + (2LL * t + 1) * key_stride + ioff + pos);
        double2 wa[EL / 2];
#pragma unroll
        for (int k = 0; k < EL / 2; ++k) wa[k] = __ldg(ka + k);
        const double2* kb = reinterpret_cast<const double2*>(bst);
#pragma unroll
        for (int k = 0; k < EL / 2; ++k) {
            const double2 wb = kb[k];
            s0[2 * k] += ntt::fmodmul(v[2 * k], wb.x, q, qinv);
            s0[2 * k + 1] += ntt::fmodmul(v[2 * k + 1], wb.y, q, qinv);
        }
        double c1[EL];
        tmem_ld_d<EL>(tcol, c1);
#pragma unroll
        for (int k = 0; k < EL / 2; ++k) {
            c1[2 * k] += ntt::fmodmul(v[2 * k], wa[k].x, q, qinv);
            c1[2 * k + 1] += ntt::fmodmul(v[2 * k + 1], wa[k].y, q, qinv);
        }
        tmem_st_d<EL>(tcol, c1);
    }
};

struct IntKey {
    const u64 *evk, *evk_sh;
    long long key_stride, ioff;
    u64 q, two_q;
    template <int EL, class S1>
    __device__ __forceinline__ void unit(int t, long long pos, const u64* v, u64* s0, S1 s1) const {
        const long long kb = (2LL * t) * key_stride + ioff + pos, ka = kb + key_stride;
        const ulonglong2* b = reinterpret_cast<const ulonglong2*>(evk + kb);
        const ulonglong2* bs = reinterpret_cast<const ulonglong2*>(evk_sh + kb);
        const ulonglong2* a = reinterpret_cast<const ulonglong2*>(evk + ka);
        const ulonglong2* as = reinterpret_cast<const ulonglong2*>(evk_sh + ka);
#pragma unroll
        for (int k = 0; k < EL / 2; ++k) {
            const ulonglong2 wb = __ldg(b + k), wbs = __ldg(bs + k), wa = __ldg(a + k), was = __ldg(as + k);
            const u64 kbv[2] = {wb.x, wb.y}, kbs[2] = {wbs.x, wbs.y}, kav[2] = {wa.x, wa.y}, kas[2] = {was.x, was.y};
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int e = 2 * k + h;
                const u64 x0 = s0[e] + mul_shoup_lazy(v[e], kbv[h], kbs[h], q);
                u64& r1 = s1(e);
                const u64 x1 = r1 + mul_shoup_lazy(v[e], kav[h], kas[h], q);
                s0[e] = x0 >= two_q ? x0 - two_q : x0;
                r1 = x1 >= two_q ? x1 - two_q : x1;
            }
        }
    }
    // c1 read-modify-written in this thread's tensor-memory columns
    template <int EL>
    __device__ __forceinline__ void unit_tm(int t, long long pos, const u64* v, u64* s0, uint32_t tcol) const {
        u64 c1[EL];
        tmem_ld_u<EL>(tcol, c1);
        unit<EL>(t, pos, v, s0, [&](int e) -> u64& { return c1[e]; });
        tmem_st_u<EL>(tcol, c1);
    }
};

// Persistent, one launch for both limb kinds: CTAs [0, g_int) walk the
// integer-limb items (60-bit primes, IMAD pipes), CTAs [g_int, grid) the
// FP64-limb items, each group with its own grid stride over
// item = (ct * nsel + i - limb0) * nblocks + b for its limb range
// (ciphertext-major, so the CTAs in flight share the ciphertexts' digits in
// L2). A limb range may cover limbs of the other kind (mixed chains); those
// items are skipped.
template <int LOGN, int LOGB, int LOGE, int T, bool FPK, bool LIFT, bool AUXK>
__device__ __forceinline__ void ks_walk(const DevRing& R, const u32* digits, const u64* evk, const u64* evk_sh,
                                        const double* evk_f, u64* acc01, int level, int D, int limb0, int nsel,
                                        long long items, long long first, long long stride, int mode, const u64* fy,
                                        uint32_t tm_lane, unsigned& bphase, unsigned& tphase, u64* aux_out) {
    constexpr int C = LOGN - LOGB;
    const long long n = 1LL << LOGN;
    const long long key_stride = static_cast<long long>(R.limbs) * n;  // one evk polynomial
    int tw_key = -1;  // (limb, block) whose twiddle table is in shared memory
    for (long long item = first; item < items; item += stride) {
        const int b = static_cast<int>(item & ((1 << C) - 1));
        const long long row = item >> C;  // ct * nsel + (i - limb0)
        const long long ct = row / nsel;
        const int i = limb0 + static_cast<int>(row % nsel);
        const u64 q = R.mod[i].q;
        if (ntt::fp_limb(q) != FPK) continue;
        const long long ioff = static_cast<long long>(i) * n;
        const int key_now = (i << C) + b;
        const bool load_tw = key_now != tw_key;
        tw_key = key_now;
        if constexpr (FPK) {
            const ntt::FpArith ar{static_cast<double>(q), R.inv_q[i]};
            const FpKey key{evk_f, key_stride, ioff, ar.q, ar.qinv};
            const int aux_slot = AUXK && aux_out && i >= 1 && i <= 3 ? i : -1;
            ks_item<LOGN, LOGB, LOGE, T, LIFT, AUXK>(R, ar, R.ks_tw_f + ioff + (static_cast<long long>(b) << LOGB),
                                                     load_tw, digits, key, acc01, level, D, ct, i, b, q, mode, fy,
                                                     tm_lane, bphase, tphase, aux_slot, R.aux_tab, aux_out);
        } else {
            // primes >= 2^42 only: digits < 2^20 < q are residues already
            const ntt::IntArith ar{q, q << 1};
            const IntKey key{evk, evk_sh, key_stride, ioff, q, q << 1};
            ks_item<LOGN, LOGB, LOGE, T, false, AUXK>(R, ar, R.ks_tw + ioff + (static_cast<long long>(b) << LOGB),
                                                      load_tw, digits, key, acc01, level, D, ct, i, b, q, mode, fy,
                                                      tm_lane, bphase, tphase, -1, nullptr, nullptr);
        }
    }
}

template <int LOGN, int LOGB, int LOGE, int T, int MINB, bool LIFT, bool AUXK>
__global__ void __launch_bounds__(T, MINB) k_keyswitch(DevRing R, const u32* __restrict__ digits, const u64* __restrict__ evk,
                                                 const u64* __restrict__ evk_sh, const double* __restrict__ evk_f,
                                                 u64* __restrict__ acc01, int level, int D, int fp0, int nfp,
                                                 long long items_fp, int int0, int nint, long long items_int, int g_int,
                                                 int mode, const u64* __restrict__ fy, u64* __restrict__ aux_out) {
    constexpr int B = 1 << LOGB;
    using SF = KsShape<LOGN, LOGB, LOGE, T, true, AUXK>;
    using SI = KsShape<LOGN, LOGB, LOGE, T, false, AUXK>;
    static_assert(SF::USE_TMEM == SI::USE_TMEM && SF::TCW == SI::TCW, "both limb kinds share the TMEM layout");
    extern __shared__ u64 smem[];
    uint64_t* bbar = reinterpret_cast<uint64_t*>(smem + 3 * B);
    uint64_t* tbar = bbar + 1;
    uint32_t tm_lane = 0;
    __shared__ uint32_t tm_slot;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(ntt::smem_addr(bbar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(ntt::smem_addr(tbar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if constexpr (SF::USE_TMEM) {
        if (threadIdx.x < 32) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(ntt::smem_addr(&tm_slot)),
                         "n"(SF::TCOLS));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    }
    __syncthreads();
    if constexpr (SF::USE_TMEM) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int w = threadIdx.x >> 5;
        tm_lane = tm_slot + (static_cast<uint32_t>((w & 3) * 32) << 16) + static_cast<uint32_t>((w >> 2) * SF::TCW);
    }
    unsigned bphase = 0, tphase = 0;
    if (static_cast<int>(blockIdx.x) < g_int)
        ks_walk<LOGN, LOGB, LOGE, T, false, false, AUXK>(R, digits, evk, evk_sh, evk_f, acc01, level, D, int0, nint,
                                                         items_int, blockIdx.x, g_int, mode, fy, tm_lane, bphase, tphase,
                                                         nullptr);
    else
        ks_walk<LOGN, LOGB, LOGE, T, true, LIFT, AUXK>(R, digits, evk, evk_sh, evk_f, acc01, level, D, fp0, nfp,
                                                       items_fp, blockIdx.x - g_int, gridDim.x - g_int, mode, fy,
                                                       tm_lane, bphase, tphase, aux_out);
    if constexpr (SF::USE_TMEM) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        if (threadIdx.x < 32) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm_slot), "n"(SF::TCOLS));
        }
    }
}

// block size: the block twiddle tables (DevRing::ks_tw) are built for 2^13
constexpr int HECNN_KS_LOGB = 13;
#ifndef HECNN_KS_LOGE
#define HECNN_KS_LOGE 3
#endif
#ifndef HECNN_KS_MAXT
#define HECNN_KS_MAXT 512
#endif
#ifndef HECNN_KS_MINB
#define HECNN_KS_MINB 1
#endif
#ifndef HECNN_KS_MAXT_COL
#define HECNN_KS_MAXT_COL 1024
#endif

template <int LOGN>
struct KsPlan {
    static constexpr int LOGB = LOGN <= HECNN_KS_LOGB ? LOGN : HECNN_KS_LOGB;
    static constexpr int LOGE = LOGB >= 8 ? HECNN_KS_LOGE : 3;
    static constexpr int B = 1 << LOGB;
    static constexpr int UNITS = B >> LOGE;
    // N > 2^13 (column stages recomputed per block): 1024 threads, 8 words
    // each, measured 6% faster at N = 2^14 than 512 x 16; 512 at N <= 2^13
    static constexpr int MAXT = LOGN > LOGB ? HECNN_KS_MAXT_COL : HECNN_KS_MAXT;
    static constexpr int T = UNITS >= MAXT ? MAXT : (UNITS >= 32 ? UNITS : (B < 32 ? B : 32));
    static constexpr int MINB = T >= 256 ? HECNN_KS_MINB : 1;
};

// ---- limb 0 through limbs 1..3 ("aux") --------------------------------------
// The reference's limb-0 accumulators are sum_t NTT_q0(d_t) (.) b_{t,0} =
// NTT_q0(E mod q0) with E = sum_t d_t (*) B_t the exact negacyclic integer
// convolution of the digits with B_t = INTT_q0(b_{t,0}) in [0, q0) (likewise
// for a). |E| < D N 2^20 q0 < P/2 for P = q1 q2 q3, so E is recovered exactly
// from E mod q_s, s = 1..3 -- which the FP64 items of limbs 1..3 accumulate
// beside their own key switch from the digit transforms they already compute
// (Tb / Ta = NTT_{q_s}(B_t mod q_s), DevRing::aux_tab) -- by an inverse NTT in
// each limb, a 3-prime CRT and a forward NTT mod q0. The 60-bit limb's D
// integer-pipe digit NTTs disappear; every word stays the reference's.

// E mod q_s (s = 1..3, canonical) -> centred E mod q0. X = sum_s y_s (P / q_s)
// with y_s = r_s (P / q_s)^-1 mod q_s is E + k P, k = rint(sum_s y_s / q_s)
// (= X / P, whose distance to k is |E| / P < 1/4: keyswitch_aux_ok keeps that
// margin, far above the double sum's 2^-50 error), so
// E mod q0 = sum_s y_s ((P / q_s) mod q0) - k (P mod q0): three Shoup
// products mod q0, no 128-bit arithmetic
__device__ __forceinline__ u64 aux_crt_value(const DevRing& R, const u64 (&res)[3]) {
    const u64 q0 = R.mod[0].q;
    double f = 0.0;
    u64 acc = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const u64 qa = R.mod[1 + a].q;
        const u64 y = mul_shoup(res[a], R.aux_inv[a].x, R.aux_inv[a].y, qa);  // < q_s < 2^42
        f += static_cast<double>(y) * R.inv_q[1 + a];
        acc = add_mod(acc, mul_shoup(y, R.aux_Mq0[a].x, R.aux_Mq0[a].y, q0), q0);
    }
    const int k = static_cast<int>(rint(f));  // 0..3
    // (selects, not a runtime index into the kernel-parameter array, which would
    // copy DevRing to the stack)
    const u64 kp = k == 0 ? 0 : (k == 1 ? R.aux_kPq0[1] : (k == 2 ? R.aux_kPq0[2] : R.aux_kPq0[3]));
    return sub_mod(acc, kp, q0);
}

// CRT of each coefficient fused into the first round of the forward NTT mod
// q0: e0 [ct * 2 + comp][n] = NTT_q0(E mod q0); one CTA per polynomial (N <= 2^14)
template <int LOGN, int T, int MINB>
__global__ void __launch_bounds__(T, MINB) k_aux_crt_ntt(DevRing R, const u64* __restrict__ aux_out, u64* __restrict__ e0) {
    extern __shared__ u64 smem[];
    const long long row = blockIdx.x;  // ct * 2 + comp
    const long long n = 1LL << LOGN;
    const u64* a1 = aux_out + (row * 4 + 1) * n;
    u64* g = e0 + row * n;
    const u64 q = R.mod[0].q;
    const ntt::IntArith ar{q, q << 1};
    ntt::fwd_block<LOGN, 3, T>(
        smem, ar, R.fwd, 0, 0,
        [=](int i) {
            const u64 res[3] = {a1[i], a1[n + i], a1[2 * n + i]};
            return aux_crt_value(R, res);
        },
        [=](int i, u64 v, int, int) { g[i] = reduce_4q(v, q); });
}

// limb 0 of acc01 (NTT domain): the tensor product's (d0, d1) (mode as in
// keyswitch_mac) plus NTT_q0(E) of each component
__global__ void k_limb0_combine(DevRing R, u64* __restrict__ acc01, const u64* __restrict__ e0, const u64* __restrict__ fy,
                                int limbs, int mode, long long count) {
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= count * R.n) return;
    const long long ct = t / R.n;
    const int j = static_cast<int>(t % R.n);
    const ModConst m = R.mod[0];
    u64* o0 = acc01 + (ct * 2) * limbs * R.n + j;
    u64* o1 = o0 + static_cast<long long>(limbs) * R.n;
    const u64 xa = *o0, xb = *o1;
    u64 b0, b1;
    if (mode == 0) {
        b0 = xa, b1 = xb;
    } else if (mode == 1) {
        b0 = mul_mod(xa, xa, m);
        const u64 c = mul_mod(xa, xb, m);
        b1 = add_mod(c, c, m.q);
    } else {
        const u64* y0 = fy + (ct * 2) * limbs * R.n + j;
        const u64 va = y0[0], vb = y0[static_cast<long long>(limbs) * R.n];
        b0 = mul_mod(xa, va, m);
        b1 = add_mod(mul_mod(xa, vb, m), mul_mod(xb, va, m), m.q);
    }
    *o0 = add_mod(b0, e0[(ct * 2) * R.n + j], m.q);
    *o1 = add_mod(b1, e0[(ct * 2 + 1) * R.n + j], m.q);
}

// deferred variant (the caller inverse-transforms acc01 next): limb 0 of
// acc01 gets the tensor product's (d0, d1) only, and e0 [ct * 2 + comp][n]
// receives E mod q0 as coefficients, to be added after the caller's INTT --
// NTT_q0 followed by INTT_q0 of E cancels, so neither runs
__global__ void __launch_bounds__(256, 4) k_limb0_crt_combine(DevRing R, u64* __restrict__ acc01, const u64* __restrict__ aux_out,
                                    u64* __restrict__ e0, const u64* __restrict__ fy, int limbs, int mode,
                                    long long count) {
    // two consecutive coefficients per thread (16-byte accesses); the four CRT
    // chains (2 coefficients x 2 components) are independent
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long n = R.n;
    if (t >= count * (n >> 1)) return;
    const long long ct = t / (n >> 1);
    const int j = static_cast<int>(t % (n >> 1)) * 2;
    u64 res[2][2][3];
#pragma unroll
    for (int comp = 0; comp < 2; ++comp)
#pragma unroll
        for (int s = 0; s < 3; ++s) {
            const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(aux_out + ((ct * 2 + comp) * 4 + 1 + s) * n + j));
            res[comp][0][s] = v.x, res[comp][1][s] = v.y;
        }
    u64 e[2][2];
#pragma unroll
    for (int comp = 0; comp < 2; ++comp)
#pragma unroll
        for (int h = 0; h < 2; ++h) e[comp][h] = aux_crt_value(R, res[comp][h]);
#pragma unroll
    for (int comp = 0; comp < 2; ++comp)
        *reinterpret_cast<ulonglong2*>(e0 + (ct * 2 + comp) * n + j) = make_ulonglong2(e[comp][0], e[comp][1]);
    if (mode == 0) return;
    const ModConst m = R.mod[0];
    u64* o0 = acc01 + (ct * 2) * limbs * n + j;
    u64* o1 = o0 + static_cast<long long>(limbs) * n;
    const ulonglong2 xa = *reinterpret_cast<const ulonglong2*>(o0), xb = *reinterpret_cast<const ulonglong2*>(o1);
    const u64 a[2] = {xa.x, xa.y}, bb[2] = {xb.x, xb.y};
    u64 r0[2], r1[2];
    if (mode == 1) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            r0[h] = mul_mod(a[h], a[h], m);
            const u64 c = mul_mod(a[h], bb[h], m);
            r1[h] = add_mod(c, c, m.q);
        }
    } else {
        const u64* y0 = fy + (ct * 2) * limbs * n + j;
        const ulonglong2 va2 = *reinterpret_cast<const ulonglong2*>(y0);
        const ulonglong2 vb2 = *reinterpret_cast<const ulonglong2*>(y0 + static_cast<long long>(limbs) * n);
        const u64 va[2] = {va2.x, va2.y}, vb[2] = {vb2.x, vb2.y};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            r0[h] = mul_mod(a[h], va[h], m);
            r1[h] = add_mod(mul_mod(a[h], vb[h], m), mul_mod(bb[h], va[h], m), m.q);
        }
    }
    *reinterpret_cast<ulonglong2*>(o0) = make_ulonglong2(r0[0], r0[1]);
    *reinterpret_cast<ulonglong2*>(o1) = make_ulonglong2(r1[0], r1[1]);
}

// aux_tab build: rows of B (coefficients mod q0) -> slot s of [rows][4][n] = B mod q_s
__global__ void k_aux_rows(DevRing R, const u64* __restrict__ b, u64* __restrict__ w, long long rows) {
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= rows * R.n) return;
    const long long row = t / R.n;
    const int j = static_cast<int>(t % R.n);
    const u64 v = b[row * R.n + j];
    w[(row * 4) * R.n + j] = 0;
#pragma unroll
    for (int s = 1; s <= 3; ++s) w[(row * 4 + s) * R.n + j] = reduce128(v, 0, R.mod[s]);
}

template <int LOGN>
const u64* run_keyswitch(const DevRing& R, const u32* digits, const u64* evk, const u64* evk_sh, const double* evk_f,
                         u64* acc01, int level, int D, std::size_t count, const Launch& L, int mode, const u64* fy,
                         u64* aux_scratch, bool defer) {
    using P = KsPlan<LOGN>;
#ifdef HECNN_KS_FORCE_LIFT
    const bool lift = true;
#else
    const bool lift = R.small_primes;
#endif
    const bool aux = aux_scratch && keyswitch_aux_ok(R, level, D);
    auto pick = [&](bool lf, bool ax) {
        if constexpr (LOGN >= 10 && LOGN <= 14 && KsShape<LOGN, P::LOGB, P::LOGE, P::T, true, true>::TM) {
            if (ax)
                return lf ? k_keyswitch<LOGN, P::LOGB, P::LOGE, P::T, P::MINB, true, true>
                          : k_keyswitch<LOGN, P::LOGB, P::LOGE, P::T, P::MINB, false, true>;
        }
        return lf ? k_keyswitch<LOGN, P::LOGB, P::LOGE, P::T, P::MINB, true, false>
                  : k_keyswitch<LOGN, P::LOGB, P::LOGE, P::T, P::MINB, false, false>;
    };
    auto kern = pick(lift, aux);
    // data + staged twiddles (u64 Shoup pairs on the integer path; double
    // twiddles + the b_t stage or c1 accumulators on the FP64 path) + mbarriers
    const int smem = P::B * (8 + 16) + 64;
    smem_opt_in(kern, smem);
    const int limbs = level + 1;
    const unsigned long long lmask = limbs >= 64 ? ~0ull : (1ull << limbs) - 1;
    const unsigned long long int_mask = R.int_limbs & lmask;
    // exact limb ranges when only q0 is an integer limb (the presets); otherwise
    // both CTA groups cover every limb and skip the other kind's items
    int fp0 = 0, nfp = limbs, int0 = 0, nint = limbs;
    if (int_mask == 0) nint = 0;
    else if (int_mask == lmask) nfp = 0;
    else if (int_mask == 1) { fp0 = 1; nfp = limbs - 1; nint = 1; }
    if (aux) nint = 0;  // limb 0 rides on limbs 1..3
    const double n = double(1 << LOGN), cl = double(count) * limbs;
    // per (ct, limb, digit): one N-point NTT + 2N MACs; bytes: evk once + digits + acc r/w
    L.begin("k_keyswitch", cl * D * (n / 2 * LOGN + 2 * n),
            2.0 * D * limbs * n * 8 + double(count) * D * n * 4 + cl * 2 * n * 8 * 2);
    // Persistent grid = resident CTAs per SM x SMs, split between the two CTA
    // groups in proportion to their work (an integer-limb item costs
    // HECNN_KS_INT_COST FP64 items), so both groups finish together.
    static int sms = 0, occ = 0;
    if (!sms) {
        int dev = 0;
        cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
        cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "cudaDeviceGetAttribute");
        cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, P::T, smem), "occupancy");
        occ = std::max(occ, 1);
    }
#ifndef HECNN_KS_INT_COST
#define HECNN_KS_INT_COST 2.75
#endif
    const long long nb = 1LL << (LOGN - P::LOGB);
    const long long items_fp = static_cast<long long>(count) * nfp * nb, items_int = static_cast<long long>(count) * nint * nb;
    const int n_int_limbs = nint ? __builtin_popcountll(int_mask) : 0;
    const double w_fp = double(count) * (limbs - n_int_limbs) * nb, w_int = double(count) * n_int_limbs * nb * HECNN_KS_INT_COST;
    const long long cap = static_cast<long long>(sms) * occ;
    long long g_int = 0, g_fp = 0;
    if (!items_int) {
        g_fp = std::min(cap, items_fp);
    } else if (!items_fp) {
        g_int = std::min(cap, items_int);
    } else {
        g_int = std::llround(double(cap) * w_int / (w_int + w_fp));
        g_int = std::min(std::max(g_int, 1LL), cap - 1);
        g_fp = cap - g_int;
        g_int = std::min(g_int, items_int);
        g_fp = std::min(g_fp, items_fp);
    }
    u64* aux_out = aux ? aux_scratch : nullptr;
    kern<<<static_cast<unsigned>(g_int + g_fp), P::T, smem, L.stream>>>(R, digits, evk, evk_sh, evk_f, acc01, level, D, fp0,
                                                                       nfp, items_fp, int0, nint, items_int,
                                                                       static_cast<int>(g_int), mode, fy, aux_out);
    L.count(1);
    if (aux) {
        // E mod q_s -> coefficients (limbs 1..3 of [ct][comp][4][n]), CRT -> E mod q0,
        // NTT_q0, then limb 0 = d + NTT_q0(E)
        u64* e0 = aux_scratch + count * 2 * 4 * (1ull << LOGN);
        if constexpr (LOGN > P::LOGB) ntt_inverse_limbs(R, aux_scratch, 4, 1, 3, count * 2, L, "k_ks_aux_intt");
        // (N <= 2^13: the key-switch CTAs of limbs 1..3 wrote coefficients already)
        const long long pos = static_cast<long long>(count) << LOGN;
        if (defer) {
            L.begin("k_ks_aux_crt", double(pos) * 2 * 12, 8.0 * pos * (6 + 2 + (mode ? 4 : 0) + (mode == 2 ? 2 : 0)));
            k_limb0_crt_combine<<<static_cast<unsigned>((pos / 2 + 255) / 256), 256, 0, L.stream>>>(
                R, acc01, aux_scratch, e0, fy, limbs, mode, static_cast<long long>(count));
            L.count();
            return e0;
        }
        constexpr int TN = (1 << LOGN) / 8 >= 512 ? 512 : ((1 << LOGN) / 8 >= 32 ? (1 << LOGN) / 8 : 32);
        constexpr int MB = LOGN <= 13 ? 2 : 1;
        auto kc = k_aux_crt_ntt<LOGN, TN, MB>;
        const int csm = (1 << LOGN) * 8;
        smem_opt_in(kc, csm);
        const double cells = double(count) * 2 * (1 << LOGN);
        L.begin("k_ks_aux_crt_ntt", cells * (LOGN / 2.0 + 6), 8.0 * cells * 4);
        kc<<<static_cast<unsigned>(count * 2), TN, csm, L.stream>>>(R, aux_scratch, e0);
        L.count();
        L.begin("k_ks_aux_combine", double(pos) * 4, 8.0 * pos * 6);
        k_limb0_combine<<<static_cast<unsigned>((pos + 255) / 256), 256, 0, L.stream>>>(R, acc01, e0, fy, limbs, mode,
                                                                                      static_cast<long long>(count));
        L.count();
    }
    return nullptr;
}

}  // namespace

void crt_digits(const DevRing& R, const u64* d2, u32* digits, int level, int D, std::size_t count, const Launch& L) {
    if (!count) return;
    const long long total = static_cast<long long>(count) * R.n;
    const unsigned grid = static_cast<unsigned>((total + 127) / 128);
    const int W = R.crt_words;
#ifndef HECNN_CRT_GARNER
#define HECNN_CRT_GARNER 1
#endif
    const unsigned long long lmask = level + 1 >= 64 ? ~0ull : (1ull << (level + 1)) - 1;
    if (HECNN_CRT_GARNER && R.garner_inv && (R.int_limbs & lmask) == 1) {
        const int smem = 128 * (level + 1) * 8;
#define HECNN_CRT_CASE(WW) \
    case WW: smem_opt_in(k_crt_digits_garner<WW>, smem); L.begin("k_crt_digits", double(count) * R.n * (level + 1) * (WW + 1), double(count) * R.n * ((level + 1) * 8 + D * 4)); k_crt_digits_garner<WW><<<grid, 128, smem, L.stream>>>(R, d2, digits, level, D, static_cast<long long>(count)); break;
        switch (W) {
            HECNN_CRT_CASE(2) HECNN_CRT_CASE(3) HECNN_CRT_CASE(4) HECNN_CRT_CASE(5) HECNN_CRT_CASE(6) HECNN_CRT_CASE(7)
            HECNN_CRT_CASE(8) HECNN_CRT_CASE(9) HECNN_CRT_CASE(10) HECNN_CRT_CASE(11) HECNN_CRT_CASE(12)
            HECNN_CRT_CASE(13) HECNN_CRT_CASE(14) HECNN_CRT_CASE(15) HECNN_CRT_CASE(16) HECNN_CRT_CASE(17)
            HECNN_CRT_CASE(18) HECNN_CRT_CASE(19) HECNN_CRT_CASE(20)
            default: throw std::invalid_argument("key_switch: modulus chain too long for the device CRT kernel");
        }
#undef HECNN_CRT_CASE
        L.count();
        check_launch("crt_digits");
        return;
    }
#define HECNN_CRT_CASE(WW) \
    case WW: L.begin("k_crt_digits", double(count) * R.n * (level + 1) * (WW + 1), double(count) * R.n * ((level + 1) * 8 + D * 4)); k_crt_digits<WW><<<grid, 128, 0, L.stream>>>(R, d2, digits, level, D, static_cast<long long>(count)); break;
    switch (W) {
        HECNN_CRT_CASE(2) HECNN_CRT_CASE(3) HECNN_CRT_CASE(4) HECNN_CRT_CASE(5) HECNN_CRT_CASE(6) HECNN_CRT_CASE(7)
        HECNN_CRT_CASE(8) HECNN_CRT_CASE(9) HECNN_CRT_CASE(10) HECNN_CRT_CASE(11) HECNN_CRT_CASE(12)
        HECNN_CRT_CASE(13) HECNN_CRT_CASE(14) HECNN_CRT_CASE(15) HECNN_CRT_CASE(16) HECNN_CRT_CASE(17)
        HECNN_CRT_CASE(18) HECNN_CRT_CASE(19) HECNN_CRT_CASE(20)
        default: throw std::invalid_argument("key_switch: modulus chain too long for the device CRT kernel");
    }
#undef HECNN_CRT_CASE
    L.count();
    check_launch("crt_digits");
}

namespace {
// the FP64 key-switch items keep c1 in tensor memory at this ring degree (the
// aux accumulators live beside it)
template <int LOGN>
constexpr bool aux_shape() {
    using P = KsPlan<LOGN>;
    return KsShape<LOGN, P::LOGB, P::LOGE, P::T, true, true>::TM;
}
bool aux_shape_ok(int logn) {
    switch (logn) {
        case 10: return aux_shape<10>();
        case 11: return aux_shape<11>();
        case 12: return aux_shape<12>();
        case 13: return aux_shape<13>();
        case 14: return aux_shape<14>();
        default: return false;
    }
}
}  // namespace

bool keyswitch_aux_ok(const DevRing& R, int level, int D) {
#ifndef HECNN_KS_AUX
#define HECNN_KS_AUX 1
#endif
    if (!HECNN_KS_AUX || !R.aux_tab || level < 3 || !aux_shape_ok(R.logn)) return false;
    const unsigned long long lmask = level + 1 >= 64 ? ~0ull : (1ull << (level + 1)) - 1;
    if ((R.int_limbs & lmask) != 1) return false;  // the 60-bit limb 0 alone on the integer path
    // |E| < D N 2^20 q0 must stay below P / 2 (one bit of margin)
    const double bits = std::log2(double(D)) + R.logn + 20.0 + 61.0 + 2.0;
    return bits < R.aux_log2P;
}

void keyswitch_aux_tables(const DevRing& R, const u64* evk, std::size_t evk_limbs, int Dtop, double* out, u64* tmp,
                          const Launch& L) {
    const std::size_t n = static_cast<std::size_t>(R.n), rows = 2 * static_cast<std::size_t>(Dtop);
    // limb 0 of every evk polynomial, back to coefficients (INTT mod q0)
    cuda_check(cudaMemcpy2DAsync(tmp, n * 8, evk, evk_limbs * n * 8, n * 8, rows, cudaMemcpyDeviceToDevice, L.stream),
               "copy evk limb 0");
    ntt_inverse(R, tmp, 0, rows, L);
    // slots 1..3: B mod q_s, then NTT in each slot's limb, as exact doubles
    u64* w = tmp + rows * n;
    const long long cells = static_cast<long long>(rows * n);
    k_aux_rows<<<static_cast<unsigned>((cells + 255) / 256), 256, 0, L.stream>>>(R, tmp, w, static_cast<long long>(rows));
    L.count();
    ntt_forward(R, w, 3, rows, L);
    fp_table(R, w, out, 4, rows, L);
    check_launch("keyswitch_aux_tables");
}

const u64* keyswitch_mac(const DevRing& R, const u32* digits, const u64* evk, const u64* evk_sh, const double* evk_f,
                         u64* acc01, int level, int D, std::size_t count, const Launch& L, int mode, const u64* fy,
                         u64* aux_scratch, bool defer_limb0) {
    if (!count) return nullptr;
    const u64* e0 = nullptr;
    if (mode == 2 && !fy) throw std::invalid_argument("keyswitch_mac: product mode needs the second operand");
#define HECNN_KS_CASE(LG) \
    case LG: e0 = run_keyswitch<LG>(R, digits, evk, evk_sh, evk_f, acc01, level, D, count, L, mode, fy, aux_scratch, defer_limb0); break;
    switch (R.logn) {
        HECNN_KS_CASE(3) HECNN_KS_CASE(4) HECNN_KS_CASE(5) HECNN_KS_CASE(6) HECNN_KS_CASE(7) HECNN_KS_CASE(8)
        HECNN_KS_CASE(9) HECNN_KS_CASE(10) HECNN_KS_CASE(11) HECNN_KS_CASE(12) HECNN_KS_CASE(13)
        HECNN_KS_CASE(14) HECNN_KS_CASE(15) HECNN_KS_CASE(16)
        default: throw std::invalid_argument("key_switch: ring degree outside 2^3..2^16 is not supported on the device");
    }
#undef HECNN_KS_CASE
    check_launch("keyswitch_mac");
    return e0;
}

__global__ void k_add_limb0(DevRing R, u64* __restrict__ d, const u64* __restrict__ add0, int limbs, long long groups) {
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= groups * R.n) return;
    const long long g = t / R.n;
    const int j = static_cast<int>(t % R.n);
    u64* p = d + g * limbs * R.n + j;
    *p = add_mod(*p, add0[t], R.mod[0].q);
}

void add_limb0(const DevRing& R, u64* d, const u64* add0, int limbs, std::size_t groups, const Launch& L) {
    if (!groups) return;
    const long long cells = static_cast<long long>(groups) * R.n;
    L.begin("k_ks_aux_add", double(cells), 24.0 * cells);
    k_add_limb0<<<static_cast<unsigned>((cells + 255) / 256), 256, 0, L.stream>>>(R, d, add0, limbs,
                                                                               static_cast<long long>(groups));
    L.count();
    check_launch("add_limb0");
}

}  // namespace hecnn_b200
