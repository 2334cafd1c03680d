// Register-blocked negacyclic NTT rounds shared by the NTT kernels (ntt.cu)
// and the fused key-switch kernel (keyswitch.cu).
//
// A block of B = 2^LOGB words of one limb is transformed by one CTA. Stages
// are grouped in rounds of R <= LOGE stages; in a round a thread owns units
// of 2^R words (stride G >> R inside a group of G = B >> S0 words) and runs
// the R stages on registers. Between rounds words live in shared memory at
// swizzled addresses (swz, conflict free for every round shape; see
// DESIGN.md). The first round may load from anywhere and the last round may
// store anywhere through functors, so kernels fuse their input lift and
// output epilogue into the transform instead of extra shared-memory passes.
//
// Butterflies follow the reference's networks exactly (NttTables::forward /
// inverse, ring.hpp:83-137): forward CT with twiddle psi^bitrev(2^s + i),
// inverse GS with psi^-bitrev(2^s + i). Two arithmetic policies:
//   IntArith -- 64-bit Shoup on the integer pipes, lazy [0,4q) / [0,2q)
//               (any q < 2^61; used for the 60-bit chain prime),
//   FpArith  -- exact modular arithmetic on the FP64 pipe for q < 2^42:
//               signed doubles, fmodmul() below, no per-stage corrections in
//               the forward network, one centring per inverse round. B200
//               runs it 2.7x faster than integer Shoup (tools/modmul_probe.cu).
// Both produce the same residues; the caller's epilogue makes them canonical.
#pragma once
#include <cstdint>
#include <type_traits>

#include "kernels.hpp"

namespace hecnn_b200 {
namespace ntt {

__host__ __device__ __forceinline__ constexpr int swz(int i) {
    return i ^ static_cast<int>((0x1eb4d278963c5af0ull >> (4 * ((i >> 4) & 15))) & 15);
}
// swz is GF(2)-linear (the nibble table is a linear map of bits 4..7 onto
// bits 0..3), so for a unit's positions base | k * STRIDE (disjoint bit
// fields) swz(base | k * STRIDE) == swz(base) ^ swz(k * STRIDE): one XOR with
// a compile-time constant per element instead of the table lookup.
static_assert(swz(0x50) == (swz(0x10) ^ swz(0x40)) && swz(0xf3) == (swz(0xf0) ^ 3) &&
                  swz(0xa7) == (swz(0x80) ^ swz(0x20) ^ 7),
              "swizzle must be GF(2)-linear");

__device__ __forceinline__ void ct_butterfly(u64& a, u64& b, ulonglong2 w, u64 q, u64 two_q) {
    u64 u = a;
    if (u >= two_q) u -= two_q;
    const u64 v = mul_shoup_lazy(b, w.x, w.y, q);
    a = u + v;
    b = u + two_q - v;
}

__device__ __forceinline__ void gs_butterfly(u64& a, u64& b, ulonglong2 w, u64 q, u64 two_q) {
    const u64 u = a, v = b;
    u64 s = u + v;
    if (s >= two_q) s -= two_q;
    a = s;
    b = mul_shoup_lazy(u + two_q - v, w.x, w.y, q);
}

// ---- exact FP64 modular arithmetic (q < 2^42) -------------------------------
constexpr double kMagicRound = 6755399441055744.0;  // 1.5 * 2^52: x + M - M == rint(x), |x| < 2^51
constexpr double kTwo52 = 4503599627370496.0;

// x * w mod q in (-q, q) for |x| < 2^45, 0 <= w < q < 2^42, qinv = fl(1/q):
// h + l == x*w exactly (FMA error-free product); t = rint(h * qinv) is within
// 0.5 + 2^-6 of x*w/q (|h - xw| <= 2^35, relative error of qinv 2^-53), so
// h - t*q and (h - t*q) + l are integers below 2^52 and both steps are exact.
// Verified exhaustively on 2^26 signed inputs by tools/modmul_probe.cu.
__device__ __forceinline__ double fmodmul(double x, double w, double q, double qinv) {
    const double h = x * w;
    const double l = fma(x, w, -h);
    const double t = fma(h, qinv, kMagicRound) - kMagicRound;
    return fma(-t, q, h) + l;
}

// |v| < 2^51 -> centred residue in (-q/2 - 1, q/2 + 1)
__device__ __forceinline__ double fcentre(double v, double q, double qinv) {
    const double t = fma(v, qinv, kMagicRound) - kMagicRound;
    return fma(-t, q, v);
}

// |v| < 2^51 -> canonical residue as u64
__device__ __forceinline__ u64 fcanon(double v, double q, double qinv) {
    double r = fcentre(v, q, qinv);
    if (r < 0) r += q;
    if (r >= q) r -= q;
    return static_cast<u64>(__double_as_longlong(r + kTwo52) - __double_as_longlong(kTwo52));
}

// u64 < 2^52 -> exact double
__device__ __forceinline__ double to_fp(u64 v) {
    return __longlong_as_double(static_cast<long long>(v | 0x4330000000000000ull)) - kTwo52;
}

struct IntArith {
    using V = u64;
    using TW = ulonglong2;
    u64 q, two_q;
    __device__ void ct(V& a, V& b, TW w) const { ct_butterfly(a, b, w, q, two_q); }
    __device__ void gs(V& a, V& b, TW w) const { gs_butterfly(a, b, w, q, two_q); }
    __device__ void round_end_inv(V&) const {}
};

struct FpArith {
    using V = double;
    using TW = double;  // the twiddle as an exact double
    double q, qinv;
    __device__ void ct(V& a, V& b, TW w) const {
        const double v = fmodmul(b, w, q, qinv);
        const double u = a;
        a = u + v;
        b = u - v;
    }
    __device__ void gs(V& a, V& b, TW w) const {
        const double u = a, v = b;
        a = u + v;
        b = fmodmul(u - v, w, q, qinv);
    }
    // GS sums double per stage; centre once per round (<= 4 stages) so every
    // value stays below 2^45 in magnitude.
    __device__ void round_end_inv(V& x) const { x = fcentre(x, q, qinv); }
};

__host__ __device__ constexpr int ceil_div(int a, int b) { return (a + b - 1) / b; }
// Balanced split of the remaining LOGB - s stages into rounds of <= LOGE.
__host__ __device__ constexpr int round_size(int LOGB, int LOGE, int s) {
    return ceil_div(LOGB - s, ceil_div(LOGB - s, LOGE));
}
// Stage index where the last round starts.
__host__ __device__ constexpr int last_round_start(int LOGB, int LOGE, int s = 0) {
    return s + round_size(LOGB, LOGE, s) >= LOGB ? s : last_round_start(LOGB, LOGE, s + round_size(LOGB, LOGE, s));
}

template <class V>
struct SmemLoad {
    const V* s;
    __device__ V operator()(int idx) const { return s[swz(idx)]; }
};
template <class V>
struct SmemStore {
    V* s;
    __device__ void operator()(int idx, V v, int, int) const { s[swz(idx)] = v; }
};

// Forward round: block-local stages S0..S0+R-1; global stage = c + local;
// `b` is the block index inside the N-point transform (twiddle offset).
#ifndef HECNN_NTT_BATCH
#define HECNN_NTT_BATCH 0
#endif
template <int LOGB, int R, int S0, int T, class A, class Load, class Store>
__device__ __forceinline__ void fwd_round(const A& ar, const typename A::TW* __restrict__ tw, int b, int c, Load load,
                                          Store store, int tid) {
    using V = typename A::V;
    constexpr int B = 1 << LOGB, G = B >> S0, STRIDE = G >> R, E = 1 << R, UNITS = B >> R;
    constexpr int PER = (UNITS + T - 1) / T;
    if constexpr (HECNN_NTT_BATCH && PER > 1 && UNITS % T == 0 && PER * E <= 16 &&
                  std::is_same<Store, SmemStore<V>>::value) {
        // all of the thread's units loaded first, butterflies interleaved
        // across units (2x the independent chains), then stored in order
        V x[PER][E];
#pragma unroll
        for (int uu = 0; uu < PER; ++uu) {
            const int u = tid + uu * T;
            const int base = (u / STRIDE) * G + u % STRIDE;
#pragma unroll
            for (int k = 0; k < E; ++k) {
                if constexpr (std::is_invocable_v<Load, int, int, int>) x[uu][k] = load(base + k * STRIDE, uu, k);
                else x[uu][k] = load(base + k * STRIDE);
            }
        }
#pragma unroll
        for (int rho = 0; rho < R; ++rho) {
            const int half = E >> (rho + 1);
#pragma unroll
            for (int blk = 0; blk < (1 << rho); ++blk) {
#pragma unroll
                for (int uu = 0; uu < PER; ++uu) {
                    const int grp = (tid + uu * T) / STRIDE;
                    const typename A::TW w = tw[(1 << (c + S0 + rho)) + (b << (S0 + rho)) + (grp << rho) + blk];
#pragma unroll
                    for (int kk = 0; kk < half; ++kk) ar.ct(x[uu][blk * 2 * half + kk], x[uu][blk * 2 * half + kk + half], w);
                }
            }
        }
#pragma unroll
        for (int uu = 0; uu < PER; ++uu) {
            const int u = tid + uu * T;
            const int base = (u / STRIDE) * G + u % STRIDE;
#pragma unroll
            for (int k = 0; k < E; ++k) store(base + k * STRIDE, x[uu][k], uu, k);
        }
    } else {
#pragma unroll
    for (int uu = 0; uu < PER; ++uu) {
        const int u = tid + uu * T;
        if (UNITS % T != 0 && u >= UNITS) break;
        const int grp = u / STRIDE, col = u % STRIDE;
        const int base = grp * G + col;
        const int sb = swz(base);
        V x[E];
#pragma unroll
        for (int k = 0; k < E; ++k) {
            // loads that can use the (unit, element) slot, e.g. prefetched registers
            if constexpr (std::is_same<Load, SmemLoad<V>>::value) x[k] = load.s[sb ^ swz(k * STRIDE)];
            else if constexpr (std::is_invocable_v<Load, int, int, int>) x[k] = load(base + k * STRIDE, uu, k);
            else x[k] = load(base + k * STRIDE);
        }
#pragma unroll
        for (int rho = 0; rho < R; ++rho) {
            const int half = E >> (rho + 1);
            const int tbase = (1 << (c + S0 + rho)) + (b << (S0 + rho)) + (grp << rho);
#pragma unroll
            for (int blk = 0; blk < (1 << rho); ++blk) {
                const typename A::TW w = tw[tbase + blk];
#pragma unroll
                for (int kk = 0; kk < half; ++kk) ar.ct(x[blk * 2 * half + kk], x[blk * 2 * half + kk + half], w);
            }
        }
#pragma unroll
        for (int k = 0; k < E; ++k) {
            if constexpr (std::is_same<Store, SmemStore<V>>::value) store.s[sb ^ swz(k * STRIDE)] = x[k];
            else store(base + k * STRIDE, x[k], uu, k);
        }
    }
    }
}

struct NoHook {
    __device__ void operator()() const {}
};

#ifndef HECNN_NTT_SPLIT
#define HECNN_NTT_SPLIT 1
#endif
// Group split: after the first forward round (stages 0..R0-1) the block falls
// apart into NG = 2^R0 independent sub-blocks of B >> R0 words, so the later
// rounds of sub-block g run on its own TG = T / NG threads (whole warps) and
// synchronise with a named barrier over those warps instead of the whole CTA
// (the inverse mirrors it: local rounds first, the global round last). Warps
// drift apart between the two CTA-wide barriers, so one warp group's shared
// memory traffic overlaps another's FP64 butterflies.
template <int LOGB, int LOGE, int T>
struct Split {
    static constexpr int R0 = round_size(LOGB, LOGE, 0);
    static constexpr int NG = 1 << R0, TG = T / NG, LB = LOGB - R0;
    static constexpr bool on = HECNN_NTT_SPLIT && R0 < LOGB && LB >= 8 && NG > 1 && NG <= 15 && T % NG == 0 &&
                               TG % 32 == 0;
};

__device__ __forceinline__ void group_sync(int g, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "r"(nthreads) : "memory");
}

// The rounds of one (sub-)block after its first: loads from `s`, the last
// round stores with `last`; `sync` separates rounds.
template <int LOGB, int LOGE, int T, class A, int S0, class Last, class Sync>
__device__ __forceinline__ void fwd_rest(typename A::V* s, const A& ar, const typename A::TW* tw, int b, int c, Last last,
                                         Sync sync, int tid) {
    using V = typename A::V;
    if constexpr (S0 < LOGB) {
        constexpr int R = round_size(LOGB, LOGE, S0);
        if constexpr (S0 + R >= LOGB) {
            fwd_round<LOGB, R, S0, T>(ar, tw, b, c, SmemLoad<V>{s}, last, tid);
        } else {
            fwd_round<LOGB, R, S0, T>(ar, tw, b, c, SmemLoad<V>{s}, SmemStore<V>{s}, tid);
            sync();
            fwd_rest<LOGB, LOGE, T, A, S0 + R>(s, ar, tw, b, c, last, sync, tid);
        }
    }
}

// All forward rounds of a block: first round loads with `first`, last round
// stores with `last`, the rest go through shared memory `s`. `after_first`
// runs once the first round's inputs are consumed (e.g. to start loading the
// next transform's inputs into the same registers).
template <int LOGB, int LOGE, int T, class A, class First, class Last, class Hook = NoHook, class Hook2 = NoHook>
__device__ __forceinline__ void fwd_block(typename A::V* s, const A& ar, const typename A::TW* tw, int b, int c,
                                          First first, Last last, Hook after_first = Hook{}, Hook2 after_sync = Hook2{}) {
    using V = typename A::V;
    constexpr int R0 = round_size(LOGB, LOGE, 0);
    if constexpr (R0 >= LOGB) {
        fwd_round<LOGB, R0, 0, T>(ar, tw, b, c, first, last, threadIdx.x);
        after_first();
    } else {
        fwd_round<LOGB, R0, 0, T>(ar, tw, b, c, first, SmemStore<V>{s}, threadIdx.x);
        after_first();
        __syncthreads();
        after_sync();  // every thread is past the first round (its inputs are consumed)
        using SP = Split<LOGB, LOGE, T>;
        if constexpr (SP::on) {
            const int g = threadIdx.x / SP::TG, lt = threadIdx.x % SP::TG;
            constexpr int BL = 1 << SP::LB;
            fwd_rest<SP::LB, LOGE, SP::TG, A, 0>(
                s + g * BL, ar, tw, (b << R0) + g, c + R0,
                [&](int i, V v, int uu, int k) { last(g * BL + i, v, uu, k); }, [g] { group_sync(g, SP::TG); }, lt);
        } else {
            fwd_rest<LOGB, LOGE, T, A, R0>(s, ar, tw, b, c, last, [] { __syncthreads(); }, threadIdx.x);
        }
    }
}

// Block position of the calling thread's unit slot `uu` in the last forward
// round (whose units are runs of 2^RL consecutive words).
template <int LOGB, int LOGE, int T>
__device__ __forceinline__ int fwd_last_base(int uu) {
    constexpr int RL = LOGB - last_round_start(LOGB, LOGE);
    using SP = Split<LOGB, LOGE, T>;
    if constexpr (SP::on && round_size(LOGB, LOGE, 0) < LOGB) {
        const int g = threadIdx.x / SP::TG, lt = threadIdx.x % SP::TG;
        return (g << SP::LB) + ((lt + uu * SP::TG) << RL);
    } else {
        return (static_cast<int>(threadIdx.x) + uu * T) << RL;
    }
}

// Inverse round: stages S0+R-1 down to S0.
template <int LOGB, int R, int S0, int T, class A, class Load, class Store>
__device__ __forceinline__ void inv_round(const A& ar, const typename A::TW* __restrict__ tw, int b, int c, Load load,
                                          Store store, int tid) {
    using V = typename A::V;
    constexpr int B = 1 << LOGB, G = B >> S0, STRIDE = G >> R, E = 1 << R, UNITS = B >> R;
    constexpr int PER = (UNITS + T - 1) / T;
#pragma unroll
    for (int uu = 0; uu < PER; ++uu) {
        const int u = tid + uu * T;
        if (UNITS % T != 0 && u >= UNITS) break;
        const int grp = u / STRIDE, col = u % STRIDE;
        const int base = grp * G + col;
        const int sb = swz(base);
        V x[E];
#pragma unroll
        for (int k = 0; k < E; ++k) {
            if constexpr (std::is_same<Load, SmemLoad<V>>::value) x[k] = load.s[sb ^ swz(k * STRIDE)];
            else x[k] = load(base + k * STRIDE);
        }
#pragma unroll
        for (int rho = R - 1; rho >= 0; --rho) {
            const int half = E >> (rho + 1);
            const int tbase = (1 << (c + S0 + rho)) + (b << (S0 + rho)) + (grp << rho);
#pragma unroll
            for (int blk = 0; blk < (1 << rho); ++blk) {
                const typename A::TW w = tw[tbase + blk];
#pragma unroll
                for (int kk = 0; kk < half; ++kk) ar.gs(x[blk * 2 * half + kk], x[blk * 2 * half + kk + half], w);
            }
        }
#pragma unroll
        for (int k = 0; k < E; ++k) {
            ar.round_end_inv(x[k]);
            if constexpr (std::is_same<Store, SmemStore<V>>::value) store.s[sb ^ swz(k * STRIDE)] = x[k];
            else store(base + k * STRIDE, x[k], uu, k);
        }
    }
}

// Inverse rounds S0 .. of a (sub-)block, highest S0 first; the round with the
// highest S0 loads with `first`, the S0 = 0 round stores with `last` (or into
// `s` when STORE_LAST is false, for a caller that continues the transform).
template <int LOGB, int LOGE, int T, class A, int S0, class First, class Last, class Sync>
__device__ __forceinline__ void inv_rest(typename A::V* s, const A& ar, const typename A::TW* tw, int b, int c,
                                         First first, Last last, Sync sync, int tid) {
    using V = typename A::V;
    if constexpr (S0 < LOGB) {
        constexpr int R = round_size(LOGB, LOGE, S0);
        constexpr bool runs_first = S0 + R >= LOGB, runs_last = S0 == 0;
        inv_rest<LOGB, LOGE, T, A, S0 + R>(s, ar, tw, b, c, first, last, sync, tid);
        if constexpr (runs_first && runs_last) {
            inv_round<LOGB, R, S0, T>(ar, tw, b, c, first, last, tid);
        } else if constexpr (runs_first) {
            inv_round<LOGB, R, S0, T>(ar, tw, b, c, first, SmemStore<V>{s}, tid);
            sync();
        } else if constexpr (runs_last) {
            inv_round<LOGB, R, S0, T>(ar, tw, b, c, SmemLoad<V>{s}, last, tid);
        } else {
            inv_round<LOGB, R, S0, T>(ar, tw, b, c, SmemLoad<V>{s}, SmemStore<V>{s}, tid);
            sync();
        }
    }
}

// All inverse rounds: the forward decomposition traversed backwards; the
// round with the highest S0 runs first and loads with `first`, the S0 = 0
// round runs last and stores with `last`. With the group split the rounds
// above R0 run per sub-block (named barriers), then one CTA barrier, then the
// global S0 = 0 round.
template <int LOGB, int LOGE, int T, class A, class First, class Last>
__device__ __forceinline__ void inv_block(typename A::V* s, const A& ar, const typename A::TW* tw, int b, int c,
                                          First first, Last last) {
    using V = typename A::V;
    using SP = Split<LOGB, LOGE, T>;
    if constexpr (SP::on) {
        constexpr int R0 = SP::R0, BL = 1 << SP::LB;
        const int g = threadIdx.x / SP::TG, lt = threadIdx.x % SP::TG;
        inv_rest<SP::LB, LOGE, SP::TG, A, 0>(
            s + g * BL, ar, tw, (b << R0) + g, c + R0, [&](int i) { return first(g * BL + i); }, SmemStore<V>{s + g * BL},
            [g] { group_sync(g, SP::TG); }, lt);
        __syncthreads();
        inv_round<LOGB, R0, 0, T>(ar, tw, b, c, SmemLoad<V>{s}, last, threadIdx.x);
    } else {
        inv_rest<LOGB, LOGE, T, A, 0>(s, ar, tw, b, c, first, last, [] { __syncthreads(); }, threadIdx.x);
    }
}

// ---- mbarrier / bulk-copy helpers (cp.async.bulk into shared memory)
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(b)));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    asm volatile(
        "{.reg .pred P1;\n"
        "WAIT_%=: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;}" ::"r"(smem_addr(b)),
        "r"(parity)
        : "memory");
}
// one bulk copy of `bytes` (multiple of 16) from global into shared memory,
// completing on `bar`; the caller has ordered earlier generic accesses to dst
// (barrier) -- the proxy fence makes them visible to the async proxy
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("{.reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;}" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}

// Limbs whose prime fits the FP64 path.
__device__ __forceinline__ bool fp_limb(u64 q) { return q < (1ull << 42); }

}  // namespace ntt
}  // namespace hecnn_b200
