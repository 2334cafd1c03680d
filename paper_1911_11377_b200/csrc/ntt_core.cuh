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
// inverse GS with psi^-bitrev(2^s + i); lazy ranges [0,4q) forward and
// [0,2q) inverse, made canonical by the caller's epilogue.
#pragma once
#include "kernels.hpp"

namespace hecnn_b200 {
namespace ntt {

__device__ __forceinline__ int swz(int i) {
    return i ^ static_cast<int>((0x1eb4d278963c5af0ull >> (4 * ((i >> 4) & 15))) & 15);
}

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

__host__ __device__ constexpr int ceil_div(int a, int b) { return (a + b - 1) / b; }
// Balanced split of the remaining LOGB - s stages into rounds of <= LOGE.
__host__ __device__ constexpr int round_size(int LOGB, int LOGE, int s) {
    return ceil_div(LOGB - s, ceil_div(LOGB - s, LOGE));
}
// Stage index where the last round starts.
__host__ __device__ constexpr int last_round_start(int LOGB, int LOGE, int s = 0) {
    return s + round_size(LOGB, LOGE, s) >= LOGB ? s : last_round_start(LOGB, LOGE, s + round_size(LOGB, LOGE, s));
}

struct SmemLoad {
    const u64* s;
    __device__ u64 operator()(int idx) const { return s[swz(idx)]; }
};
struct SmemStore {
    u64* s;
    __device__ void operator()(int idx, u64 v, int, int) const { s[swz(idx)] = v; }
};

// Forward round: block-local stages S0..S0+R-1; global stage = c + local;
// `b` is the block index inside the N-point transform (twiddle offset).
template <int LOGB, int R, int S0, int T, class Load, class Store>
__device__ __forceinline__ void fwd_round(const ulonglong2* __restrict__ tw, u64 q, int b, int c, Load load,
                                          Store store) {
    constexpr int B = 1 << LOGB, G = B >> S0, STRIDE = G >> R, E = 1 << R, UNITS = B >> R;
    constexpr int PER = (UNITS + T - 1) / T;
    const u64 two_q = q << 1;
#pragma unroll
    for (int uu = 0; uu < PER; ++uu) {
        const int u = threadIdx.x + uu * T;
        if (UNITS % T != 0 && u >= UNITS) break;
        const int grp = u / STRIDE, col = u % STRIDE;
        const int base = grp * G + col;
        u64 x[E];
#pragma unroll
        for (int k = 0; k < E; ++k) x[k] = load(base + k * STRIDE);
#pragma unroll
        for (int rho = 0; rho < R; ++rho) {
            const int half = E >> (rho + 1);
            const int tbase = (1 << (c + S0 + rho)) + (b << (S0 + rho)) + (grp << rho);
#pragma unroll
            for (int blk = 0; blk < (1 << rho); ++blk) {
                const ulonglong2 w = tw[tbase + blk];
#pragma unroll
                for (int kk = 0; kk < half; ++kk)
                    ct_butterfly(x[blk * 2 * half + kk], x[blk * 2 * half + kk + half], w, q, two_q);
            }
        }
#pragma unroll
        for (int k = 0; k < E; ++k) store(base + k * STRIDE, x[k], uu, k);
    }
}

// All forward rounds of a block: first round loads with `first`, last round
// stores with `last`, the rest go through shared memory `s`.
template <int LOGB, int LOGE, int T, int S0 = 0, class First, class Last>
__device__ __forceinline__ void fwd_block(u64* s, const ulonglong2* tw, u64 q, int b, int c, First first, Last last) {
    if constexpr (S0 < LOGB) {
        constexpr int R = round_size(LOGB, LOGE, S0);
        constexpr bool is_first = S0 == 0, is_last = S0 + R >= LOGB;
        if constexpr (is_first && is_last) {
            fwd_round<LOGB, R, S0, T>(tw, q, b, c, first, last);
        } else if constexpr (is_first) {
            fwd_round<LOGB, R, S0, T>(tw, q, b, c, first, SmemStore{s});
            __syncthreads();
        } else if constexpr (is_last) {
            fwd_round<LOGB, R, S0, T>(tw, q, b, c, SmemLoad{s}, last);
        } else {
            fwd_round<LOGB, R, S0, T>(tw, q, b, c, SmemLoad{s}, SmemStore{s});
            __syncthreads();
        }
        fwd_block<LOGB, LOGE, T, S0 + R>(s, tw, q, b, c, first, last);
    }
}

// Inverse round: stages S0+R-1 down to S0.
template <int LOGB, int R, int S0, int T, class Load, class Store>
__device__ __forceinline__ void inv_round(const ulonglong2* __restrict__ tw, u64 q, int b, int c, Load load,
                                          Store store) {
    constexpr int B = 1 << LOGB, G = B >> S0, STRIDE = G >> R, E = 1 << R, UNITS = B >> R;
    constexpr int PER = (UNITS + T - 1) / T;
    const u64 two_q = q << 1;
#pragma unroll
    for (int uu = 0; uu < PER; ++uu) {
        const int u = threadIdx.x + uu * T;
        if (UNITS % T != 0 && u >= UNITS) break;
        const int grp = u / STRIDE, col = u % STRIDE;
        const int base = grp * G + col;
        u64 x[E];
#pragma unroll
        for (int k = 0; k < E; ++k) x[k] = load(base + k * STRIDE);
#pragma unroll
        for (int rho = R - 1; rho >= 0; --rho) {
            const int half = E >> (rho + 1);
            const int tbase = (1 << (c + S0 + rho)) + (b << (S0 + rho)) + (grp << rho);
#pragma unroll
            for (int blk = 0; blk < (1 << rho); ++blk) {
                const ulonglong2 w = tw[tbase + blk];
#pragma unroll
                for (int kk = 0; kk < half; ++kk)
                    gs_butterfly(x[blk * 2 * half + kk], x[blk * 2 * half + kk + half], w, q, two_q);
            }
        }
#pragma unroll
        for (int k = 0; k < E; ++k) store(base + k * STRIDE, x[k], uu, k);
    }
}

// All inverse rounds: the forward decomposition traversed backwards; the
// round with the highest S0 runs first and loads with `first`, the S0 = 0
// round runs last and stores with `last`.
template <int LOGB, int LOGE, int T, int S0 = 0, class First, class Last>
__device__ __forceinline__ void inv_block(u64* s, const ulonglong2* tw, u64 q, int b, int c, First first, Last last) {
    if constexpr (S0 < LOGB) {
        constexpr int R = round_size(LOGB, LOGE, S0);
        constexpr bool runs_first = S0 + R >= LOGB, runs_last = S0 == 0;
        inv_block<LOGB, LOGE, T, S0 + R>(s, tw, q, b, c, first, last);
        if constexpr (runs_first && runs_last) {
            inv_round<LOGB, R, S0, T>(tw, q, b, c, first, last);
        } else if constexpr (runs_first) {
            inv_round<LOGB, R, S0, T>(tw, q, b, c, first, SmemStore{s});
            __syncthreads();
        } else if constexpr (runs_last) {
            inv_round<LOGB, R, S0, T>(tw, q, b, c, SmemLoad{s}, last);
        } else {
            inv_round<LOGB, R, S0, T>(tw, q, b, c, SmemLoad{s}, SmemStore{s});
            __syncthreads();
        }
    }
}

}  // namespace ntt
}  // namespace hecnn_b200
