// Batched negacyclic NTT / INTT over RNS limbs (K1/K2 in SURVEY.md §2.3).
//
// Transform: the reference's merged Cooley-Tukey forward NTT
// (NttTables::forward, ring.hpp:83-108), whose output is in bit-reversed
// evaluation order a_hat[j] = a(psi^(2*bitrev(j)+1)), and its exact inverse
// (NttTables::inverse, ring.hpp:110-137, Gentleman-Sande + n^-1). Twiddles are
// the reference's tables roots[m+i] = psi^bitrev(m+i) (Shoup pairs). The
// butterfly network is the same; only the schedule differs:
//
//   * one CTA per (poly, limb, block); a block of 2^LOGB words lives in
//     shared memory (<= 128 KB),
//   * stages are grouped into rounds of up to 4; in a round each thread holds
//     2^R words in registers and runs R butterfly stages on them, so shared
//     memory is touched once per round, not once per stage,
//   * shared-memory addresses use a GF(2)-linear XOR swizzle chosen (by
//     exhaustive search) so every round's access pattern is bank-conflict free,
//   * for N > 2^13 the first (forward) / last (inverse) LOGN-13 stages run in a
//     separate column pass over HBM, leaving 2^13-word independent blocks.
//
// Values stay lazily reduced ([0,4q) forward, [0,2q) inverse) and are made
// canonical at the end, so results are word-identical to the CPU reference.

#include <algorithm>
#include <stdexcept>

#include "ntt_core.cuh"

namespace hecnn_b200 {

namespace {

using ntt::ct_butterfly;
using ntt::gs_butterfly;

// Block kernels: blockIdx.x = (poly * nblocks + block); limb = poly % limbs.
// The first forward round reads HBM and the last round writes HBM directly
// (canonical values); the inverse likewise, with n^-1 folded into the store.
template <int LOGN, int LOGB, int LOGE, int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) k_ntt_fwd_block(DevRing R, const u64* src, u64* dst, int limbs) {
    extern __shared__ u64 smem[];
    constexpr int C = LOGN - LOGB;
    const long long cta = blockIdx.x;
    const long long poly = cta >> C;
    const int b = static_cast<int>(cta & ((1 << C) - 1));
    const int limb = static_cast<int>(poly % limbs);
    const u64 q = R.mod[limb].q;
    // src may equal dst: every element is read in the first round and written
    // in the last, with barriers in between
    const long long off = (poly << LOGN) + (static_cast<long long>(b) << LOGB);
    const u64* gi = src + off;
    u64* g = dst + off;
    const long long toff = static_cast<long long>(limb) << LOGN;
    if (ntt::fp_limb(q)) {
        const ntt::FpArith ar{static_cast<double>(q), R.inv_q[limb]};
        ntt::fwd_block<LOGB, LOGE, THREADS>(
            reinterpret_cast<double*>(smem), ar, R.fwd_f + toff, b, C, [=](int i) { return ntt::to_fp(gi[i]); },
            [=](int i, double v, int, int) { g[i] = ntt::fcanon(v, ar.q, ar.qinv); });
    } else {
        const ntt::IntArith ar{q, q << 1};
        ntt::fwd_block<LOGB, LOGE, THREADS>(
            smem, ar, R.fwd + toff, b, C, [=](int i) { return gi[i]; },
            [=](int i, u64 v, int, int) { g[i] = reduce_4q(v, q); });
    }
}

template <int LOGN, int LOGB, int LOGE, int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) k_ntt_inv_block(DevRing R, u64* __restrict__ data, int limbs) {
    extern __shared__ u64 smem[];
    constexpr int C = LOGN - LOGB;
    const long long cta = blockIdx.x;
    const long long poly = cta >> C;
    const int b = static_cast<int>(cta & ((1 << C) - 1));
    const int limb = static_cast<int>(poly % limbs);
    const u64 q = R.mod[limb].q;
    u64* g = data + (poly << LOGN) + (static_cast<long long>(b) << LOGB);
    const long long toff = static_cast<long long>(limb) << LOGN;
    if (ntt::fp_limb(q)) {
        const ntt::FpArith ar{static_cast<double>(q), R.inv_q[limb]};
        const double ni = R.n_inv_f[limb];
        ntt::inv_block<LOGB, LOGE, THREADS>(
            reinterpret_cast<double*>(smem), ar, R.inv_f + toff, b, C, [=](int i) { return ntt::to_fp(g[i]); },
            [=](int i, double v, int, int) {
                if constexpr (C == 0) v = ntt::fmodmul(v, ni, ar.q, ar.qinv);
                g[i] = ntt::fcanon(v, ar.q, ar.qinv);  // [0,q) is inside the column pass's [0,2q) contract
            });
    } else {
        const ntt::IntArith ar{q, q << 1};
        const ulonglong2 ni = R.n_inv[limb];
        ntt::inv_block<LOGB, LOGE, THREADS>(
            smem, ar, R.inv + toff, b, C, [=](int i) { return g[i]; },
            [=](int i, u64 v, int, int) {
                if constexpr (C == 0) g[i] = reduce_2q(mul_shoup_lazy(v, ni.x, ni.y, q), q);
                else g[i] = v;  // [0,2q); the column pass finishes
            });
    }
}

// Inverse NTT of limbs [limb0, limb0 + nsel) of every poly group
// (groups = ciphertext components, `limbs` limbs each), single block pass
// (N <= 2^LOGB). RESCALE: the last round stores rescale_poly's output
// (ring.hpp:419-442) for limb i < L = limbs - 1 straight into `out`
// ([groups][limbs - 1][n]), reading the top limb's coefficients, which a
// previous launch (RESCALE = false, limb0 = L) transformed in place.
template <int LOGN, int LOGE, int THREADS, int MINB, bool RESCALE>
__global__ void __launch_bounds__(THREADS, MINB) k_ntt_inv_sel(DevRing R, u64* __restrict__ data, u64* __restrict__ out,
                                                               int limbs, int limb0, int nsel,
                                                               const u64* __restrict__ add0) {
    extern __shared__ u64 smem[];
    const long long cta = blockIdx.x;
    const long long grp = cta / nsel;
    const int limb = limb0 + static_cast<int>(cta % nsel);
    const u64 q = R.mod[limb].q;
    u64* g = data + ((grp * limbs + limb) << LOGN);
    const long long toff = static_cast<long long>(limb) << LOGN;
    const int L = limbs - 1;
    const u64* top = data + ((grp * limbs + L) << LOGN);
    u64* o = out + ((grp * L + limb) << LOGN);
    auto store = [=](int i, u64 c) {
        if constexpr (RESCALE) {
            const ModConst m = R.mod[limb];
            const u64 vt = top[i];
            u64 centred = reduce_near(vt, m);
            if (vt > (R.mod[L].q >> 1)) centred = sub_mod(centred, R.p_mod[L * R.limbs + limb], m.q);
            const ulonglong2 inv = R.inv_dropped[L * R.limbs + limb];
            if (limb == 0 && add0) c = add_mod(c, add0[(grp << LOGN) + i], m.q);
            o[i] = mul_shoup(sub_mod(c, centred, m.q), inv.x, inv.y, m.q);
        } else {
            g[i] = c;
        }
    };
    if (ntt::fp_limb(q)) {
        const ntt::FpArith ar{static_cast<double>(q), R.inv_q[limb]};
        const double ni = R.n_inv_f[limb];
        if constexpr (RESCALE) {
            // the rescale on the FP64 pipe too: (c - centre(top)) p_L^-1 with exact
            // FP64 modmuls (|x - cen| < 3q); the canonical result is the integer path's
            const u64 qtop_half = R.mod[L].q >> 1;
            const double pm = ntt::to_fp(R.p_mod[L * R.limbs + limb]);
            const double invf = ntt::to_fp(R.inv_dropped[L * R.limbs + limb].x);
            ntt::inv_block<LOGN, LOGE, THREADS>(
                reinterpret_cast<double*>(smem), ar, R.inv_f + toff, 0, 0, [=](int i) { return ntt::to_fp(g[i]); },
                [=](int i, double v, int, int) {
                    const double x = ntt::fmodmul(v, ni, ar.q, ar.qinv);
                    const u64 vt = top[i];
                    double cen = ntt::fcentre(ntt::to_fp(vt), ar.q, ar.qinv);
                    if (vt > qtop_half) cen -= pm;
                    o[i] = ntt::fcanon(ntt::fmodmul(x - cen, invf, ar.q, ar.qinv), ar.q, ar.qinv);
                });
        } else {
            ntt::inv_block<LOGN, LOGE, THREADS>(
                reinterpret_cast<double*>(smem), ar, R.inv_f + toff, 0, 0, [=](int i) { return ntt::to_fp(g[i]); },
                [=](int i, double v, int, int) { store(i, ntt::fcanon(ntt::fmodmul(v, ni, ar.q, ar.qinv), ar.q, ar.qinv)); });
        }
    } else {
        const ntt::IntArith ar{q, q << 1};
        const ulonglong2 ni = R.n_inv[limb];
        ntt::inv_block<LOGN, LOGE, THREADS>(
            smem, ar, R.inv + toff, 0, 0, [=](int i) { return g[i]; },
            [=](int i, u64 v, int, int) { store(i, reduce_2q(mul_shoup_lazy(v, ni.x, ni.y, q), q)); });
    }
}

// d2 = INTT(x1 * y1) (CkksEngine::mul tensor step ckks.hpp:320-327 then
// the relinearisation's to_coeff, :611): blockIdx.x = (poly * nblocks + b)
// over the output polys [count][limbs]; the operands are the component-1
// rows of the forward-transformed ciphertexts.
template <int LOGN, int LOGB, int LOGE, int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) k_ntt_inv_prod(DevRing R, const u64* __restrict__ x,
                                                                const u64* __restrict__ y, u64* __restrict__ out,
                                                                int limbs) {
    extern __shared__ u64 smem[];
    constexpr int C = LOGN - LOGB;
    const long long cta = blockIdx.x;
    const long long poly = cta >> C;
    const int b = static_cast<int>(cta & ((1 << C) - 1));
    const int limb = static_cast<int>(poly % limbs);
    const long long ct = poly / limbs;
    const u64 q = R.mod[limb].q;
    const long long boff = static_cast<long long>(b) << LOGB;
    const long long in_off = (((ct * 2 + 1) * limbs + limb) << LOGN) + boff;
    const u64* xa = x + in_off;
    const u64* ya = y + in_off;
    u64* g = out + (poly << LOGN) + boff;
    const long long toff = static_cast<long long>(limb) << LOGN;
    if (ntt::fp_limb(q)) {
        const ntt::FpArith ar{static_cast<double>(q), R.inv_q[limb]};
        const double ni = R.n_inv_f[limb];
        ntt::inv_block<LOGB, LOGE, THREADS>(
            reinterpret_cast<double*>(smem), ar, R.inv_f + toff, b, C,
            [=](int i) { return ntt::fmodmul(ntt::to_fp(xa[i]), ntt::to_fp(ya[i]), ar.q, ar.qinv); },
            [=](int i, double v, int, int) {
                if constexpr (C == 0) v = ntt::fmodmul(v, ni, ar.q, ar.qinv);
                g[i] = ntt::fcanon(v, ar.q, ar.qinv);
            });
    } else {
        const ntt::IntArith ar{q, q << 1};
        const ulonglong2 ni = R.n_inv[limb];
        const ModConst m = R.mod[limb];
        ntt::inv_block<LOGB, LOGE, THREADS>(
            smem, ar, R.inv + toff, b, C, [=](int i) { return mul_mod(xa[i], ya[i], m); },
            [=](int i, u64 v, int, int) {
                if constexpr (C == 0) g[i] = reduce_2q(mul_shoup_lazy(v, ni.x, ni.y, q), q);
                else g[i] = v;
            });
    }
}

// Column passes for N > 2^LOGB: the C stages that couple the 2^C blocks.
// Thread = one column (poly, col), elements col + k * (N >> C).
template <int LOGN, int C>
__global__ void __launch_bounds__(256) k_ntt_fwd_cols(DevRing R, const u64* src, u64* data, int limbs, long long total) {
    constexpr int E = 1 << C, STRIDE = 1 << (LOGN - C);
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= total) return;
    const long long poly = t >> (LOGN - C);
    const int col = static_cast<int>(t & (STRIDE - 1));
    const int limb = static_cast<int>(poly % limbs);
    const u64 q = R.mod[limb].q, two_q = q << 1;
    const ulonglong2* tw = R.fwd + (static_cast<long long>(limb) << LOGN);
    const u64* gi = src + (poly << LOGN) + col;
    u64* g = data + (poly << LOGN) + col;
    u64 x[E];
#pragma unroll
    for (int k = 0; k < E; ++k) x[k] = gi[static_cast<long long>(k) * STRIDE];
#pragma unroll
    for (int rho = 0; rho < C; ++rho) {
        const int half = E >> (rho + 1);
#pragma unroll
        for (int blk = 0; blk < (1 << rho); ++blk) {
            const ulonglong2 w = tw[(1 << rho) + blk];
#pragma unroll
            for (int kk = 0; kk < half; ++kk) ct_butterfly(x[blk * 2 * half + kk], x[blk * 2 * half + kk + half], w, q, two_q);
        }
    }
#pragma unroll
    for (int k = 0; k < E; ++k) g[static_cast<long long>(k) * STRIDE] = x[k];
}

template <int LOGN, int C>
__global__ void __launch_bounds__(256) k_ntt_inv_cols(DevRing R, u64* __restrict__ data, int limbs, long long total) {
    constexpr int E = 1 << C, STRIDE = 1 << (LOGN - C);
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= total) return;
    const long long poly = t >> (LOGN - C);
    const int col = static_cast<int>(t & (STRIDE - 1));
    const int limb = static_cast<int>(poly % limbs);
    const u64 q = R.mod[limb].q, two_q = q << 1;
    const ulonglong2* tw = R.inv + (static_cast<long long>(limb) << LOGN);
    u64* g = data + (poly << LOGN) + col;
    u64 x[E];
#pragma unroll
    for (int k = 0; k < E; ++k) x[k] = g[static_cast<long long>(k) * STRIDE];
#pragma unroll
    for (int rho = C - 1; rho >= 0; --rho) {
        const int half = E >> (rho + 1);
#pragma unroll
        for (int blk = 0; blk < (1 << rho); ++blk) {
            const ulonglong2 w = tw[(1 << rho) + blk];
#pragma unroll
            for (int kk = 0; kk < half; ++kk) gs_butterfly(x[blk * 2 * half + kk], x[blk * 2 * half + kk + half], w, q, two_q);
        }
    }
    const ulonglong2 ni = R.n_inv[limb];
#pragma unroll
    for (int k = 0; k < E; ++k) g[static_cast<long long>(k) * STRIDE] = reduce_2q(mul_shoup_lazy(x[k], ni.x, ni.y, q), q);
}

template <class K>
void set_smem(K kernel, int bytes) {
    smem_opt_in(kernel, bytes);
}

#ifndef HECNN_NTT_LOGE
#define HECNN_NTT_LOGE 3
#endif
#ifndef HECNN_NTT_MAXT
#define HECNN_NTT_MAXT 512
#endif
#ifndef HECNN_NTT_MINB
#define HECNN_NTT_MINB 2
#endif

template <int LOGN>
struct NttPlan {
#ifndef HECNN_NTT_MAXLOGB
#define HECNN_NTT_MAXLOGB 14
#endif
    static constexpr int LOGB = LOGN <= HECNN_NTT_MAXLOGB ? LOGN : 13;
    static constexpr int C = LOGN - LOGB;
    static constexpr int LOGE = LOGB >= 8 ? HECNN_NTT_LOGE : 3;
    static constexpr int UNITS = (1 << LOGB) >> LOGE;
    static constexpr int THREADS = UNITS >= HECNN_NTT_MAXT ? HECNN_NTT_MAXT : (UNITS >= 32 ? UNITS : 32);
    // two CTAs per SM only when two blocks' shared memory fits (2^14 words: one per SM)
    static constexpr int MINB = THREADS >= 256 && (2 << LOGB) * 8 <= 227 * 1024 ? HECNN_NTT_MINB : 1;
};

template <int LOGN>
void run_forward(const DevRing& R, const u64* src, u64* data, int limbs, std::size_t polys, const Launch& L) {
    using P = NttPlan<LOGN>;
    if constexpr (P::C > 0) {
        long long total = static_cast<long long>(polys) << (LOGN - P::C);
        L.begin("k_ntt_fwd_cols", double(polys) * (1 << (LOGN - 1)) * P::C, 16.0 * polys * (1 << LOGN));
        k_ntt_fwd_cols<LOGN, P::C><<<static_cast<unsigned>((total + 255) / 256), 256, 0, L.stream>>>(R, src, data, limbs, total);
        L.count();
        src = data;  // the block pass continues in place
    }
    auto kern = k_ntt_fwd_block<LOGN, P::LOGB, P::LOGE, P::THREADS, P::MINB>;
    const int smem = (1 << P::LOGB) * 8;
    set_smem(kern, smem);
    L.begin("k_ntt_fwd_block", double(polys) * (1 << (LOGN - 1)) * P::LOGB, 16.0 * polys * (1 << LOGN));
    kern<<<static_cast<unsigned>(polys << P::C), P::THREADS, smem, L.stream>>>(R, src, data, limbs);
    L.count();
}

template <int LOGN>
void run_inverse(const DevRing& R, u64* data, int limbs, std::size_t polys, const Launch& L) {
    using P = NttPlan<LOGN>;
    auto kern = k_ntt_inv_block<LOGN, P::LOGB, P::LOGE, P::THREADS, P::MINB>;
    const int smem = (1 << P::LOGB) * 8;
    set_smem(kern, smem);
    L.begin("k_ntt_inv_block", double(polys) * (1 << (LOGN - 1)) * P::LOGB, 16.0 * polys * (1 << LOGN));
    kern<<<static_cast<unsigned>(polys << P::C), P::THREADS, smem, L.stream>>>(R, data, limbs);
    L.count();
    if constexpr (P::C > 0) {
        long long total = static_cast<long long>(polys) << (LOGN - P::C);
        L.begin("k_ntt_inv_cols", double(polys) * (1 << (LOGN - 1)) * P::C, 16.0 * polys * (1 << LOGN));
        k_ntt_inv_cols<LOGN, P::C><<<static_cast<unsigned>((total + 255) / 256), 256, 0, L.stream>>>(R, data, limbs, total);
        L.count();
    }
}

template <int LOGN>
void run_inverse_product(const DevRing& R, const u64* x, const u64* y, u64* d2, int limbs, std::size_t polys,
                         const Launch& L) {
    using P = NttPlan<LOGN>;
    auto kern = k_ntt_inv_prod<LOGN, P::LOGB, P::LOGE, P::THREADS, P::MINB>;
    const int smem = (1 << P::LOGB) * 8;
    set_smem(kern, smem);
    L.begin("k_ntt_inv_block", double(polys) * ((1 << (LOGN - 1)) * P::LOGB + (1 << LOGN)), 24.0 * polys * (1 << LOGN));
    kern<<<static_cast<unsigned>(polys << P::C), P::THREADS, smem, L.stream>>>(R, x, y, d2, limbs);
    L.count();
    if constexpr (P::C > 0) {
        long long total = static_cast<long long>(polys) << (LOGN - P::C);
        L.begin("k_ntt_inv_cols", double(polys) * (1 << (LOGN - 1)) * P::C, 16.0 * polys * (1 << LOGN));
        k_ntt_inv_cols<LOGN, P::C><<<static_cast<unsigned>((total + 255) / 256), 256, 0, L.stream>>>(R, d2, limbs, total);
        L.count();
    }
}

template <bool FWD>
void dispatch(const DevRing& R, const u64* src, u64* data, int level, std::size_t count, const Launch& L) {
    const int limbs = level + 1;
    const std::size_t polys = count * static_cast<std::size_t>(limbs);
    if (polys == 0) return;
#define HECNN_NTT_CASE(LG)                                             \
    case LG:                                                          \
        if (FWD) run_forward<LG>(R, src, data, limbs, polys, L);      \
        else run_inverse<LG>(R, data, limbs, polys, L);               \
        break;
    switch (R.logn) {
        HECNN_NTT_CASE(3)
        HECNN_NTT_CASE(4)
        HECNN_NTT_CASE(5)
        HECNN_NTT_CASE(6)
        HECNN_NTT_CASE(7)
        HECNN_NTT_CASE(8)
        HECNN_NTT_CASE(9)
        HECNN_NTT_CASE(10)
        HECNN_NTT_CASE(11)
        HECNN_NTT_CASE(12)
        HECNN_NTT_CASE(13)
        HECNN_NTT_CASE(14)
        HECNN_NTT_CASE(15)
        HECNN_NTT_CASE(16)
        default: throw std::invalid_argument("ntt: ring degree outside 2^3..2^16 is not supported on the device");
    }
#undef HECNN_NTT_CASE
    check_launch(FWD ? "ntt_forward" : "ntt_inverse");
}

}  // namespace

void ntt_forward(const DevRing& R, u64* polys, int level, std::size_t count, const Launch& L) {
    dispatch<true>(R, polys, polys, level, count, L);
}

void ntt_forward_to(const DevRing& R, const u64* src, u64* dst, int level, std::size_t count, const Launch& L) {
    dispatch<true>(R, src, dst, level, count, L);
}

void ntt_inverse(const DevRing& R, u64* polys, int level, std::size_t count, const Launch& L) {
    dispatch<false>(R, polys, polys, level, count, L);
}

namespace {
template <int LOGN>
bool run_inverse_rescale(const DevRing& R, u64* d, u64* out, int limbs, std::size_t groups, const Launch& L,
                         const u64* add0) {
    using P = NttPlan<LOGN>;
    if constexpr (P::C > 0) {
        return false;
    } else {
        auto ktop = k_ntt_inv_sel<LOGN, P::LOGE, P::THREADS, P::MINB, false>;
        auto kres = k_ntt_inv_sel<LOGN, P::LOGE, P::THREADS, P::MINB, true>;
        const int smem = (1 << LOGN) * 8;
        set_smem(ktop, smem);
        set_smem(kres, smem);
        const double bfly = double(1 << (LOGN - 1)) * LOGN, nn = double(1 << LOGN);
        L.begin("k_ntt_inv_block", double(groups) * bfly, 16.0 * groups * nn);
        ktop<<<static_cast<unsigned>(groups), P::THREADS, smem, L.stream>>>(R, d, out, limbs, limbs - 1, 1, nullptr);
        L.count();
        const std::size_t polys = groups * static_cast<std::size_t>(limbs - 1);
        L.begin("k_ntt_inv_rescale", double(polys) * (bfly + 2 * nn), 8.0 * nn * (2.0 * polys + groups));
        kres<<<static_cast<unsigned>(polys), P::THREADS, smem, L.stream>>>(R, d, out, limbs, 0, limbs - 1, add0);
        L.count();
        return true;
    }
}
}  // namespace

namespace {
template <int LOGN>
void run_inverse_limbs(const DevRing& R, u64* data, int limbs, int limb0, int nsel, std::size_t groups, const Launch& L,
                       const char* name) {
    using P = NttPlan<LOGN>;
    if constexpr (P::C > 0) {
        throw std::invalid_argument("ntt_inverse_limbs: ring degree above one block");
    } else {
        auto kern = k_ntt_inv_sel<LOGN, P::LOGE, P::THREADS, P::MINB, false>;
        const int smem = (1 << LOGN) * 8;
        set_smem(kern, smem);
        const std::size_t polys = groups * static_cast<std::size_t>(nsel);
        L.begin(name ? name : "k_ntt_inv_block", double(polys) * (1 << (LOGN - 1)) * LOGN, 16.0 * polys * (1 << LOGN));
        kern<<<static_cast<unsigned>(polys), P::THREADS, smem, L.stream>>>(R, data, data, limbs, limb0, nsel, nullptr);
        L.count();
    }
}
}  // namespace

void ntt_inverse_limbs(const DevRing& R, u64* data, int limbs, int limb0, int nsel, std::size_t groups, const Launch& L,
                       const char* name) {
    if (!groups || nsel <= 0) return;
#define HECNN_NTT_CASE(LG) \
    case LG: run_inverse_limbs<LG>(R, data, limbs, limb0, nsel, groups, L, name); break;
    switch (R.logn) {
        HECNN_NTT_CASE(3) HECNN_NTT_CASE(4) HECNN_NTT_CASE(5) HECNN_NTT_CASE(6) HECNN_NTT_CASE(7)
        HECNN_NTT_CASE(8) HECNN_NTT_CASE(9) HECNN_NTT_CASE(10) HECNN_NTT_CASE(11) HECNN_NTT_CASE(12)
        HECNN_NTT_CASE(13) HECNN_NTT_CASE(14) HECNN_NTT_CASE(15) HECNN_NTT_CASE(16)
        default: throw std::invalid_argument("ntt: ring degree outside 2^3..2^16 is not supported on the device");
    }
#undef HECNN_NTT_CASE
    check_launch("ntt_inverse_limbs");
}

bool ntt_inverse_rescale(const DevRing& R, u64* d, u64* out, int level, std::size_t groups, const Launch& L,
                         const u64* add0) {
    if (level < 1 || !groups) return false;
    bool done = false;
#define HECNN_NTT_CASE(LG) \
    case LG: done = run_inverse_rescale<LG>(R, d, out, level + 1, groups, L, add0); break;
    switch (R.logn) {
        HECNN_NTT_CASE(3) HECNN_NTT_CASE(4) HECNN_NTT_CASE(5) HECNN_NTT_CASE(6) HECNN_NTT_CASE(7)
        HECNN_NTT_CASE(8) HECNN_NTT_CASE(9) HECNN_NTT_CASE(10) HECNN_NTT_CASE(11) HECNN_NTT_CASE(12)
        HECNN_NTT_CASE(13) HECNN_NTT_CASE(14) HECNN_NTT_CASE(15) HECNN_NTT_CASE(16)
        default: return false;
    }
#undef HECNN_NTT_CASE
    check_launch("ntt_inverse_rescale");
    return done;
}

void ntt_inverse_product(const DevRing& R, const u64* x, const u64* y, u64* d2, int level, std::size_t count,
                         const Launch& L) {
    const int limbs = level + 1;
    const std::size_t polys = count * static_cast<std::size_t>(limbs);
    if (!polys) return;
#define HECNN_NTT_CASE(LG) \
    case LG: run_inverse_product<LG>(R, x, y, d2, limbs, polys, L); break;
    switch (R.logn) {
        HECNN_NTT_CASE(3) HECNN_NTT_CASE(4) HECNN_NTT_CASE(5) HECNN_NTT_CASE(6) HECNN_NTT_CASE(7)
        HECNN_NTT_CASE(8) HECNN_NTT_CASE(9) HECNN_NTT_CASE(10) HECNN_NTT_CASE(11) HECNN_NTT_CASE(12)
        HECNN_NTT_CASE(13) HECNN_NTT_CASE(14) HECNN_NTT_CASE(15) HECNN_NTT_CASE(16)
        default: throw std::invalid_argument("ntt: ring degree outside 2^3..2^16 is not supported on the device");
    }
#undef HECNN_NTT_CASE
    check_launch("ntt_inverse_product");
}

}  // namespace hecnn_b200
