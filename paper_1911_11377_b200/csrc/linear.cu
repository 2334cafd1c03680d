// Plaintext-weight x ciphertext layers (K8 in SURVEY.md §2.3).
//
// conv2d_encrypted (layers.hpp:174-211) and dense_encrypted (:269-293) are,
// per (component, limb, coefficient) column, an exact integer GEMM with a
// gather: y[pixel*OC + oc] = sum_k w[wrow(pixel,k)][oc] * x[src(pixel,k)]
// (mod q_i), followed by the bias on coefficient 0 of c0 and a rescale.
// mul_scalar_mac (ckks.hpp:448-465) does one Shoup multiply + add per tap;
// here a thread owns one column and a tile of OCT output channels, so each
// ciphertext word it loads feeds OCT multiply-accumulates (register reuse of
// the input across output channels), and the partial sums stay lazily
// reduced in [0, 2q). Modular sums are order independent, so the result is
// word-identical to the reference's sequential accumulation.

#include <algorithm>
#include <stdexcept>

#include "ntt_core.cuh"

namespace hecnn_b200 {

namespace {

constexpr int TPB = 256;
#ifndef HECNN_GM_TPB
#define HECNN_GM_TPB 256
#endif
#ifndef HECNN_GM_OCT
#define HECNN_GM_OCT 8
#endif
#ifndef HECNN_GM_TAPB
#define HECNN_GM_TAPB 4
#endif
#ifndef HECNN_GM_MINB
#define HECNN_GM_MINB 2
#endif
constexpr int GM_TPB = HECNN_GM_TPB;
constexpr int OCT = HECNN_GM_OCT;  // output channels per thread; weights are padded to 16
static_assert(16 % OCT == 0, "OCT must divide the weight padding");

constexpr int KCHUNK = 256;
constexpr int TAPB = HECNN_GM_TAPB;  // input words in flight per thread
#ifndef HECNN_GM_PG
#define HECNN_GM_PG 8
#endif
constexpr int PG = HECNN_GM_PG;  // pixels per CTA when all K taps fit one staged chunk

// One thread = one (component, limb, coefficient) column of OCT output
// channels, for a group of pixels. Tap k of every pixel uses weight row k, so
// when K <= KCHUNK the CTA stages the limb's weights for its OCT channels and
// the taps of all its pixels once, then runs the pixel loop out of shared
// memory; larger K streams chunks of KCHUNK taps for one pixel. The inner loop
// issues TAPB independent coalesced loads of input words, then OCT
// multiply-accumulates each against broadcast shared words. The grid is
// column-block major (column block slowest, channel tile fastest), so while
// one column block is in flight every input cell's slice of it stays in L2 and
// is reused by all pixels whose window covers it and by all channel tiles.
struct GmTile {
    long long cell_words, col;
    const u64* xc;
    int p_begin, p_end, oc0, i, limbs, comp, j, tpb;
    bool resident, live;
    u64 q;
    double qd, qinv;
};

template <bool SPLIT>
__device__ __forceinline__ void gm_body(const GatherMac& g, const GmTile& T, const ModConst& m, u64* __restrict__ y,
                                        unsigned char* s_raw, int (*s_src)[KCHUNK]) {
    auto s_w = reinterpret_cast<double2(*)[OCT]>(s_raw);
    auto s_ws = reinterpret_cast<ulonglong2(*)[OCT]>(s_raw);
    const u64 q = T.q, two_q = q << 1;
    const double qd = T.qd, qinv = T.qinv;
    const long long wbase = static_cast<long long>(T.i) * g.K;
    for (int p = T.p_begin; p < T.p_end; ++p) {
        // SPLIT: f00 = sum x0 w0, fm0 = sum x0 w1, fm1 = sum x1 w0, f11 = sum x1 w1
        double f00[OCT], fm0[OCT], fm1[OCT], f11[OCT];
        u64 s00[OCT];
#pragma unroll
        for (int o = 0; o < OCT; ++o) {
            if (SPLIT) f00[o] = fm0[o] = fm1[o] = f11[o] = 0.0;
            else s00[o] = 0;
        }
        for (int k0 = 0; k0 < g.K; k0 += KCHUNK) {
            const int kn = min(KCHUNK, g.K - k0);
            const int kpad = (kn + TAPB - 1) / TAPB * TAPB;  // taps kn..kpad: src -1, weight 0
            if (!T.resident || p == T.p_begin) {
                __syncthreads();
                for (int t = threadIdx.x; t < kpad * OCT; t += T.tpb) {
                    const int k = t / OCT, o = t % OCT;
                    const bool ok = k < kn;
                    const long long at = ok ? (wbase + k0 + k) * g.oc_pad + T.oc0 + o : 0;
                    if (SPLIT) {
                        const uint2 w = ok ? g.wsplit[at] : make_uint2(0, 0);
                        s_w[k][o] = make_double2(static_cast<double>(w.x), static_cast<double>(w.y));
                    } else {
                        s_ws[k][o] = ok ? g.weights[at] : make_ulonglong2(0, 0);
                    }
                }
                const int np = T.p_end - p;
                for (int t = threadIdx.x; t < np * kpad; t += T.tpb) {
                    const int pp = t / kpad, k = t - pp * kpad;
                    s_src[pp][k] = k < kn ? g.src[static_cast<long long>(p + pp) * g.K + k0 + k] : -1;
                }
                __syncthreads();
            }
            if (!T.live) continue;
            const int* ss = s_src[T.resident ? p - T.p_begin : 0];
            // invalid taps (s < 0, zero padding) load nothing and contribute 0
            for (int kb = 0; kb < kpad; kb += TAPB) {
                u64 v[TAPB];
#pragma unroll
                for (int u = 0; u < TAPB; ++u) {
                    const int s = ss[kb + u];
                    v[u] = s >= 0 ? __ldg(T.xc + s * T.cell_words) : 0;
                }
#pragma unroll
                for (int u = 0; u < TAPB; ++u) {
                    const int k = kb + u;
                    if (SPLIT) {
                        const double v0 = ntt::to_fp(v[u] & 0x1FFFFFull), v1 = ntt::to_fp(v[u] >> 21);
#pragma unroll
                        for (int o = 0; o < OCT; ++o) {
                            const double2 c = s_w[k][o];
                            f00[o] = fma(v0, c.x, f00[o]);
                            fm0[o] = fma(v0, c.y, fm0[o]);
                            fm1[o] = fma(v1, c.x, fm1[o]);
                            f11[o] = fma(v1, c.y, f11[o]);
                        }
                    } else {
#pragma unroll
                        for (int o = 0; o < OCT; ++o) {
                            const ulonglong2 c = s_ws[k][o];
                            const u64 t = s00[o] + mul_shoup_lazy(v[u], c.x, c.y, q);
                            s00[o] = t >= two_q ? t - two_q : t;
                        }
                    }
                }
            }
            if (SPLIT) {
#pragma unroll
                for (int o = 0; o < OCT; ++o) {
                    f00[o] = ntt::fcentre(f00[o], qd, qinv);
                    fm0[o] = ntt::fcentre(fm0[o], qd, qinv);
                    fm1[o] = ntt::fcentre(fm1[o], qd, qinv);
                    f11[o] = ntt::fcentre(f11[o], qd, qinv);
                }
            }
        }
        if (!T.live) continue;
        const ulonglong2 c21 = g.recomb[2 * T.i], c42 = g.recomb[2 * T.i + 1];
#pragma unroll
        for (int o = 0; o < OCT; ++o) {
            const int oc = T.oc0 + o;
            if (oc >= g.oc) break;
            u64 v;
            if (SPLIT) {
                const double t = f00[o] + ntt::fmodmul(fm0[o] + fm1[o], static_cast<double>(c21.x), qd, qinv) +
                                 ntt::fmodmul(f11[o], static_cast<double>(c42.x), qd, qinv);
                v = ntt::fcanon(t, qd, qinv);
            } else {
                v = reduce_2q(s00[o], q);
            }
            if (g.bias && T.comp == 0 && T.j == 0) v = add_mod(v, g.bias[static_cast<long long>(oc) * T.limbs + T.i], q);
            y[(static_cast<long long>(p) * g.out_stride_pixel + oc) * T.cell_words + T.col] = v;
        }
    }
}

__global__ void __launch_bounds__(GM_TPB, HECNN_GM_MINB) k_gather_mac(DevRing R, GatherMac g, const u64* __restrict__ x,
                                                                     u64* __restrict__ y, int level, int oc_tiles,
                                                                     int groups, int pg, int limb0, int nl) {
    // staged weights: split doubles (FP64 limbs) or (residue, shoup) (q0); one per CTA
    __shared__ __align__(16) unsigned char s_raw[KCHUNK * OCT * 16];
    __shared__ int s_src[PG][KCHUNK];
    GmTile T;
    T.limbs = level + 1;
    const long long poly_words = static_cast<long long>(T.limbs) * R.n;
    T.cell_words = 2 * poly_words;
    T.tpb = blockDim.x;  // <= n, so a CTA's columns share one limb
    const long long per_block = static_cast<long long>(groups) * oc_tiles;
    const long long bid = blockIdx.x;
    const long long cb = bid / per_block;
    const int rest = static_cast<int>(bid - cb * per_block);
    const int grp = rest / oc_tiles;
    T.oc0 = (rest - grp * oc_tiles) * OCT;
    T.p_begin = grp * pg;
    T.p_end = min(T.p_begin + pg, g.pixels);
    T.resident = g.K <= KCHUNK;  // host sets pg = 1 otherwise
    // cb -> (component, limb in [limb0, limb0 + nl), block of tpb coefficients)
    const int nb = R.n / T.tpb;
    const int rowc = static_cast<int>(cb / nb);
    const long long col0 = (rowc / nl) * poly_words + static_cast<long long>(limb0 + rowc % nl) * R.n + (cb % nb) * T.tpb;
    T.col = col0 + threadIdx.x;
    T.live = T.col < T.cell_words;
    T.comp = static_cast<int>(T.col / poly_words);
    T.i = static_cast<int>(((T.live ? T.col : col0) / R.n) % T.limbs);  // uniform when n >= TPB
    T.j = static_cast<int>(T.col % R.n);
    const ModConst m = R.mod[T.i];
    T.q = m.q;
    T.qd = static_cast<double>(T.q);
    T.qinv = R.inv_q[T.i];
    T.xc = x + (T.live ? T.col : 0);
    // q < 2^42: x, w split at bit 21 into exact doubles; every partial product
    // is < 2^42 and each accumulator sums at most KCHUNK of them (< 2^50), so
    // the FP64 pipe accumulates exactly; accumulators are centred mod q after
    // each chunk. The middle term uses two accumulators so no two dependent
    // FMAs are issued back to back. The 60-bit q0 limb uses lazy Shoup.
    if (ntt::fp_limb(T.q)) gm_body<true>(g, T, m, y, s_raw, s_src);
    else gm_body<false>(g, T, m, y, s_raw, s_src);
}

// avg_pool2d_encrypted (layers.hpp:213-239): sum of the window, times
// round(Delta / area) (one Shoup multiply), rescale done by the caller.
__global__ void k_pool(DevRing R, const u64* __restrict__ x, const int* __restrict__ srcs, int taps,
                       const ulonglong2* __restrict__ w, u64* __restrict__ y, int level, int accumulate) {
    const int limbs = level + 1;
    const long long poly_words = static_cast<long long>(limbs) * R.n;
    const long long cell_words = 2 * poly_words;
    const long long col = static_cast<long long>(blockIdx.x) * TPB + threadIdx.x;
    if (col >= cell_words) return;
    const int i = static_cast<int>((col / R.n) % limbs);
    const long long cell = blockIdx.y;
    const u64 q = R.mod[i].q;
    u64 s = accumulate ? y[cell * cell_words + col] : 0;
    for (int k = 0; k < taps; ++k) s = add_mod(s, x[srcs[cell * taps + k] * cell_words + col], q);
    if (w) {
        const ulonglong2 c = w[i];
        s = mul_shoup(s, c.x, c.y, q);
    }
    y[cell * cell_words + col] = s;
}

__global__ void k_gather_cells(const u64* __restrict__ x, const int* __restrict__ idx, u64* __restrict__ y,
                               long long cell_words) {
    const long long cell = blockIdx.y;
    const int s = idx[cell];
    if (s < 0) return;
    for (long long w = static_cast<long long>(blockIdx.x) * TPB + threadIdx.x; w < cell_words;
         w += static_cast<long long>(gridDim.x) * TPB)
        y[cell * cell_words + w] = x[s * cell_words + w];
}

}  // namespace

void gather_mac(const DevRing& R, const GatherMac& g, const u64* x, u64* y, int level, int limb0, int limb1,
                const Launch& L) {
    const int nl = limb1 - limb0;
    const long long cell_words = 2LL * nl * R.n;  // columns this launch covers
    const int tpb = std::min(GM_TPB, R.n);
    if (!g.pixels || !g.oc || nl <= 0) return;
    const int oc_tiles = (g.oc + OCT - 1) / OCT;
    const int pg = g.K <= KCHUNK ? PG : 1;
    const int groups = (g.pixels + pg - 1) / pg;
    const long long blocks = (cell_words + tpb - 1) / tpb * groups * oc_tiles;
    if (blocks > 0x7fffffffLL) throw std::runtime_error("gather_mac: grid too large");
    const unsigned grid = static_cast<unsigned>(blocks);
    L.begin("k_gather_mac", double(g.pixels) * g.K * g.oc * cell_words,
            8.0 * cell_words * (double(g.pixels) * g.oc + g.pixels * g.K));
    k_gather_mac<<<grid, tpb, 0, L.stream>>>(R, g, x, y, level, oc_tiles, groups, pg, limb0, nl);
    L.count();
    check_launch("gather_mac");
}

void pool_sum_scale(const DevRing& R, const u64* x, const int* srcs, int taps, const ulonglong2* w, u64* y, int level,
                    std::size_t out_cells, const Launch& L, bool accumulate) {
    if (!out_cells) return;
    const long long cell_words = 2LL * (level + 1) * R.n;
    for (std::size_t off = 0; off < out_cells; off += 65535) {
        const std::size_t m = std::min<std::size_t>(65535, out_cells - off);
        dim3 grid(static_cast<unsigned>((cell_words + TPB - 1) / TPB), static_cast<unsigned>(m));
        L.begin("k_pool", double(m) * cell_words, 8.0 * cell_words * m * (taps + 1));
        k_pool<<<grid, TPB, 0, L.stream>>>(R, x, srcs + off * taps, taps, w, y + off * cell_words, level,
                                             accumulate ? 1 : 0);
        L.count();
    }
    check_launch("pool_sum_scale");
}

void gather_cells(const u64* x, const int* idx, u64* y, std::size_t cell_words, std::size_t cells, const Launch& L) {
    if (!cells) return;
    const long long cw = static_cast<long long>(cell_words);
    unsigned gx = static_cast<unsigned>(std::min<long long>((cw + TPB - 1) / TPB, 1024));
    for (std::size_t off = 0; off < cells; off += 65535) {
        const std::size_t m = std::min<std::size_t>(65535, cells - off);
        dim3 grid(gx, static_cast<unsigned>(m));
        L.begin("k_gather_cells", 0, 16.0 * cell_words * m);
        k_gather_cells<<<grid, TPB, 0, L.stream>>>(x, idx + off, y + off * cell_words, cw);
        L.count();
    }
    check_launch("gather_cells");
}

}  // namespace hecnn_b200
