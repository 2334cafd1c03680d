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
constexpr int OCT = 8;

constexpr int KCHUNK = 128;
constexpr int TAPB = 4;  // input words in flight per thread

// One thread = one (component, limb, coefficient) column of OCT output
// channels of one pixel. The pixel's taps (source cell, weight row) and the
// limb's weights for the OCT channels are staged in shared memory per chunk
// of KCHUNK taps, so the inner loop is: TAPB independent coalesced loads of
// input words, then OCT multiply-accumulates each against broadcast shared
// words. The grid is column-block major (blockIdx.x = (column block, pixel,
// channel tile), channel tile fastest), so while one column block is in
// flight every input cell's slice of it (cells x TPB words) stays in L2 and
// is reused by all pixels whose window covers it and by all channel tiles.
__global__ void __launch_bounds__(TPB, 2) k_gather_mac(DevRing R, GatherMac g, const u64* __restrict__ x,
                                                    u64* __restrict__ y, int level, int oc_tiles) {
    __shared__ int s_src[KCHUNK];
    __shared__ double2 s_w[KCHUNK][OCT];
    __shared__ ulonglong2 s_ws[KCHUNK][OCT];
    const int limbs = level + 1;
    const long long poly_words = static_cast<long long>(limbs) * R.n;
    const long long cell_words = 2 * poly_words;
    const int tpb = blockDim.x;  // <= n, so a CTA's columns share one limb
    const long long per_block = static_cast<long long>(g.pixels) * oc_tiles;
    const long long bid = blockIdx.x;
    const long long cb = bid / per_block;
    const int pz = static_cast<int>(bid - cb * per_block);
    const int pixel = pz / oc_tiles;
    const int oc0 = (pz - pixel * oc_tiles) * OCT;
    const long long col0 = cb * tpb;
    const long long col = col0 + threadIdx.x;
    const bool live = col < cell_words;
    const int comp = static_cast<int>(col / poly_words);
    const int i = static_cast<int>(((live ? col : col0) / R.n) % limbs);  // uniform when n >= TPB
    const int j = static_cast<int>(col % R.n);
    const ModConst m = R.mod[i];
    const u64 q = m.q, two_q = q << 1;
    const int* src = g.src + static_cast<long long>(pixel) * g.K;
    const int* wrow = g.wrow + static_cast<long long>(pixel) * g.K;
    const long long wbase = static_cast<long long>(i) * g.rows;
    const u64* xc = x + (live ? col : 0);
    // q < 2^42: x, w split at bit 21 into exact doubles; every partial product
    // is < 2^42 and a chunk of KCHUNK taps sums below 2^51, so the FP64 pipe
    // accumulates exactly; accumulators are centred mod q after each chunk.
    const bool split = ntt::fp_limb(q);
    const double qd = static_cast<double>(q), qinv = R.inv_q[i];

    u64 s00[OCT];
    double f00[OCT], fmid[OCT], f11[OCT];
#pragma unroll
    for (int o = 0; o < OCT; ++o) {
        s00[o] = 0;
        f00[o] = fmid[o] = f11[o] = 0.0;
    }

    for (int k0 = 0; k0 < g.K; k0 += KCHUNK) {
        const int kn = min(KCHUNK, g.K - k0);
        const int kpad = (kn + TAPB - 1) / TAPB * TAPB;  // taps kn..kpad: src -1, weight 0
        __syncthreads();
        for (int t = threadIdx.x; t < kpad * OCT; t += tpb) {
            const int k = t / OCT, o = t % OCT;
            const bool ok = k < kn;
            const long long at = ok ? (wbase + wrow[k0 + k]) * g.oc_pad + oc0 + o : 0;
            if (split) {
                const uint2 w = ok ? g.wsplit[at] : make_uint2(0, 0);
                s_w[k][o] = make_double2(static_cast<double>(w.x), static_cast<double>(w.y));
            } else {
                s_ws[k][o] = ok ? g.weights[at] : make_ulonglong2(0, 0);
            }
            if (o == 0) s_src[k] = ok ? src[k0 + k] : -1;
        }
        __syncthreads();
        if (!live) continue;
        // invalid taps (s < 0, zero padding) load nothing and contribute 0
        if (split) {
            for (int kb = 0; kb < kpad; kb += TAPB) {
                u64 v[TAPB];
#pragma unroll
                for (int u = 0; u < TAPB; ++u) {
                    const int s = s_src[kb + u];
                    v[u] = s >= 0 ? __ldg(xc + s * cell_words) : 0;
                }
#pragma unroll
                for (int u = 0; u < TAPB; ++u) {
                    const int k = kb + u;
                    const double v0 = ntt::to_fp(v[u] & 0x1FFFFFull), v1 = ntt::to_fp(v[u] >> 21);
#pragma unroll
                    for (int o = 0; o < OCT; ++o) {
                        const double2 c = s_w[k][o];
                        f00[o] = fma(v0, c.x, f00[o]);
                        fmid[o] = fma(v0, c.y, fmid[o]);
                        fmid[o] = fma(v1, c.x, fmid[o]);
                        f11[o] = fma(v1, c.y, f11[o]);
                    }
                }
            }
#pragma unroll
            for (int o = 0; o < OCT; ++o) {
                f00[o] = ntt::fcentre(f00[o], qd, qinv);
                fmid[o] = ntt::fcentre(fmid[o], qd, qinv);
                f11[o] = ntt::fcentre(f11[o], qd, qinv);
            }
        } else {
            for (int kb = 0; kb < kpad; kb += TAPB) {
                u64 v[TAPB];
#pragma unroll
                for (int u = 0; u < TAPB; ++u) {
                    const int s = s_src[kb + u];
                    v[u] = s >= 0 ? __ldg(xc + s * cell_words) : 0;
                }
#pragma unroll
                for (int u = 0; u < TAPB; ++u) {
                    const int k = kb + u;
#pragma unroll
                    for (int o = 0; o < OCT; ++o) {
                        const ulonglong2 c = s_ws[k][o];
                        const u64 t = s00[o] + mul_shoup_lazy(v[u], c.x, c.y, q);
                        s00[o] = t >= two_q ? t - two_q : t;
                    }
                }
            }
        }
    }
    if (!live) return;
    const ulonglong2 c21 = g.recomb[2 * i], c42 = g.recomb[2 * i + 1];
#pragma unroll
    for (int o = 0; o < OCT; ++o) {
        const int oc = oc0 + o;
        if (oc >= g.oc) break;
        u64 v;
        if (split) {
            const double t = f00[o] + ntt::fmodmul(fmid[o], static_cast<double>(c21.x), qd, qinv) +
                             ntt::fmodmul(f11[o], static_cast<double>(c42.x), qd, qinv);
            v = ntt::fcanon(t, qd, qinv);
        } else {
            v = reduce_2q(s00[o], q);
        }
        if (g.bias && comp == 0 && j == 0) v = add_mod(v, g.bias[static_cast<long long>(oc) * limbs + i], q);
        y[(static_cast<long long>(pixel) * g.out_stride_pixel + oc) * cell_words + col] = v;
    }
}

// avg_pool2d_encrypted (layers.hpp:213-239): sum of the window, times
// round(Delta / area) (one Shoup multiply), rescale done by the caller.
__global__ void k_pool(DevRing R, const u64* __restrict__ x, const int* __restrict__ srcs, int taps,
                       const ulonglong2* __restrict__ w, u64* __restrict__ y, int level) {
    const int limbs = level + 1;
    const long long poly_words = static_cast<long long>(limbs) * R.n;
    const long long cell_words = 2 * poly_words;
    const long long col = static_cast<long long>(blockIdx.x) * TPB + threadIdx.x;
    if (col >= cell_words) return;
    const int i = static_cast<int>((col / R.n) % limbs);
    const long long cell = blockIdx.y;
    const u64 q = R.mod[i].q;
    u64 s = 0;
    for (int k = 0; k < taps; ++k) s = add_mod(s, x[srcs[cell * taps + k] * cell_words + col], q);
    const ulonglong2 c = w[i];
    y[cell * cell_words + col] = mul_shoup(s, c.x, c.y, q);
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

void gather_mac(const DevRing& R, const GatherMac& g, const u64* x, u64* y, int level, const Launch& L) {
    const long long cell_words = 2LL * (level + 1) * R.n;
    const int tpb = std::min(TPB, R.n);
    if (!g.pixels || !g.oc) return;
    const int oc_tiles = (g.oc + OCT - 1) / OCT;
    const long long blocks = (cell_words + tpb - 1) / tpb * g.pixels * oc_tiles;
    if (blocks > 0x7fffffffLL) throw std::runtime_error("gather_mac: grid too large");
    const unsigned grid = static_cast<unsigned>(blocks);
    L.begin("k_gather_mac", double(g.pixels) * g.K * g.oc * cell_words,
            8.0 * cell_words * (double(g.pixels) * g.oc + g.pixels * g.K));
    k_gather_mac<<<grid, tpb, 0, L.stream>>>(R, g, x, y, level, oc_tiles);
    L.count();
    check_launch("gather_mac");
}

void pool_sum_scale(const DevRing& R, const u64* x, const int* srcs, int taps, const ulonglong2* w, u64* y, int level,
                    std::size_t out_cells, const Launch& L) {
    if (!out_cells) return;
    const long long cell_words = 2LL * (level + 1) * R.n;
    for (std::size_t off = 0; off < out_cells; off += 65535) {
        const std::size_t m = std::min<std::size_t>(65535, out_cells - off);
        dim3 grid(static_cast<unsigned>((cell_words + TPB - 1) / TPB), static_cast<unsigned>(m));
        L.begin("k_pool", double(m) * cell_words, 8.0 * cell_words * m * (taps + 1));
        k_pool<<<grid, TPB, 0, L.stream>>>(R, x, srcs + off * taps, taps, w, y + off * cell_words, level);
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
