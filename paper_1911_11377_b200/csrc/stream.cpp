// Row-streamed forward pass for layer tensors that do not fit in device
// memory.
//
// The reference materialises every layer tensor (forward_encrypted,
// layers.hpp:299-368): one ciphertext per tensor position, so AlexNet's conv1
// output at 32x32x3 is 98,304 ciphertexts of 6 MiB (576 GiB). Here the
// spatial layers are grouped into stages -- [zero_pad2d] (conv2d
// [activation] [avg_pool2d] | activation | avg_pool2d) -- and each stage's
// output is kept only as a ring of the rows its consumer still needs. A stage
// produces one output row at a time in column tiles: conv (linear_apply) ->
// activation (eval_activation) -> pool, all on tile-sized transients, the pool
// result written straight into the next ring. Zero-pad margins are fresh
// encryptions written into the ring rows of the consumer (the same seeds as
// zero_pad2d_encrypted, layers.hpp:241-267), produced only where some
// consumer reads them. Every output word is computed by the same kernels in
// the same arithmetic as the whole-tensor path, so the result is identical
// word for word (tests/test_gpu_stream.py).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <map>
#include <stdexcept>
#include <string>

#include "engine_detail.hpp"

namespace hecnn_b200 {

namespace {

constexpr std::size_t GiB = std::size_t(1) << 30;

bool trace_on() {  // HECNN_STREAM_TRACE=1: plan decisions on stderr
    static const bool v = std::getenv("HECNN_STREAM_TRACE") != nullptr;
    return v;
}

// One stage of the segment; layer indices, -1 when absent.
struct Stage {
    int pad = -1, conv = -1, act = -1, pool = -1;
    std::size_t first = 0, last = 0;  // layers covered
    // input store geometry (logical rows/cols include the pad margins)
    std::size_t in_h = 0, in_w = 0, in_c = 0, margin = 0;
    std::uint32_t in_level = 0;
    double in_scale = 0;
    // conv output (pre-pool) dims, pool size (1 = none), stage output dims
    std::size_t ch = 0, cw = 0, oc = 0, p = 1, oh = 0, ow = 0;
    long long pad_top = 0, pad_left = 0;
    std::uint32_t conv_level = 0, act_level = 0, out_level = 0;  // levels after each piece
    double conv_scale = 0, act_scale = 0, out_scale = 0;
    // rows of the input store needed by output row y
    std::size_t row_lo(std::size_t y) const {
        if (conv < 0) return y * p;
        const long long r = static_cast<long long>(y * p * stride()) - pad_top;
        return static_cast<std::size_t>(std::max(0LL, r));
    }
    std::size_t row_hi(std::size_t y) const {
        if (conv < 0) return y * p + p - 1;
        const long long r = static_cast<long long>((y * p + p - 1) * stride()) - pad_top + static_cast<long long>(kh()) - 1;
        return static_cast<std::size_t>(std::min<long long>(static_cast<long long>(in_h) - 1, r));
    }
    std::size_t window() const {
        std::size_t w = 1;
        for (std::size_t y = 0; y < oh; ++y) w = std::max(w, row_hi(y) - row_lo(y) + 1);
        return w;
    }
    const Layer* cl = nullptr;
    std::size_t stride() const { return cl ? cl->stride : 1; }
    std::size_t kh() const { return cl ? cl->kh : 1; }
};

std::size_t cell_bytes(const Context& C, std::uint32_t level) { return 2 * (level + 1) * C.n() * 8; }

// rough device bytes of a conv / dense layer's weight caches at `level`
std::size_t weight_cache_bytes(const Model& M, std::size_t li, const Shape& in, std::uint32_t level) {
    const Layer& l = M.layers[li];
    const std::size_t rows = l.kind == 0 ? l.kh * l.kw * in.c : in.positions();
    const std::size_t oc = l.kind == 0 ? l.filters : l.units;
    return rows * ((oc + 15) / 16 * 16) * (level + 1) * 40;
}

}  // namespace

struct StreamPlan {
    std::vector<Stage> stages;
    std::size_t first = 0, end = 0;  // layers [first, end)
    std::vector<std::size_t> ring;   // rows kept per store (store s = input of stage s; last = output)
    std::vector<std::size_t> tile;   // output columns per tile, per stage
    // per stage: conv tap tables in (row, tile, dy, column) pixel order and the
    // first pixel of each (row, tile); pool tap tables (fused: per tile width;
    // pool-only: per output row over the ring)
    std::vector<Model::Taps> taps;
    std::vector<std::vector<std::size_t>> tile_pixel0;
    std::vector<std::map<std::size_t, DevBuf>> pool_local;
    std::vector<DevBuf> pool_ring;
    std::vector<DevBuf> pool_w;  // (1/area residue, shoup) per limb at the pool's level
    std::size_t transient = 0;   // bytes budgeted for tile transients
};

namespace detail {

namespace {

std::vector<Stage> parse_stages(const Model& M, const Tensor& x, std::size_t first) {
    std::vector<Stage> st;
    std::size_t i = first;
    Shape cur = x.shape;
    const std::size_t nl = M.layers.size();
    while (i < nl && !cur.flat) {
        Stage s;
        s.first = i;
        std::size_t margin = 0;
        Shape in = cur;
        if (M.layers[i].kind == 2) {
            if (st.empty()) break;  // a leading pad runs as a whole-tensor layer
            s.pad = static_cast<int>(i);
            margin = M.layers[i].pad;
            in = M.shapes[i];
            ++i;
        }
        if (i >= nl) break;
        const int k = M.layers[i].kind;
        if (k != 0 && k != 1 && k != 4) break;
        s.margin = margin;
        s.in_h = in.h, s.in_w = in.w, s.in_c = in.c;
        s.ch = in.h, s.cw = in.w, s.oc = in.c;
        if (k == 0) {
            s.conv = static_cast<int>(i);
            s.cl = &M.layers[i];
            const Shape& o = M.shapes[i];
            s.ch = o.h, s.cw = o.w, s.oc = o.c;
            conv_offsets(M.layers[i], in.h, in.w, o.h, o.w, s.pad_top, s.pad_left);
            ++i;
            if (i < nl && M.layers[i].kind == 4) s.act = static_cast<int>(i++);
            if (i < nl && M.layers[i].kind == 1) s.pool = static_cast<int>(i++);
        } else if (k == 4) {
            s.act = static_cast<int>(i++);
        } else {
            s.pool = static_cast<int>(i++);
        }
        s.p = s.pool >= 0 ? M.layers[static_cast<std::size_t>(s.pool)].pool : 1;
        s.oh = s.ch / s.p, s.ow = s.cw / s.p;
        s.last = i - 1;
        cur = M.shapes[s.last];
        st.push_back(s);
    }
    return st;
}

// Forward the scale/level ledger through the stages exactly as the whole-
// tensor path does (linear: x.scale * Delta / p_l; activation: eval plan;
// pool: x.scale * Delta / p_l). Activation levels/scales are found by a dry
// evaluation of the ledger (activation.hpp:228-265).
void ledger(const Context& C, const Model& M, std::vector<Stage>& st, std::uint32_t level, double scale) {
    for (Stage& s : st) {
        s.in_level = level, s.in_scale = scale;
        if (s.conv >= 0) {
            if (level == 0) throw std::invalid_argument("conv2d: no level headroom");
            scale = scale * C.scale / static_cast<double>(C.ring.primes[level]);
            level -= 1;
        }
        s.conv_level = level, s.conv_scale = scale;
        if (s.act >= 0) {
            // same plan as eval_activation_cells: powers by squaring / mul, terms
            // mul_plain'ed to Delta at one level below their power, summed at the
            // lowest; only the output ledger matters here
            const Activation& a = M.acts[static_cast<std::size_t>(M.layers[static_cast<std::size_t>(s.act)].act)];
            const std::size_t d = a.degree();
            std::map<std::size_t, std::pair<std::uint32_t, double>> pw;
            pw[1] = {level, scale};
            std::function<std::pair<std::uint32_t, double>(std::size_t)> power = [&](std::size_t k) {
                auto it = pw.find(k);
                if (it != pw.end()) return it->second;
                std::pair<std::uint32_t, double> r;
                if (k % 2 == 0) {
                    auto h = power(k / 2);
                    r = {h.first - 1, h.second * h.second / static_cast<double>(C.ring.primes[h.first])};
                } else {
                    auto h = power((k + 1) / 2), lo = power(k / 2);
                    const std::uint32_t lv = std::min(h.first, lo.first);
                    r = {lv - 1, h.second * lo.second / static_cast<double>(C.ring.primes[lv])};
                }
                pw[k] = r;
                return r;
            };
            // the sum keeps the scale of the first term (c_1 x rescaled) and the
            // level of the lowest one
            std::uint32_t out_level = UINT32_MAX;
            double out_scale = 0;
            for (std::size_t k = 1; k <= d; ++k) {
                auto p = power(k);
                const double u = C.scale * static_cast<double>(C.ring.primes[p.first]) / p.second;
                const double sc = p.second * u / static_cast<double>(C.ring.primes[p.first]);
                if (k == 1) out_scale = sc;
                out_level = std::min(out_level, p.first - 1);
            }
            level = out_level, scale = out_scale;
        }
        s.act_level = level, s.act_scale = scale;
        if (s.pool >= 0) {
            if (level == 0) throw std::invalid_argument("avg_pool2d: no level headroom");
            scale = scale * C.scale / static_cast<double>(C.ring.primes[level]);
            level -= 1;
        }
        s.out_level = level, s.out_scale = scale;
    }
}

// store s geometry: logical (padded) rows/cols/channels and level
struct StoreDims {
    std::size_t h, w, c, margin;
    std::uint32_t level;
};

StoreDims store_dims(const std::vector<Stage>& st, std::size_t s, const Tensor& x) {
    if (s == 0) return {x.shape.h, x.shape.w, x.shape.c, 0, x.level};
    const Stage& prev = st[s - 1];
    const std::size_t m = s < st.size() ? st[s].margin : 0;
    return {prev.oh + 2 * m, prev.ow + 2 * m, prev.oc, m, prev.out_level};
}

std::size_t avail_bytes(Context& C) {
    std::size_t fr = 0, tot = 0;
    cuda_check(cudaMemGetInfo(&fr, &tot), "cudaMemGetInfo");
    return fr + C.arena.free_bytes();
}

}  // namespace

TensorPtr forward_streamed(Context& C, Model& M, const Tensor& x, std::size_t first, std::size_t& end, u64 seed,
                           std::vector<double>* layer_ms, const PadNoiseMap& pads) {
    end = first;
    if (M.stream_mode == 2 || x.shape.flat || first >= M.layers.size()) return nullptr;
    std::vector<Stage> st = parse_stages(M, x, first);
    if (st.empty()) return nullptr;
    ledger(C, M, st, x.level, x.scale);
    for (const Stage& s : st)
        if (s.act >= 0 && (s.conv >= 0 ? s.conv_level : s.in_level) <
                              M.acts[static_cast<std::size_t>(M.layers[static_cast<std::size_t>(s.act)].act)].encrypted_depth())
            return nullptr;  // the whole-tensor path raises the reference's error

    // ---- memory plan
    const std::size_t avail = M.mem_budget ? M.mem_budget : avail_bytes(C);
    if (trace_on()) {
        std::size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        std::fprintf(stderr, "[hecnn] stream plan: device free %.1f GiB, arena reserved %.1f GiB (free %.1f)\n",
                     fr / double(GiB), C.arena.reserved() / double(GiB), C.arena.free_bytes() / double(GiB));
    }
    const std::size_t margin = std::min<std::size_t>(2 * GiB, avail / 32);
    // working set besides the stores and tiles: the linear pre-rescale chunk or
    // the activation's power / key-switch chunks (never both at once)
    const std::size_t fixed = 2 * kScratchBytes;
    // whole-tensor peak of layers [first, ...): input + output + scratch per layer
    auto full_peak = [&](std::size_t from, Shape in_shape, std::uint32_t in_level) {
        std::size_t peak = 0;
        Shape cur = in_shape;
        std::uint32_t lv = in_level;
        for (std::size_t i = from; i < M.layers.size(); ++i) {
            const Layer& l = M.layers[i];
            std::uint32_t out_lv = lv;
            if (l.kind == 0 || l.kind == 1 || l.kind == 3) out_lv = lv ? lv - 1 : 0;
            if (l.kind == 4) {
                const std::size_t d = M.acts[static_cast<std::size_t>(l.act)].encrypted_depth();
                out_lv = lv >= d ? static_cast<std::uint32_t>(lv - d) : 0;
            }
            const Shape& o = M.shapes[i];
            std::size_t bytes = cur.positions() * cell_bytes(C, lv) + o.positions() * cell_bytes(C, out_lv);
            if (l.kind == 0 || l.kind == 3) bytes += kScratchBytes + weight_cache_bytes(M, i, cur, lv);
            if (l.kind == 4) bytes += fixed;
            if (l.kind == 1) bytes += o.positions() * cell_bytes(C, lv);
            peak = std::max(peak, bytes);
            cur = o, lv = out_lv;
        }
        return peak;
    };
    const bool fits_whole = full_peak(first, x.shape, x.level) + margin <= avail;
    if (M.stream_mode == 0 && fits_whole) return nullptr;
    // (the stores come from the arena's free blocks; when a store does not fit
    // one, Arena::alloc hands wholly free segments back and retries)

    // rings: store s (s >= 1) keeps the window of rows stage s reads
    const std::size_t S = st.size();
    auto ring_rows = [&](std::size_t s, std::size_t k) -> std::size_t {  // store s of a k-stage segment
        const StoreDims d = store_dims(st, s, x);
        if (s == 0 || s == k) return d.h;  // segment input / output: whole tensors
        return std::min(d.h, st[s].window());
    };
    auto store_bytes = [&](std::size_t s, std::size_t k) {
        const StoreDims d = store_dims(st, s, x);
        const std::size_t w = s == k ? d.w - 2 * d.margin : d.w, h = s == k ? d.h - 2 * d.margin : ring_rows(s, k);
        return h * w * d.c * cell_bytes(C, d.level);
    };
    auto per_col = [&](const Stage& s) {  // transient bytes per output column of a tile
        std::size_t b = 0;
        const std::size_t cells = s.p * s.oc;  // one conv row of the pool window at a time
        if (s.conv >= 0) b += cells * cell_bytes(C, s.conv_level);
        if (s.act >= 0) b += cells * cell_bytes(C, s.act_level);
        if (s.pool >= 0) b += s.oc * cell_bytes(C, s.act_level);
        return std::max<std::size_t>(b, 1);
    };
    std::size_t best = 0, best_tail_ok = 0;
    for (std::size_t k = 1; k <= S; ++k) {
        std::size_t mem = fixed + margin;
        for (std::size_t s = 1; s <= k; ++s) mem += store_bytes(s, k);
        for (std::size_t s = 0; s < k; ++s)
            if (st[s].conv >= 0) {
                const StoreDims d = store_dims(st, s, x);
                mem += weight_cache_bytes(M, static_cast<std::size_t>(st[s].conv), Shape::spatial(d.h, d.w, d.c), d.level);
            }
        std::size_t min_tile = 0;
        for (std::size_t s = 0; s < k; ++s) min_tile = std::max(min_tile, per_col(st[s]));
        if (mem + min_tile > avail) break;
        best = k;
        const std::size_t next = st[k - 1].last + 1;
        const bool tail_ok = next >= M.layers.size() ||
                             full_peak(next, M.shapes[st[k - 1].last], st[k - 1].out_level) + margin <= avail;
        if (tail_ok && !best_tail_ok) best_tail_ok = k;
        if (trace_on())
            std::fprintf(stderr, "[hecnn] stream plan from layer %zu: k=%zu mem %.1f GiB (+tile %.1f) of %.1f, tail %s\n",
                         first, k, mem / double(GiB), min_tile / double(GiB), avail / double(GiB), tail_ok ? "fits" : "no");
    }
    if (!best)
        throw std::runtime_error("forward_encrypted: layer " + std::to_string(first) + " (" + M.layers[first].kind_name() +
                                 "): its row window does not fit in device memory even when streamed");
    std::size_t k = M.stream_mode == 1 ? best : (best_tail_ok ? best_tail_ok : best);
    end = st[k - 1].last + 1;
    st.resize(k);

    // ---- plan (cached per input level and segment)
    char key[160];
    std::snprintf(key, sizeof key, "%zu/%zu/%u/%a/%zu/%zu/%zu", first, end, x.level, x.scale, M.stream_tile,
                  M.mem_budget, x.cells);
    std::shared_ptr<StreamPlan>& slot = M.plans[key];
    if (!slot) {
        auto P = std::make_shared<StreamPlan>();
        P->stages = st;
        P->first = first, P->end = end;
        P->ring.resize(k + 1);
        for (std::size_t s = 0; s <= k; ++s) P->ring[s] = ring_rows(s, k);
        std::size_t mem = 0;
        for (std::size_t s = 1; s <= k; ++s) mem += store_bytes(s, k);
        const std::size_t tbudget = avail > mem + fixed + margin ? avail - mem - fixed - margin : 0;
        P->transient = std::min<std::size_t>(tbudget, 16 * GiB);
        P->tile.resize(k);
        P->taps.resize(k);
        P->tile_pixel0.resize(k);
        P->pool_local.resize(k);
        P->pool_ring.resize(k);
        P->pool_w.resize(k);
        for (std::size_t s = 0; s < k; ++s) {
            Stage& g = P->stages[s];
            const std::size_t want = M.stream_tile ? M.stream_tile : std::max<std::size_t>(1, P->transient / per_col(g));
            P->tile[s] = std::min(g.ow, want);
            const StoreDims in = store_dims(P->stages, s, x);
            const std::size_t R = P->ring[s];
            if (g.conv >= 0) {
                const Layer& l = M.layers[static_cast<std::size_t>(g.conv)];
                const std::size_t K = l.kh * l.kw * in.c;
                Model::LinearCache& lc = linear_weights(C, M, static_cast<std::size_t>(g.conv), g.in_level, K);
                std::vector<int> src;
                const std::size_t tw = P->tile[s];
                for (std::size_t y = 0; y < g.oh; ++y)
                    for (std::size_t x0 = 0; x0 < g.ow; x0 += tw) {
                        P->tile_pixel0[s].push_back(src.size() / K);
                        const std::size_t x1 = std::min(g.ow, x0 + tw);
                        for (std::size_t dy = 0; dy < g.p; ++dy)
                            for (std::size_t cx = g.p * x0; cx < g.p * x1; ++cx) {
                                const std::size_t cy = g.p * y + dy;
                                for (std::size_t ky = 0; ky < l.kh; ++ky)
                                    for (std::size_t kx = 0; kx < l.kw; ++kx)
                                        for (std::size_t ic = 0; ic < in.c; ++ic) {
                                            const long long iy = static_cast<long long>(cy * l.stride + ky) - g.pad_top;
                                            const long long ix = static_cast<long long>(cx * l.stride + kx) - g.pad_left;
                                            const bool ok = iy >= 0 && ix >= 0 && iy < static_cast<long long>(in.h) &&
                                                            ix < static_cast<long long>(in.w);
                                            src.push_back(ok ? static_cast<int>(((static_cast<std::size_t>(iy) % R) * in.w +
                                                                                 static_cast<std::size_t>(ix)) * in.c + ic)
                                                             : -1);
                                        }
                            }
                    }
                P->taps[s] = make_taps(C, lc, src);
            }
            if (g.pool >= 0) {
                const std::size_t p = g.p, taps = p * p;
                std::vector<u64> res = C.enc->scalar_residues(1.0 / static_cast<double>(taps), C.scale, g.act_level);
                std::vector<ulonglong2> w(res.size());
                for (std::size_t i = 0; i < res.size(); ++i)
                    w[i] = make_ulonglong2(res[i], shoup_of(res[i], C.ring.primes[i]));
                P->pool_w[s] = C.upload_vec(w);
                if (g.conv >= 0 || g.act >= 0) {
                    // tile-local, one conv row at a time: pre-pool cells [cx - p x0][c]
                    for (std::size_t tw : {P->tile[s], g.ow % P->tile[s]}) {
                        if (!tw || P->pool_local[s].count(tw)) continue;
                        std::vector<int> srcs;
                        for (std::size_t xx = 0; xx < tw; ++xx)
                            for (std::size_t c = 0; c < g.oc; ++c)
                                for (std::size_t dx = 0; dx < p; ++dx)
                                    srcs.push_back(static_cast<int>((xx * p + dx) * g.oc + c));
                        P->pool_local[s].emplace(tw, C.upload_vec(srcs));
                    }
                } else {
                    std::vector<int> srcs;  // [oh][ow][c][taps] over the input ring
                    for (std::size_t y = 0; y < g.oh; ++y)
                        for (std::size_t xx = 0; xx < g.ow; ++xx)
                            for (std::size_t c = 0; c < g.oc; ++c)
                                for (std::size_t dy = 0; dy < p; ++dy)
                                    for (std::size_t dx = 0; dx < p; ++dx)
                                        srcs.push_back(static_cast<int>((((y * p + dy) % R) * in.w + xx * p + dx) * in.c + c));
                    P->pool_ring[s] = C.upload_vec(srcs);
                }
            }
        }
        slot = P;
    }
    StreamPlan& P = *slot;
    st = P.stages;

    // ---- stores
    // One arena block [segment output | rings]: a single contiguous request
    // (fragmented free space cannot strand a ring), and after the segment the
    // ring part is handed back while the output stays.
    std::vector<u64*> base(k + 1);
    std::vector<StoreDims> dims(k + 1);
    base[0] = x.data();
    for (std::size_t s = 0; s <= k; ++s) dims[s] = store_dims(st, s, x);
    const Stage& lastst = st[k - 1];
    const std::size_t out_cells = lastst.oh * lastst.ow * lastst.oc;
    const std::size_t out_bytes = (out_cells * cell_bytes(C, lastst.out_level) + 255) & ~std::size_t(255);
    std::vector<std::size_t> ring_off(k + 1, 0);
    std::size_t total = out_bytes;
    for (std::size_t s = 1; s < k; ++s) {
        ring_off[s] = total;
        total += (P.ring[s] * dims[s].w * dims[s].c * cell_bytes(C, dims[s].level) + 255) & ~std::size_t(255);
    }
    DevBuf block(&C, total);
    char* blk = block.as<char>();
    for (std::size_t s = 1; s < k; ++s) base[s] = reinterpret_cast<u64*>(blk + ring_off[s]);
    TensorPtr out = std::make_unique<Tensor>();
    out->ctx = &C;
    out->cells = out_cells;
    out->level = lastst.out_level;
    out->scale = lastst.out_scale;
    out->shape = M.shapes[lastst.last];
    out->batch = x.batch;
    base[k] = reinterpret_cast<u64*>(blk);

    // columns of store s any consumer reads (border encryptions elsewhere are skipped)
    std::vector<std::size_t> used_w(k + 1, 0);
    for (std::size_t s = 0; s < k; ++s) {
        const Stage& g = st[s];
        std::size_t hi = 0;
        if (g.conv >= 0) {
            const Layer& l = M.layers[static_cast<std::size_t>(g.conv)];
            const long long r = static_cast<long long>((g.p * g.ow - 1) * l.stride + l.kw) - g.pad_left;
            hi = static_cast<std::size_t>(std::min<long long>(static_cast<long long>(dims[s].w), r));
        } else {
            hi = g.p * g.ow;
        }
        used_w[s] = hi;
    }
    used_w[k] = dims[k].w;

    std::vector<std::size_t> produced(k + 1, 0);
    produced[0] = dims[0].h;  // the segment input is a whole tensor
    Launch L = C.L();

    // per-layer device time (layer_seconds of forward_encrypted)
    struct Mark {
        int layer;
        cudaEvent_t a, b;
    };
    std::vector<Mark> marks;
    auto timed = [&](int layer, auto&& fn) {
        if (!layer_ms) {
            fn();
            return;
        }
        Mark m{layer, C.prof.take(), C.prof.take()};
        cudaEventRecord(m.a, C.stream);
        fn();
        cudaEventRecord(m.b, C.stream);
        marks.push_back(m);
    };

    auto words = [&](std::uint32_t level) { return 2 * (static_cast<std::size_t>(level) + 1) * C.n(); };
    std::vector<bool> checked(k + 1, false);
    // zero_pad2d border: fresh encryptions of 0 at store s row q, cols [c0, c1)
    // (layers.hpp:255-262: seed derive_seed(layer_seed, 0xbad0 + position))
    auto fresh = [&](std::size_t s, std::size_t q, std::size_t c0, std::size_t c1) {
        c1 = std::min(c1, used_w[s]);
        if (c0 >= c1) return;
        const Stage& g = st[s];
        const StoreDims& d = dims[s];
        if (!checked[s]) {  // encode_const(0, scale, top) range check
            C.enc->check_encode(1, 0.0, st[s - 1].out_scale, C.top());
            checked[s] = true;
        }
        u64* dst = base[s] + ((q % P.ring[s]) * d.w + c0) * d.c * words(d.level);
        const std::size_t p0 = (q * d.w + c0) * d.c, cnt = (c1 - c0) * d.c;
        auto it = pads.find(static_cast<std::size_t>(g.pad));
        if (it != pads.end()) {  // sampled on host threads while earlier rows ran: positions
            const PadNoise& N = *it->second.get();  // p0.. are consecutive border cells
            const std::size_t k0 = static_cast<std::size_t>(N.border[p0]), nn = C.n();
            timed(g.pad, [&] { encrypt_sampled(C, cnt, &N.r[k0 * nn], &N.e0[k0 * nn], &N.e1[k0 * nn], d.level, dst); });
        } else {
            const u64 layer_seed = derive_seed(seed, 0x1a7e + static_cast<u64>(g.pad));
            std::vector<u64> seeds(cnt);
            for (std::size_t k = 0; k < cnt; ++k) seeds[k] = derive_seed(layer_seed, 0xbad0 + p0 + k);
            timed(g.pad, [&] { encrypt_into(C, seeds.size(), seeds.data(), nullptr, d.level, dst); });
        }
    };

    // a tensor view over device cells (no ownership)
    auto view = [&](u64* p, std::size_t cells, std::uint32_t level, double scale) {
        auto t = std::make_unique<Tensor>();
        t->ctx = &C;
        t->cells = cells;
        t->level = level;
        t->scale = scale;
        t->batch = x.batch;
        t->buf = DevBuf::alias(p, cells * words(level) * 8);
        return t;
    };

    std::function<void(std::size_t, std::size_t)> ensure;
    // stage s computes its output row y into store s + 1
    auto compute_row = [&](std::size_t s, std::size_t y) {
        const Stage& g = st[s];
        ensure(s, g.row_hi(y));
        const StoreDims& in = dims[s];
        const StoreDims& od = dims[s + 1];
        const std::size_t q = y + od.margin;
        u64* orow = base[s + 1] + ((q % P.ring[s + 1]) * od.w + od.margin) * od.c * words(od.level);
        const std::size_t tw = P.tile[s], ntiles = (g.ow + tw - 1) / tw;
        for (std::size_t x0 = 0, t = 0; x0 < g.ow; x0 += tw, ++t) {
            const std::size_t w = std::min(g.ow, x0 + tw) - x0;
            u64* dst = orow + x0 * g.oc * words(od.level);
            if (g.conv < 0 && g.act < 0) {  // pool over the input ring
                const std::size_t taps = g.p * g.p;
                DevBuf pre(&C, w * g.oc * words(g.act_level) * 8);
                timed(g.pool, [&] {
                    pool_sum_scale(C.dev, base[s], P.pool_ring[s].as<int>() + (y * g.ow + x0) * g.oc * taps,
                                   static_cast<int>(taps), P.pool_w[s].as<ulonglong2>(), pre.as<u64>(),
                                   static_cast<int>(g.act_level), w * g.oc, L);
                    rescale(C.dev, pre.as<u64>(), dst, static_cast<int>(g.act_level), 2 * w * g.oc, L);
                });
                continue;
            }
            // conv rows of the pool window one at a time: conv -> activation ->
            // accumulate into the pool sum; the last row scales by 1/area
            DevBuf pre;
            if (g.pool >= 0) pre = DevBuf(&C, w * g.oc * words(g.act_level) * 8);
            for (std::size_t dy = 0; dy < g.p; ++dy) {
                const std::size_t row_cells = g.p * w * g.oc;  // p * w conv pixels x oc
                DevBuf t1, a1;
                const u64* cur = nullptr;
                if (g.conv >= 0) {
                    const Layer& l = M.layers[static_cast<std::size_t>(g.conv)];
                    const std::size_t K = l.kh * l.kw * in.c;
                    Model::LinearCache& lc = linear_weights(C, M, static_cast<std::size_t>(g.conv), g.in_level, K);
                    const u64* bias = linear_bias(C, M, static_cast<std::size_t>(g.conv), g.in_level, g.in_scale * C.scale);
                    u64* t1p = dst;
                    if (g.act >= 0 || g.pool >= 0) {
                        t1 = DevBuf(&C, row_cells * words(g.conv_level) * 8);
                        t1p = t1.as<u64>();
                    }
                    timed(g.conv, [&] {
                        linear_apply(C, lc, P.taps[s], bias, base[s], g.in_level,
                                     P.tile_pixel0[s][y * ntiles + t] + dy * g.p * w, g.p * w, t1p);
                    });
                    cur = t1p;
                }
                if (g.act >= 0) {
                    const Activation& act =
                        M.acts[static_cast<std::size_t>(M.layers[static_cast<std::size_t>(g.act)].act)];
                    TensorPtr v = g.conv >= 0
                                      ? view(const_cast<u64*>(cur), row_cells, g.conv_level, g.conv_scale)
                                      : view(base[s] + ((y % P.ring[s]) * in.w + x0) * in.c * words(in.level),
                                             w * in.c, in.level, g.in_scale);
                    u64* adst = dst;
                    if (g.pool >= 0) {
                        a1 = DevBuf(&C, row_cells * words(g.act_level) * 8);
                        adst = a1.as<u64>();
                    }
                    TensorPtr r;
                    timed(g.act, [&] { r = eval_activation(C, act, *v, adst); });
                    if (r->level != g.act_level || r->scale != g.act_scale)
                        throw std::logic_error("forward_encrypted: streamed activation ledger mismatch");
                    cur = adst;
                    t1.reset();
                }
                if (g.pool >= 0) {
                    const bool last_row = dy + 1 == g.p;
                    timed(g.pool, [&] {
                        pool_sum_scale(C.dev, cur, P.pool_local[s].at(w).as<int>(), static_cast<int>(g.p),
                                       last_row ? P.pool_w[s].as<ulonglong2>() : nullptr, pre.as<u64>(),
                                       static_cast<int>(g.act_level), w * g.oc, L, dy > 0);
                        if (last_row) rescale(C.dev, pre.as<u64>(), dst, static_cast<int>(g.act_level), 2 * w * g.oc, L);
                    });
                }
            }
        }
        if (s + 1 < k && od.margin) {  // the consumer's pad margins on this row
            fresh(s + 1, q, 0, od.margin);
            fresh(s + 1, q, od.margin + g.ow, od.w);
        }
    };
    ensure = [&](std::size_t s, std::size_t r) {
        while (produced[s] <= r) {
            const std::size_t q = produced[s];
            const std::size_t m = dims[s].margin, inner = st[s - 1].oh;
            if (q < m || q >= m + inner) fresh(s, q, 0, dims[s].w);
            else compute_row(s - 1, q - m);
            ++produced[s];
        }
    };
    if (trace_on())
        std::fprintf(stderr, "[hecnn] stream layers [%zu, %zu): %zu stages, transient %.1f GiB\n", first, end, k,
                     P.transient / double(GiB));
    for (std::size_t y = 0; y < st[k - 1].oh; ++y) compute_row(k - 1, y);
    // rings done (later work on the stream is ordered after their last use):
    // keep the output part of the block
    C.arena.shrink(block.get(), out_bytes);
    out->buf = DevBuf::adopt(&C, block.release_ownership(), out_bytes);
    if (layer_ms) {
        C.sync();
        for (const Mark& m : marks) {
            float ms = 0;
            cudaEventElapsedTime(&ms, m.a, m.b);
            (*layer_ms)[static_cast<std::size_t>(m.layer)] += ms;
            C.prof.pool.push_back(m.a);
            C.prof.pool.push_back(m.b);
        }
    }
    return out;
}

}  // namespace detail
}  // namespace hecnn_b200
