// Device-resident CKKS engine (see engine.hpp).
#include "engine.hpp"
#include "engine_detail.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <functional>
#include <future>
#include <stdexcept>
#include <thread>
#include <tuple>

namespace hecnn_b200 {

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

namespace {

// HECNN_TRACE=1 prints host wall time of the engine's phases (diagnostics).
struct Trace {
    const char* what;
    std::chrono::steady_clock::time_point t0;
    static bool on() {
        static const bool v = std::getenv("HECNN_TRACE") != nullptr;
        return v;
    }
    explicit Trace(const char* w) : what(w), t0(std::chrono::steady_clock::now()) {}
    ~Trace() {
        if (on())
            std::fprintf(stderr, "[hecnn] %-28s %9.3f ms\n", what,
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
};

using detail::kScratchBytes;

unsigned host_threads() {
    unsigned t = std::thread::hardware_concurrency();
    return t ? std::min(t, 64u) : 4u;
}

// Disjoint-output parallel loop for host-side sampling (results do not
// depend on the chunking: every item owns its seed and output slot).
void parallel_items(std::size_t count, const std::function<void(std::size_t)>& fn) {
    unsigned workers = static_cast<unsigned>(std::min<std::size_t>(host_threads(), count));
    if (workers <= 1) {
        for (std::size_t i = 0; i < count; ++i) fn(i);
        return;
    }
    std::vector<std::thread> pool;
    std::size_t chunk = (count + workers - 1) / workers;
    for (unsigned w = 0; w < workers; ++w) {
        std::size_t b = w * chunk, e = std::min(count, b + chunk);
        if (b >= e) break;
        pool.emplace_back([&fn, b, e] {
            for (std::size_t i = b; i < e; ++i) fn(i);
        });
    }
    for (auto& t : pool) t.join();
}

std::vector<ulonglong2> with_shoup(const RingTables& R, const std::vector<u64>& res) {
    std::vector<ulonglong2> out(res.size());
    for (std::size_t i = 0; i < res.size(); ++i) out[i] = make_ulonglong2(res[i], shoup_of(res[i], R.primes[i]));
    return out;
}

void require_scale_match(double sx, double sy, const char* op) {
    double m = std::max(std::abs(sx), std::abs(sy));
    if (std::abs(sx - sy) > 0x1p-30 * m)
        throw std::invalid_argument(std::string(op) + ": scale mismatch (no silent alignment)");
}

void check_scale_headroom(const Context& C, double sx, double sy, std::size_t level) {
    if (std::log2(sx) + std::log2(sy) >= C.ring.log2_mod[level] - 1.0)
        throw std::invalid_argument("mul: scale overflow for the active modulus");
}

std::vector<long long> sample_error(const Context& C, u64 seed) {
    if (C.degenerate || C.sigma == 0.0) return std::vector<long long>(C.n(), 0);
    return sample_gaussian(C.n(), C.sigma, seed);
}

std::vector<long long> sample_secretish(const Context& C, double density, u64 seed) {
    if (C.degenerate) return std::vector<long long>(C.n(), 0);
    return sample_ternary(C.n(), density, seed);
}

void to_int8(const std::vector<long long>& v, signed char* out) {
    for (std::size_t i = 0; i < v.size(); ++i) {
        if (v[i] < -127 || v[i] > 127)
            throw std::invalid_argument("encrypt: noise coefficient outside the device sampler's int8 range");
        out[i] = static_cast<signed char>(v[i]);
    }
}

}  // namespace

// ---------------------------------------------------------------- memory

Arena::~Arena() {
    for (auto& s : segs_)
        if (s.first) cudaFree(s.first);
}

void* Arena::alloc(std::size_t bytes) {
    bytes = (bytes + 255) & ~std::size_t(255);
    auto best = free_.end();
    for (auto it = free_.begin(); it != free_.end(); ++it)
        if (it->second.size >= bytes && (best == free_.end() || it->second.size < best->second.size)) best = it;
    if (best == free_.end()) {
        const std::size_t seg = std::max(bytes, std::size_t(1) << 30);
        void* p = nullptr;
        cudaError_t e = cudaMalloc(&p, seg);
        if (e != cudaSuccess) {  // give back wholly free segments and retry once
            cudaGetLastError();
            trim();
            e = cudaMalloc(&p, seg);
        }
        if (e != cudaSuccess && seg > bytes) {  // fall back to an exact-size segment
            cudaGetLastError();
            e = cudaMalloc(&p, bytes);
            if (e == cudaSuccess) {
                segs_.push_back({static_cast<char*>(p), bytes});
                reserved_ += bytes;
                best = free_.emplace(static_cast<char*>(p), Block{bytes, static_cast<int>(segs_.size() - 1)}).first;
            }
        } else if (e == cudaSuccess) {
            segs_.push_back({static_cast<char*>(p), seg});
            reserved_ += seg;
            best = free_.emplace(static_cast<char*>(p), Block{seg, static_cast<int>(segs_.size() - 1)}).first;
        }
        if (e != cudaSuccess) {
            cudaGetLastError();
            throw std::runtime_error("device arena: out of memory allocating " + std::to_string(bytes) + " bytes (" +
                                     std::to_string(reserved_) + " reserved)");
        }
    }
    char* p = best->first;
    Block blk = best->second;
    free_.erase(best);
    if (blk.size > bytes) free_.emplace(p + bytes, Block{blk.size - bytes, blk.seg});
    used_.emplace(p, Block{bytes, blk.seg});
    return p;
}

std::size_t Arena::trim() {
    std::size_t freed = 0;
    for (auto it = free_.begin(); it != free_.end();) {
        const int seg = it->second.seg;
        if (seg >= 0 && segs_[seg].first == it->first && segs_[seg].second == it->second.size) {
            cudaFree(segs_[seg].first);
            freed += segs_[seg].second;
            reserved_ -= segs_[seg].second;
            segs_[seg] = {nullptr, 0};  // ids stay stable; slot is dead
            it = free_.erase(it);
        } else {
            ++it;
        }
    }
    return freed;
}

void Arena::release(void* ptr) {
    auto it = used_.find(static_cast<char*>(ptr));
    if (it == used_.end()) return;
    char* p = it->first;
    Block blk = it->second;
    used_.erase(it);
    auto next = free_.lower_bound(p);
    if (next != free_.end() && next->second.seg == blk.seg && p + blk.size == next->first) {
        blk.size += next->second.size;
        next = free_.erase(next);
    }
    if (next != free_.begin()) {
        auto prev = std::prev(next);
        if (prev->second.seg == blk.seg && prev->first + prev->second.size == p) {
            prev->second.size += blk.size;
            return;
        }
    }
    free_.emplace(p, blk);
}

void Arena::shrink(void* ptr, std::size_t bytes) {
    bytes = (bytes + 255) & ~std::size_t(255);
    auto it = used_.find(static_cast<char*>(ptr));
    if (it == used_.end() || it->second.size <= bytes) return;
    const std::size_t rest = it->second.size - bytes;
    const int seg = it->second.seg;
    it->second.size = bytes;
    char* tail = static_cast<char*>(ptr) + bytes;
    used_.emplace(tail, Block{rest, seg});
    release(tail);  // coalesces with a free neighbour
}

DevBuf DevBuf::adopt(Context* ctx, void* ptr, std::size_t bytes) {
    DevBuf b;
    b.ctx_ = ctx;
    b.ptr_ = ptr;
    b.bytes_ = bytes;
    return b;
}

DevBuf::DevBuf(Context* ctx, std::size_t bytes) : ctx_(ctx), bytes_(bytes) {
    Trace tr(bytes > (64u << 20) ? "alloc>64MiB" : "alloc");
    if (bytes) ptr_ = ctx->arena.alloc(bytes);
}

DevBuf& DevBuf::operator=(DevBuf&& o) noexcept {
    if (this != &o) {
        reset();
        ctx_ = o.ctx_;
        ptr_ = o.ptr_;
        bytes_ = o.bytes_;
        o.ptr_ = nullptr;
        o.bytes_ = 0;
    }
    return *this;
}

DevBuf DevBuf::alias(void* ptr, std::size_t bytes) {
    DevBuf b;
    b.ptr_ = ptr;
    b.bytes_ = bytes;  // ctx_ stays null: the view never releases the memory
    return b;
}

void DevBuf::reset() {
    if (ptr_ && ctx_) ctx_->arena.release(ptr_);
    ptr_ = nullptr;
    bytes_ = 0;
}

std::string Shape::str() const {
    if (flat) return "(" + std::to_string(feat) + ")";
    return "(" + std::to_string(h) + "x" + std::to_string(w) + "x" + std::to_string(c) + ")";
}

// ---------------------------------------------------------------- profiler

cudaEvent_t Profiler::take() {
    if (pool.empty()) {
        cudaEvent_t e;
        cuda_check(cudaEventCreate(&e), "cudaEventCreate");
        return e;
    }
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
}

void Profiler::begin(const char* name, cudaStream_t s, double ops, double bytes) {
    open_name = name;
    open_ops = ops;
    open_bytes = bytes;
    open_start = take();
    cudaEventRecord(open_start, s);
}

void Profiler::end(cudaStream_t s) {
    if (!open_name) return;
    cudaEvent_t stop = take();
    cudaEventRecord(stop, s);
    pending.push_back({open_name, open_start, stop, open_ops, open_bytes});
    open_name = nullptr;
}

void Profiler::collect() {
    for (auto& p : pending) {
        float ms = 0;
        cudaEventElapsedTime(&ms, p.start, p.stop);
        Stat& st = stats[p.name];
        st.ms += ms;
        st.ops += p.ops;
        st.bytes += p.bytes;
        st.launches += 1;
        pool.push_back(p.start);
        pool.push_back(p.stop);
    }
    pending.clear();
}

void Profiler::reset() {
    collect();
    stats.clear();
}

// ---------------------------------------------------------------- context

Context::Context(std::size_t n, const std::vector<u64>& primes, double sc, double sg, bool degen, int dev_id)
    : device(dev_id), scale(sc), sigma(sg), degenerate(degen) {
    validate_chain(n, primes);  // RingContext ctor (ring.hpp:173-175)
    if (!(scale > 1.0)) throw std::invalid_argument("CkksParams: scale must be > 1");
    if (sigma < 0.0) throw std::invalid_argument("CkksParams: sigma must be >= 0");
    ring.build(n, primes);
    enc = std::make_unique<Encoder>(ring, scale);

    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    cuda_check(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "cudaStreamCreate");
    own_stream = true;
    cuda_check(cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaEventCreateWithFlags(&fork_ev, cudaEventDisableTiming), "cudaEventCreate");
    cuda_check(cudaEventCreateWithFlags(&join_ev, cudaEventDisableTiming), "cudaEventCreate");

    std::vector<ModConst> mods;
    for (const auto& m : ring.mods) mods.push_back(ModConst{m.q, 2 * m.q, m.ratio_lo, m.ratio_hi});
    std::vector<double> inv_q;
    for (u64 q : ring.primes) inv_q.push_back(1.0 / static_cast<double>(q));

    tables.push_back(upload_vec(mods));
    dev.mod = tables.back().as<ModConst>();
    tables.push_back(upload_vec(ring.fwd));
    dev.fwd = tables.back().as<ulonglong2>();
    tables.push_back(upload_vec(ring.inv));
    dev.inv = tables.back().as<ulonglong2>();
    tables.push_back(upload_vec(ring.n_inv));
    dev.n_inv = tables.back().as<ulonglong2>();
    tables.push_back(upload_vec(ring.inv_dropped));
    dev.inv_dropped = tables.back().as<ulonglong2>();
    tables.push_back(upload_vec(ring.p_mod));
    dev.p_mod = tables.back().as<u64>();
    tables.push_back(upload_vec(ring.punct_inv));
    dev.punct_inv = tables.back().as<ulonglong2>();
    tables.push_back(upload_vec(ring.punct));
    dev.punct = tables.back().as<u64>();
    tables.push_back(upload_vec(ring.modulus));
    dev.modulus = tables.back().as<u64>();
    {
        // Garner's mixed-radix constants for k_crt_digits_garner (FP64 limbs only)
        std::vector<double> gi(ring.limbs * ring.limbs, 0.0), c30(ring.limbs, 0.0);
        for (std::size_t i = 1; i < ring.limbs; ++i) {
            if (ring.primes[i] >= (1ull << 42)) continue;
            c30[i] = static_cast<double>((1ull << 30) % ring.primes[i]);
            for (std::size_t j = 0; j < i; ++j)
                gi[i * ring.limbs + j] = static_cast<double>(ring.mods[i].inv(ring.primes[j] % ring.primes[i]));
        }
        tables.push_back(upload_vec(gi));
        dev.garner_inv = tables.back().as<double>();
        tables.push_back(upload_vec(c30));
        dev.garner_c30 = tables.back().as<double>();
    }
    tables.push_back(upload_vec(inv_q));
    dev.inv_q = tables.back().as<double>();
    tables.push_back(upload_vec(ring.fwd_f));
    dev.fwd_f = tables.back().as<double>();
    tables.push_back(upload_vec(ring.inv_f));
    dev.inv_f = tables.back().as<double>();
    tables.push_back(upload_vec(ring.n_inv_f));
    dev.n_inv_f = tables.back().as<double>();
    {
        // key-switch block twiddle tables (DevRing::ks_tw): identical to the
        // forward tables unless N > 2^13 blocks
        const std::size_t lb = std::min<std::size_t>(ring.logn, 13), B = std::size_t(1) << lb, C = ring.logn - lb;
        if (C == 0) {
            dev.ks_tw = dev.fwd;
            dev.ks_tw_f = dev.fwd_f;
        } else {
            const std::size_t nn = ring.n, NB = nn / B;
            std::vector<u64> ti(2 * ring.limbs * nn, 0);
            std::vector<double> tf(ring.limbs * nn, 0.0);
            for (std::size_t l = 0; l < ring.limbs; ++l)
                for (std::size_t b = 0; b < NB; ++b)
                    for (std::size_t j = 1; j < B; ++j) {
                        std::size_t sh = 0;
                        while ((std::size_t(2) << sh) <= j) ++sh;
                        const std::size_t m = j - (std::size_t(1) << sh);
                        const std::size_t src = (std::size_t(1) << (sh + C)) + (b << sh) + m, dst = b * B + j;
                        ti[2 * (l * nn + dst)] = ring.fwd[2 * (l * nn + src)];
                        ti[2 * (l * nn + dst) + 1] = ring.fwd[2 * (l * nn + src) + 1];
                        tf[l * nn + dst] = ring.fwd_f[l * nn + src];
                    }
            tables.push_back(upload_vec(ti));
            dev.ks_tw = tables.back().as<ulonglong2>();
            tables.push_back(upload_vec(tf));
            dev.ks_tw_f = tables.back().as<double>();
        }
    }
    // limb 0 via limbs 1..3 (keyswitch.cu "aux"): the 60-bit q0 alone on the
    // integer pipes, q1..q3 on the FP64 pipe
    if (ring.limbs >= 4 && ring.primes[0] >= (1ull << 42) && ring.primes[1] < (1ull << 42) &&
        ring.primes[2] < (1ull << 42) && ring.primes[3] < (1ull << 42)) {
        using u128 = unsigned __int128;
        const u128 Pq = static_cast<u128>(ring.primes[1]) * ring.primes[2] * ring.primes[3];
        for (int a = 0; a < 3; ++a) {
            const u64 qa = ring.primes[1 + a];
            const u128 Ma = Pq / qa;
            const u64 inv = ring.mods[1 + a].inv(static_cast<u64>(Ma % qa));
            dev.aux_inv[a] = make_ulonglong2(inv, shoup_of(inv, qa));
            const u64 mq0 = static_cast<u64>(Ma % ring.primes[0]);
            dev.aux_Mq0[a] = make_ulonglong2(mq0, shoup_of(mq0, ring.primes[0]));
        }
        for (int k = 0; k < 4; ++k) dev.aux_kPq0[k] = static_cast<u64>((Pq % ring.primes[0]) * k % ring.primes[0]);
        dev.aux_log2P = std::log2(static_cast<double>(ring.primes[1])) + std::log2(static_cast<double>(ring.primes[2])) +
                        std::log2(static_cast<double>(ring.primes[3]));
    }
    dev.n = static_cast<int>(ring.n);
    dev.logn = static_cast<int>(ring.logn);
    dev.limbs = static_cast<int>(ring.limbs);
    for (std::size_t i = 0; i < ring.limbs; ++i) {
        if (ring.primes[i] >= (1ull << 42)) dev.int_limbs |= (i < 64 ? 1ull << i : 0ull);
        if (ring.primes[i] <= (1ull << 20)) dev.small_primes = true;
    }
    if (ring.limbs > 64) throw std::invalid_argument("modulus chains longer than 64 limbs are not supported");
    dev.crt_words = static_cast<int>(ring.crt_words);
    sync();
}

Context::~Context() {
    cudaSetDevice(device);
    cudaStreamSynchronize(stream);
    prof.collect();
    for (cudaEvent_t e : prof.pool) cudaEventDestroy(e);
    s_ntt.reset();
    pk.reset();
    aux_tab.reset();
    evk.reset();
    evk_sh.reset();
    evk_f.reset();
    tables.clear();
    cudaStreamSynchronize(stream);
    cudaStreamSynchronize(aux);
    if (own_stream) cudaStreamDestroy(stream);
    cudaStreamDestroy(aux);
    cudaEventDestroy(fork_ev);
    cudaEventDestroy(join_ev);
}

void Context::upload(void* dst, const void* src, std::size_t bytes) {
    cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, stream), "cudaMemcpyAsync H2D");
    // A pageable source has been staged when cudaMemcpyAsync returns, so the
    // caller may reuse it and the stream keeps running (the engine's small
    // constant tables). A pinned source is read by the DMA later: wait, so the
    // caller's buffer-lifetime rule stays "valid for the duration of the call".
    cudaPointerAttributes a{};
    const bool pinned = cudaPointerGetAttributes(&a, src) == cudaSuccess && a.type == cudaMemoryTypeHost;
    cudaGetLastError();  // clear a possible "invalid value" from the query
    if (pinned) cuda_check(cudaStreamSynchronize(stream), "cudaStreamSynchronize");
}

void Context::download(void* dst, const void* src, std::size_t bytes) {
    cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, stream), "cudaMemcpyAsync D2H");
    cuda_check(cudaStreamSynchronize(stream), "cudaStreamSynchronize");
}

void Context::sync() { cuda_check(cudaStreamSynchronize(stream), "cudaStreamSynchronize"); }

double measure_modmul_peak(Context& C, bool fp64) {
    DevBuf sink(&C, 64);
    Launch L = C.L();
    auto probe = fp64 ? fp64_modmul_probe : modmul_probe;
    probe(C.dev, 64, sink.as<u64>(), L);  // warm-up
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 4096;
    cudaEventRecord(a, C.stream);
    double ops = probe(C.dev, iters, sink.as<u64>(), L);
    cudaEventRecord(b, C.stream);
    C.sync();
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return ops / (ms * 1e-3);
}

TensorPtr make_tensor(Context& C, std::size_t cells, std::uint32_t level, double scale) {
    auto t = std::make_unique<Tensor>();
    t->ctx = &C;
    t->cells = cells;
    t->level = level;
    t->scale = scale;
    t->shape = Shape::flattened(cells);
    t->buf = DevBuf(&C, cells * 2 * (level + 1) * C.n() * sizeof(u64));
    return t;
}

// ---------------------------------------------------------------- keys

// CkksEngine::keygen (ckks.hpp:200-236): host randomness, device arithmetic.
void keygen(Context& C, u64 seed) {
    const std::size_t n = C.n(), top = C.top(), limbs = top + 1, poly = limbs * n;
    Launch L = C.L();
    auto residues_of = [&](const std::vector<long long>& c) {
        std::vector<u64> r(poly);
        for (std::size_t i = 0; i < limbs; ++i)
            for (std::size_t j = 0; j < n; ++j) r[i * n + j] = C.ring.mods[i].from_signed(c[j]);
        return r;
    };
    std::vector<long long> s = sample_secretish(C, 2.0 / 3.0, derive_seed(seed, 0x5ec0));
    C.secret_host = residues_of(s);
    C.s_ntt = C.upload_vec(C.secret_host);
    ntt_forward(C.dev, C.s_ntt.as<u64>(), static_cast<int>(top), 1, L);

    // public key
    DevBuf a = C.upload_vec(sample_uniform(C.ring, top, derive_seed(seed, 0xa0a0)));
    ntt_forward(C.dev, a.as<u64>(), static_cast<int>(top), 1, L);
    DevBuf e = C.upload_vec(residues_of(sample_error(C, derive_seed(seed, 0xe000))));
    ntt_forward(C.dev, e.as<u64>(), static_cast<int>(top), 1, L);
    C.pk = DevBuf(&C, 2 * poly * sizeof(u64));
    u64* pkb = C.pk.as<u64>();
    u64* pka = pkb + poly;
    poly_elementwise(C.dev, EwOp::Mul, a.as<u64>(), C.s_ntt.as<u64>(), pkb, static_cast<int>(top), 1, L);
    poly_elementwise(C.dev, EwOp::Neg, pkb, nullptr, pkb, static_cast<int>(top), 1, L);
    poly_elementwise(C.dev, EwOp::Add, pkb, e.as<u64>(), pkb, static_cast<int>(top), 1, L);
    cuda_check(cudaMemcpyAsync(pka, a.get(), poly * sizeof(u64), cudaMemcpyDeviceToDevice, C.stream), "copy pk.a");

    // evaluation key: b_t = -a_t s + e_t + 2^{20 t} s^2 (NTT domain, top level)
    const std::size_t D = C.ring.relin_digits(top);
    DevBuf s2(&C, poly * sizeof(u64));
    poly_elementwise(C.dev, EwOp::Mul, C.s_ntt.as<u64>(), C.s_ntt.as<u64>(), s2.as<u64>(), static_cast<int>(top), 1, L);
    std::vector<std::vector<u64>> at(D), et(D);
    parallel_items(D, [&](std::size_t t) {
        at[t] = sample_uniform(C.ring, top, derive_seed(seed, 0xeb00 + 2 * t));
        et[t] = residues_of(sample_error(C, derive_seed(seed, 0xeb01 + 2 * t)));
    });
    C.evk = DevBuf(&C, D * 2 * poly * sizeof(u64));
    C.evk_sh = DevBuf(&C, D * 2 * poly * sizeof(u64));
    DevBuf et_dev(&C, poly * sizeof(u64));
    DevBuf consts(&C, limbs * sizeof(ulonglong2));
    for (std::size_t t = 0; t < D; ++t) {
        u64* bt = C.evk.as<u64>() + (2 * t) * poly;
        u64* a_t = bt + poly;
        C.upload(a_t, at[t].data(), poly * sizeof(u64));
        ntt_forward(C.dev, a_t, static_cast<int>(top), 1, L);
        C.upload(et_dev.get(), et[t].data(), poly * sizeof(u64));
        ntt_forward(C.dev, et_dev.as<u64>(), static_cast<int>(top), 1, L);
        poly_elementwise(C.dev, EwOp::Mul, a_t, C.s_ntt.as<u64>(), bt, static_cast<int>(top), 1, L);
        poly_elementwise(C.dev, EwOp::Neg, bt, nullptr, bt, static_cast<int>(top), 1, L);
        poly_elementwise(C.dev, EwOp::Add, bt, et_dev.as<u64>(), bt, static_cast<int>(top), 1, L);
        std::vector<u64> f(limbs);
        for (std::size_t i = 0; i < limbs; ++i) f[i] = C.ring.mods[i].pow(2, 20 * t);
        std::vector<ulonglong2> fc = with_shoup(C.ring, f);
        C.upload(consts.get(), fc.data(), limbs * sizeof(ulonglong2));
        scalar_mul(C.dev, s2.as<u64>(), consts.as<ulonglong2>(), et_dev.as<u64>(), static_cast<int>(top), 1, L);
        poly_elementwise(C.dev, EwOp::Add, bt, et_dev.as<u64>(), bt, static_cast<int>(top), 1, L);
    }
    shoup_table(C.dev, C.evk.as<u64>(), C.evk_sh.as<u64>(), static_cast<int>(limbs), 2 * D, L);
    C.evk_f = DevBuf(&C, D * 2 * poly * sizeof(double));
    fp_table(C.dev, C.evk.as<u64>(), C.evk_f.as<double>(), static_cast<int>(limbs), 2 * D, L);
    C.evk_digits = D;
    C.has_secret = C.has_pk = true;
    C.build_aux_tables();
    C.sync();
}

void Context::build_aux_tables() {
    aux_tab.reset();
    dev.aux_tab = nullptr;
    if (dev.aux_log2P <= 0.0 || !evk_digits || ring.logn < 10 || ring.logn > 14) return;
    const std::size_t nn = n(), rows = 2 * evk_digits;
    aux_tab = DevBuf(this, rows * 4 * nn * sizeof(double));
    DevBuf tmp(this, rows * 5 * nn * sizeof(u64));
    keyswitch_aux_tables(dev, evk.as<u64>(), top() + 1, static_cast<int>(evk_digits), aux_tab.as<double>(),
                         tmp.as<u64>(), L());
    dev.aux_tab = aux_tab.as<double>();
    sync();
}

void import_keys(Context& C, const u64* secret, const u64* pk_b, const u64* pk_a, const u64* evk, std::size_t digits) {
    const std::size_t poly = (C.top() + 1) * C.n();
    Launch L = C.L();
    if (secret) {
        C.secret_host.assign(secret, secret + poly);
        C.s_ntt = C.upload_vec(C.secret_host);
        ntt_forward(C.dev, C.s_ntt.as<u64>(), static_cast<int>(C.top()), 1, L);
        C.has_secret = true;
    }
    if (pk_b && pk_a) {
        C.pk = DevBuf(&C, 2 * poly * sizeof(u64));
        C.upload(C.pk.get(), pk_b, poly * sizeof(u64));
        C.upload(C.pk.as<u64>() + poly, pk_a, poly * sizeof(u64));
        C.has_pk = true;
    }
    if (evk && digits) {
        C.evk = DevBuf(&C, digits * 2 * poly * sizeof(u64));
        C.evk_sh = DevBuf(&C, digits * 2 * poly * sizeof(u64));
        C.upload(C.evk.get(), evk, digits * 2 * poly * sizeof(u64));
        shoup_table(C.dev, C.evk.as<u64>(), C.evk_sh.as<u64>(), static_cast<int>(C.top() + 1), 2 * digits, L);
        C.evk_f = DevBuf(&C, digits * 2 * poly * sizeof(double));
        fp_table(C.dev, C.evk.as<u64>(), C.evk_f.as<double>(), static_cast<int>(C.top() + 1), 2 * digits, L);
        C.evk_digits = digits;
        C.build_aux_tables();
    }
    C.sync();
}

// ---------------------------------------------------------------- scheme ops

TensorPtr ct_add(Context& C, const Tensor& x, const Tensor& y, bool subtract) {
    const char* op = subtract ? "sub" : "add";
    if (x.level != y.level)
        throw std::invalid_argument(std::string(op) + ": level mismatch (use rescale/mod_switch first)");
    require_scale_match(x.scale, y.scale, op);
    if (x.cells != y.cells) throw std::invalid_argument(std::string(op) + ": cell count mismatch");
    TensorPtr out = make_tensor(C, x.cells, x.level, x.scale);
    out->shape = x.shape;
    out->batch = x.batch;
    poly_elementwise(C.dev, subtract ? EwOp::Sub : EwOp::Add, x.data(), y.data(), out->data(),
                     static_cast<int>(x.level), 2 * x.cells, C.L());
    return out;
}

void key_switch_raw(Context& C, const u64* d2, u64* out, std::size_t level, std::size_t count) {
    if (!C.evk_digits) throw std::invalid_argument("mul: empty evaluation key");
    const std::size_t D = C.ring.relin_digits(level);
    if (D > C.evk_digits) throw std::invalid_argument("mul: evaluation key too short for level");
    const std::size_t n = C.n(), limbs = level + 1;
    Launch L = C.L();
    DevBuf tmp(&C, count * limbs * n * sizeof(u64));
    DevBuf dig(&C, count * D * n * sizeof(u32));
    cuda_check(cudaMemcpyAsync(tmp.get(), d2, count * limbs * n * sizeof(u64), cudaMemcpyDeviceToDevice, C.stream), "copy");
    crt_digits(C.dev, tmp.as<u64>(), dig.as<u32>(), static_cast<int>(level), static_cast<int>(D), count, L);
    cuda_check(cudaMemsetAsync(out, 0, count * 2 * limbs * n * sizeof(u64), C.stream), "memset");
    DevBuf aux(&C, keyswitch_aux_ok(C.dev, static_cast<int>(level), static_cast<int>(D)) ? count * 10 * n * 8 : 0);
    keyswitch_mac(C.dev, dig.as<u32>(), C.evk.as<u64>(), C.evk_sh.as<u64>(), C.evk_f.as<double>(), out,
                  static_cast<int>(level), static_cast<int>(D), count, L, 0, nullptr, aux.as<u64>());
}

// mul / square (ckks.hpp:315-369): tensor -> INTT(d2) -> key switch -> INTT -> rescale.
static TensorPtr relin_product(Context& C, const Tensor& x, const Tensor* y) {
    Trace tr("relin_product");
    const bool sq = y == nullptr;
    if (!sq) {
        if (x.level != y->level) throw std::invalid_argument("mul: level mismatch (use rescale/mod_switch first)");
        if (x.cells != y->cells) throw std::invalid_argument("mul: cell count mismatch");
    }
    if (x.level == 0) throw std::invalid_argument("mul: at last level, no room to rescale");
    const double sy = sq ? x.scale : y->scale;
    check_scale_headroom(C, x.scale, sy, x.level);
    if (!C.evk_digits) throw std::invalid_argument("mul: empty evaluation key");
    const std::size_t l = x.level, n = C.n(), limbs = l + 1;
    const std::size_t D = C.ring.relin_digits(l);
    if (D > C.evk_digits) throw std::invalid_argument("mul: evaluation key too short for level");

    TensorPtr out = make_tensor(C, x.cells, static_cast<std::uint32_t>(l - 1),
                                x.scale * sy / static_cast<double>(C.ring.primes[l]));
    out->shape = x.shape;
    out->batch = x.batch;
    const std::size_t cw = 2 * limbs * n;
    const bool aux = keyswitch_aux_ok(C.dev, static_cast<int>(l), static_cast<int>(D));
    const std::size_t aux_words = aux ? 10 * n : 0;  // limb 0 via limbs 1..3: [2][4][n] + [2][n]
    const std::size_t per_ct = (sq ? 1 : 2) * cw * 8 + limbs * n * 8 + D * n * 4 + aux_words * 8;
    const std::size_t chunk = std::max<std::size_t>(1, std::min(x.cells, kScratchBytes / per_ct));
    DevBuf d01(&C, chunk * cw * 8), fy(&C, sq ? 0 : chunk * cw * 8), d2(&C, chunk * limbs * n * 8),
        dig(&C, chunk * D * n * 4), auxs(&C, chunk * aux_words * 8);
    Launch L = C.L();
    const int lv = static_cast<int>(l);
    for (std::size_t c0 = 0; c0 < x.cells; c0 += chunk) {
        const std::size_t m = std::min(chunk, x.cells - c0);
        // tensor product fused away: d2 = x1 y1 is formed in the INTT's first
        // round, (d0, d1) in the key-switch epilogue (both from NTT(x), NTT(y))
        ntt_forward_to(C.dev, x.cell(c0), d01.as<u64>(), lv, 2 * m, L);
        if (!sq) ntt_forward_to(C.dev, y->cell(c0), fy.as<u64>(), lv, 2 * m, L);
        const u64* fyp = sq ? d01.as<u64>() : fy.as<u64>();
        ntt_inverse_product(C.dev, d01.as<u64>(), fyp, d2.as<u64>(), lv, m, L);
        crt_digits(C.dev, d2.as<u64>(), dig.as<u32>(), lv, static_cast<int>(D), m, L);
        // limb 0's E (aux path) stays in coefficients and joins after the INTT
        const u64* e0 = keyswitch_mac(C.dev, dig.as<u32>(), C.evk.as<u64>(), C.evk_sh.as<u64>(),
                                      C.evk_f.as<double>(), d01.as<u64>(), lv, static_cast<int>(D), m, L, sq ? 1 : 2,
                                      sq ? nullptr : fy.as<u64>(), aux ? auxs.as<u64>() : nullptr, true);
        if (!ntt_inverse_rescale(C.dev, d01.as<u64>(), out->cell(c0), lv, 2 * m, L, e0)) {
            ntt_inverse(C.dev, d01.as<u64>(), lv, 2 * m, L);
            if (e0) add_limb0(C.dev, d01.as<u64>(), e0, lv + 1, 2 * m, L);
            rescale(C.dev, d01.as<u64>(), out->cell(c0), lv, 2 * m, L);
        }
    }
    return out;
}

TensorPtr ct_mul(Context& C, const Tensor& x, const Tensor& y) { return relin_product(C, x, &y); }
TensorPtr ct_square(Context& C, const Tensor& x) { return relin_product(C, x, nullptr); }

TensorPtr ct_rescale(Context& C, const Tensor& x) {
    if (x.level == 0) throw std::invalid_argument("rescale: no level headroom");
    TensorPtr out = make_tensor(C, x.cells, x.level - 1, x.scale / static_cast<double>(C.ring.primes[x.level]));
    out->shape = x.shape;
    out->batch = x.batch;
    rescale(C.dev, x.data(), out->data(), static_cast<int>(x.level), 2 * x.cells, C.L());
    return out;
}

TensorPtr ct_mod_switch(Context& C, const Tensor& x, std::uint32_t to_level) {
    if (to_level > x.level) throw std::invalid_argument("mod_switch: cannot raise level");
    TensorPtr out = make_tensor(C, x.cells, to_level, x.scale);
    out->shape = x.shape;
    out->batch = x.batch;
    if (to_level == x.level)
        cuda_check(cudaMemcpyAsync(out->data(), x.data(), x.cells * x.cell_words() * 8, cudaMemcpyDeviceToDevice, C.stream),
                   "copy");
    else
        drop_limbs(C.dev, x.data(), out->data(), static_cast<int>(x.level), static_cast<int>(to_level), 2 * x.cells, C.L());
    return out;
}

// encode_const + mul_plain's checks (ckks.hpp:372-382, 395-398), then the constant's
// residues with Shoup companions on the device
static DevBuf mul_const_table(Context& C, const Tensor& x, double c, double scale) {
    C.enc->check_encode(1, std::abs(c), scale, x.level);
    std::vector<u64> res =
        C.enc->residues_of_rounded(roundl(static_cast<long double>(c) * static_cast<long double>(scale)), x.level);
    if (x.level == 0) throw std::invalid_argument("mul_plain: at last level, no room to rescale");
    check_scale_headroom(C, x.scale, scale, x.level);
    return C.upload_vec(with_shoup(C.ring, res));
}

// mul_plain(x, encode_const(c, scale, x.level)) (ckks.hpp:395-398, 372-382, 588-597)
TensorPtr ct_mul_const(Context& C, const Tensor& x, double c, double scale) {
    DevBuf dc = mul_const_table(C, x, c, scale);
    Launch L = C.L();
    const double raw_scale = x.scale * scale;
    TensorPtr out = make_tensor(C, x.cells, x.level - 1, raw_scale / static_cast<double>(C.ring.primes[x.level]));
    out->shape = x.shape;
    out->batch = x.batch;
    // the product x * c is consumed inside the rescale kernel, never stored
    rescale(C.dev, x.data(), out->data(), static_cast<int>(x.level), 2 * x.cells, L, dc.as<ulonglong2>());
    return out;
}

// add_plain(x, encode_const(c, x.scale, x.level)) (ckks.hpp:305-311)
TensorPtr ct_add_const(Context& C, const Tensor& x, double c) {
    C.enc->check_encode(1, std::abs(c), x.scale, x.level);
    std::vector<u64> res =
        C.enc->residues_of_rounded(roundl(static_cast<long double>(c) * static_cast<long double>(x.scale)), x.level);
    DevBuf dc = C.upload_vec(res);
    TensorPtr out = make_tensor(C, x.cells, x.level, x.scale);
    out->shape = x.shape;
    out->batch = x.batch;
    cuda_check(cudaMemcpyAsync(out->data(), x.data(), x.cells * x.cell_words() * 8, cudaMemcpyDeviceToDevice, C.stream),
               "copy");
    add_coeff0(C.dev, out->data(), dc.as<u64>(), static_cast<int>(x.level), x.cells, C.L());
    return out;
}

// ---------------------------------------------------------------- scalar fast path / plaintexts

// CkksEngine::make_scalar_plain (ckks.hpp:407-423)
ScalarPlain make_scalar_plain(const Context& C, double c, double scale, std::size_t level) {
    C.enc->check_encode(1, std::abs(c), scale, level);
    ScalarPlain sp;
    sp.scale = scale;
    sp.level = static_cast<std::uint32_t>(level);
    sp.residues = C.enc->residues_of_rounded(roundl(static_cast<long double>(c) * static_cast<long double>(scale)), level);
    return sp;
}

// make_zero_ciphertext (ckks.hpp:431-438)
TensorPtr ct_zero(Context& C, std::size_t cells, std::uint32_t level, double scale) {
    if (level > C.top()) throw std::invalid_argument("make_zero_ciphertext: level above the chain");
    TensorPtr out = make_tensor(C, cells, level, scale);
    cuda_check(cudaMemsetAsync(out->data(), 0, cells * out->cell_words() * 8, C.stream), "memset");
    return out;
}

// add_inplace (ckks.hpp:440-445)
void ct_add_inplace(Context& C, Tensor& acc, const Tensor& x) {
    if (acc.level != x.level) throw std::invalid_argument("add: level mismatch (use rescale/mod_switch first)");
    require_scale_match(acc.scale, x.scale, "add");
    if (acc.cells != x.cells) throw std::invalid_argument("add: cell count mismatch");
    poly_elementwise(C.dev, EwOp::Add, acc.data(), x.data(), acc.data(), static_cast<int>(acc.level), 2 * acc.cells,
                     C.L());
}

static void check_residues(const Context& C, const u64* r, std::size_t rows, std::size_t limbs, std::size_t stride,
                           const char* what) {
    for (std::size_t k = 0; k < rows; ++k)
        for (std::size_t i = 0; i < limbs; ++i)
            if (r[k * limbs * stride + i * stride] >= C.ring.primes[i])
                throw std::invalid_argument(std::string(what) + ": residue not below its prime");
}

// mul_scalar_mac (ckks.hpp:448-465)
void ct_scalar_mac(Context& C, Tensor& acc, const Tensor& x, const u64* residues, std::size_t ncs, double sp_scale,
                   std::uint32_t sp_level) {
    if (x.level != acc.level || sp_level != acc.level) throw std::invalid_argument("mul_scalar_mac: level mismatch");
    require_scale_match(acc.scale, x.scale * sp_scale, "mul_scalar_mac");
    if (acc.cells != x.cells) throw std::invalid_argument("mul_scalar_mac: cell count mismatch");
    if (ncs != 1 && ncs != acc.cells) throw std::invalid_argument("mul_scalar_mac: one scalar, or one per cell");
    const std::size_t limbs = acc.level + 1;
    check_residues(C, residues, ncs, limbs, 1, "mul_scalar_mac");
    std::vector<ulonglong2> cs(ncs * limbs);
    for (std::size_t k = 0; k < ncs; ++k)
        for (std::size_t i = 0; i < limbs; ++i) {
            const u64 r = residues[k * limbs + i];
            cs[k * limbs + i] = make_ulonglong2(r, shoup_of(r, C.ring.primes[i]));
        }
    DevBuf dc = C.upload_vec(cs);
    scalar_mac(C.dev, x.data(), dc.as<ulonglong2>(), ncs, acc.data(), static_cast<int>(acc.level), acc.cells, C.L());
}

// add_scalar_inplace (ckks.hpp:468-472)
void ct_add_scalar(Context& C, Tensor& ct, double c) {
    const ScalarPlain sp = make_scalar_plain(C, c, ct.scale, ct.level);
    DevBuf dc = C.upload_vec(sp.residues);
    add_coeff0(C.dev, ct.data(), dc.as<u64>(), static_cast<int>(ct.level), ct.cells, C.L());
}

// add_plain (ckks.hpp:305-311)
TensorPtr ct_add_plain(Context& C, const Tensor& x, const u64* pt, std::uint32_t pt_level, double pt_scale) {
    if (pt_level != x.level) throw std::invalid_argument("add_plain: level mismatch");
    require_scale_match(x.scale, pt_scale, "add_plain");
    const std::size_t n = C.n(), limbs = x.level + 1;
    for (std::size_t i = 0; i < limbs; ++i)
        for (std::size_t j = 0; j < n; ++j)
            if (pt[i * n + j] >= C.ring.primes[i]) throw std::invalid_argument("add_plain: residue not below its prime");
    DevBuf dp = C.upload_vec(std::vector<u64>(pt, pt + limbs * n));
    TensorPtr out = make_tensor(C, x.cells, x.level, x.scale);
    out->shape = x.shape;
    out->batch = x.batch;
    plain_bcast(C.dev, x.data(), dp.as<u64>(), out->data(), static_cast<int>(x.level), x.cells, 0, C.L());
    return out;
}

// mul_plain_raw / mul_plain (ckks.hpp:372-398): a constant plaintext multiplies
// every coefficient by its coefficient 0 (scalar_mul, :588-597), any other goes
// through the NTT
TensorPtr ct_mul_plain(Context& C, const Tensor& x, const u64* pt, std::uint32_t pt_level, double pt_scale,
                       bool is_constant, bool rescale) {
    if (rescale && x.level == 0) throw std::invalid_argument("mul_plain: at last level, no room to rescale");
    if (pt_level != x.level) throw std::invalid_argument("mul_plain: level mismatch");
    check_scale_headroom(C, x.scale, pt_scale, x.level);
    const std::size_t n = C.n(), limbs = x.level + 1;
    for (std::size_t i = 0; i < limbs; ++i)
        for (std::size_t j = 0; j < (is_constant ? 1 : n); ++j)
            if (pt[i * n + j] >= C.ring.primes[i]) throw std::invalid_argument("mul_plain: residue not below its prime");
    TensorPtr raw = make_tensor(C, x.cells, x.level, x.scale * pt_scale);
    raw->shape = x.shape;
    raw->batch = x.batch;
    const int lv = static_cast<int>(x.level);
    Launch L = C.L();
    if (is_constant) {
        std::vector<u64> c0(limbs);
        for (std::size_t i = 0; i < limbs; ++i) c0[i] = pt[i * n];
        DevBuf dc = C.upload_vec(with_shoup(C.ring, c0));
        scalar_mul(C.dev, x.data(), dc.as<ulonglong2>(), raw->data(), lv, 2 * x.cells, L);
    } else {
        DevBuf dp = C.upload_vec(std::vector<u64>(pt, pt + limbs * n));
        ntt_forward(C.dev, dp.as<u64>(), lv, 1, L);
        ntt_forward_to(C.dev, x.data(), raw->data(), lv, 2 * x.cells, L);
        plain_bcast(C.dev, raw->data(), dp.as<u64>(), raw->data(), lv, x.cells, 1, L);
        ntt_inverse(C.dev, raw->data(), lv, 2 * x.cells, L);
    }
    return rescale ? ct_rescale(C, *raw) : std::move(raw);
}

// ---------------------------------------------------------------- activation

std::size_t Activation::encrypted_depth() const {
    std::size_t d = degree(), lg = 0;
    while ((std::size_t(1) << lg) < d) ++lg;
    return lg + 1;
}

void Activation::validate() const {
    if (degree() < 1) throw std::invalid_argument("PolyActivation: degree must be >= 1");
    for (double c : coefficients)
        if (!std::isfinite(c)) throw std::invalid_argument("PolyActivation: non-finite coefficient");
    if (!(interval_bound > 0)) throw std::invalid_argument("PolyActivation: interval bound must be > 0");
}

// eval_encrypted (activation.hpp:228-265): power-basis plan over whole tensors.
static TensorPtr eval_activation_cells(Context& C, const Activation& act, const Tensor& x, u64* dst) {
    Trace tr("eval_activation");
    act.validate();
    const std::size_t d = act.degree(), depth = act.encrypted_depth();
    if (x.level < depth) throw std::invalid_argument("eval_encrypted: insufficient depth budget");
    std::map<std::size_t, TensorPtr> powers;
    std::function<const Tensor&(std::size_t)> power = [&](std::size_t k) -> const Tensor& {
        if (k == 1) return x;
        auto it = powers.find(k);
        if (it != powers.end()) return *it->second;
        if (k % 2 == 0) {
            TensorPtr sq = ct_square(C, power(k / 2));
            return *powers.emplace(k, std::move(sq)).first->second;
        }
        const Tensor& hi = power((k + 1) / 2);
        const Tensor& lo = power(k / 2);
        std::uint32_t lvl = std::min(hi.level, lo.level);
        TensorPtr h = ct_mod_switch(C, hi, lvl), l = ct_mod_switch(C, lo, lvl);
        TensorPtr prod = ct_mul(C, *h, *l);
        return *powers.emplace(k, std::move(prod)).first->second;
    };
    const double target = C.scale;
    std::vector<TensorPtr> terms;
    // degree 2: the linear term c1 x is not stored -- its mul_plain + rescale
    // runs inside the final fused kernel (SumTerms::rs), read straight from x
    DevBuf lazy_c;
    bool lazy = false;
    double lazy_scale = 0.0;
    for (std::size_t k = 1; k < d; ++k) {
        const Tensor& p = power(k);
        double u = target * static_cast<double>(C.ring.primes[p.level]) / p.scale;
        if (k == 1 && d == 2) {
            lazy_c = mul_const_table(C, p, act.coefficients[k], u);  // the same checks, in order
            lazy_scale = p.scale * u / static_cast<double>(C.ring.primes[p.level]);
            lazy = true;
            continue;
        }
        terms.push_back(ct_mul_const(C, p, act.coefficients[k], u));
    }
    auto materialize_lazy = [&] {
        if (!lazy) return;
        TensorPtr t = make_tensor(C, x.cells, x.level - 1, lazy_scale);
        t->shape = x.shape;
        t->batch = x.batch;
        rescale(C.dev, x.data(), t->data(), static_cast<int>(x.level), 2 * x.cells, C.L(), lazy_c.as<ulonglong2>());
        terms.insert(terms.begin(), std::move(t));
        lazy = false;
    };
    {
        // The last term (the highest power, lowest level) is rescaled with the
        // other terms and the constant added on the way out when its level is
        // the output level; checks keep the reference's order.
        const Tensor& p = power(d);
        const double u = target * static_cast<double>(C.ring.primes[p.level]) / p.scale;
        const std::uint32_t lvl = p.level - (p.level ? 1 : 0);
        bool fuse = p.level > 0 && terms.size() + 1 <= static_cast<std::size_t>(kMaxTerms);
        for (auto& t : terms) fuse = fuse && t->level >= lvl;
        // the fused kernel reads x for the lazy term: not when its output would overwrite x
        const auto xb = reinterpret_cast<std::uintptr_t>(x.data()), db = reinterpret_cast<std::uintptr_t>(dst);
        const bool dst_overlaps_x = dst && db < xb + x.cells * x.cell_words() * 8 &&
                                    xb < db + x.cells * 2 * (lvl + 1) * C.n() * 8;
        if (lazy && !(fuse && x.level - 1 >= lvl && !dst_overlaps_x)) materialize_lazy();
        if (fuse) {
            DevBuf dc = mul_const_table(C, p, act.coefficients[d], u);
            const double sc = p.scale * u / static_cast<double>(C.ring.primes[p.level]);
            // the terms in the reference's order: [c1 x (lazy)], materialized terms, c_d x^d
            std::vector<double> scales;
            if (lazy) scales.push_back(lazy_scale);
            for (auto& t : terms) scales.push_back(t->scale);
            const double s0 = scales.empty() ? sc : scales[0];
            for (std::size_t i = 1; i < scales.size(); ++i) require_scale_match(s0, scales[i], "add");
            if (!scales.empty()) require_scale_match(s0, sc, "add");
            SumTerms st{};
            if (lazy) {
                st.rs = x.data();
                st.rs_level = static_cast<int>(x.level);
                st.rs_c = lazy_c.as<ulonglong2>();
            }
            st.count = static_cast<int>(terms.size());
            for (std::size_t i = 0; i < terms.size(); ++i) {
                st.ptr[i] = terms[i]->data();
                st.limbs[i] = static_cast<int>(terms[i]->level + 1);
            }
            DevBuf d0;
            if (act.coefficients[0] != 0.0) {
                const double c = act.coefficients[0];
                C.enc->check_encode(1, std::abs(c), s0, lvl);
                d0 = C.upload_vec(
                    C.enc->residues_of_rounded(roundl(static_cast<long double>(c) * static_cast<long double>(s0)), lvl));
                st.c0 = d0.as<u64>();
            }
            TensorPtr acc = dst ? std::make_unique<Tensor>() : make_tensor(C, x.cells, lvl, s0);
            if (dst) {  // written straight into the caller's storage
                acc->ctx = &C;
                acc->cells = x.cells;
                acc->level = lvl;
                acc->scale = s0;
                acc->buf = DevBuf::alias(dst, x.cells * 2 * (lvl + 1) * C.n() * 8);
            }
            rescale(C.dev, p.data(), acc->data(), static_cast<int>(p.level), 2 * x.cells, C.L(), dc.as<ulonglong2>(),
                    &st);
            acc->shape = x.shape;
            acc->batch = x.batch;
            return acc;
        }
        materialize_lazy();
        terms.push_back(ct_mul_const(C, p, act.coefficients[d], u));
    }
    std::uint32_t out_level = terms.back()->level;
    for (auto& t : terms) out_level = std::min(out_level, t->level);
    // (more than kMaxTerms terms: the reference's chain of mod_switch / add / add_const)
    TensorPtr acc = ct_mod_switch(C, *terms[0], out_level);
    for (std::size_t i = 1; i < terms.size(); ++i) {
        TensorPtr t = ct_mod_switch(C, *terms[i], out_level);
        acc = ct_add(C, *acc, *t, false);
    }
    if (act.coefficients[0] != 0.0) acc = ct_add_const(C, *acc, act.coefficients[0]);
    acc->shape = x.shape;
    acc->batch = x.batch;
    if (dst) {
        cuda_check(cudaMemcpyAsync(dst, acc->data(), x.cells * acc->cell_words() * 8, cudaMemcpyDeviceToDevice, C.stream),
                   "copy activation");
        TensorPtr view = std::make_unique<Tensor>();
        view->ctx = &C;
        view->cells = acc->cells;
        view->level = acc->level;
        view->scale = acc->scale;
        view->shape = acc->shape;
        view->batch = acc->batch;
        view->buf = DevBuf::alias(dst, x.cells * acc->cell_words() * 8);
        return view;
    }
    return acc;
}

// Non-owning tensor over cells [c0, c0 + m) of x.
static TensorPtr cell_slice(const Tensor& x, std::size_t c0, std::size_t m) {
    auto t = std::make_unique<Tensor>();
    t->ctx = x.ctx;
    t->cells = m;
    t->level = x.level;
    t->scale = x.scale;
    t->shape = Shape::flattened(m);
    t->batch = x.batch;
    t->buf = DevBuf::alias(x.cell(c0), m * x.cell_words() * 8);
    return t;
}

// The power plan is identical for every cell, so large tensors are evaluated
// in cell chunks written straight into the output: peak memory is input +
// output + one chunk's intermediates instead of every full-size power/term.
TensorPtr eval_activation(Context& C, const Activation& act, const Tensor& x, u64* dst) {
    const std::size_t per_cell = x.cell_words() * 8;
    const std::size_t chunk = std::max<std::size_t>(1, (std::size_t(6) << 30) / (per_cell * 6));
    if (x.cells <= chunk) return eval_activation_cells(C, act, x, dst);
    TensorPtr out;
    for (std::size_t c0 = 0; c0 < x.cells; c0 += chunk) {
        const std::size_t m = std::min(chunk, x.cells - c0);
        if (out) {  // later chunks land in place
            eval_activation_cells(C, act, *cell_slice(x, c0, m), out->cell(c0));
            continue;
        }
        TensorPtr part = eval_activation_cells(C, act, *cell_slice(x, c0, m), dst);
        if (dst) {
            out = std::make_unique<Tensor>();
            out->ctx = &C;
            out->cells = x.cells;
            out->level = part->level;
            out->scale = part->scale;
            out->buf = DevBuf::alias(dst, x.cells * part->cell_words() * 8);
        } else {
            out = make_tensor(C, x.cells, part->level, part->scale);
            cuda_check(cudaMemcpyAsync(out->cell(c0), part->data(), m * part->cell_words() * 8,
                                       cudaMemcpyDeviceToDevice, C.stream),
                       "copy activation chunk");
        }
    }
    out->shape = x.shape;
    out->batch = x.batch;
    return out;
}

// ---------------------------------------------------------------- encryption

namespace detail {

// Public-key encryptions of `count` messages (or zeros) at limbs 0..level,
// randomness from make_encryption_randomness(seeds[i]) (ckks.hpp:238-266).
// out: [count][2][level+1][n] device.
// One chunk of host-side encryption inputs: randomness (int8) and the
// message as i64 coefficients (small) or full residues.
struct HostChunk {
    std::vector<signed char> r, e0, e1;
    std::vector<long long> mi;
    std::vector<u64> mres;
    bool small = true;
};
using ChunkFn = std::function<void(std::size_t c0, std::size_t m, HostChunk&)>;

// Public-key encryptions of `count` cells at limbs 0..level into out, in
// chunks: the host work of chunk k + 1 (sampling, and the encode for
// encrypt_tensor) runs on a host thread while chunk k's uploads and device
// arithmetic (NTT, key products, INTT, noise + message) are issued -- pageable
// uploads return once staged, so two host buffers alternate.
void encrypt_pipelined(Context& C, std::size_t count, std::uint32_t level, u64* out, bool with_msgs,
                       const ChunkFn& produce) {
    if (!C.has_pk) throw std::invalid_argument("encrypt: no public key loaded");
    const std::size_t n = C.n(), limbs = level + 1, cw = 2 * limbs * n;
    const std::size_t chunk = std::max<std::size_t>(1, std::min<std::size_t>(count, 512));
    Launch L = C.L();
    DevBuf dr(&C, chunk * n), de0(&C, chunk * n), de1(&C, chunk * n), rr(&C, chunk * limbs * n * 8);
    DevBuf dm(&C, with_msgs ? chunk * limbs * n * 8 : 0), dmi(&C, with_msgs ? chunk * n * 8 : 0);
    HostChunk host[2];
    auto make = [&](std::size_t c0, HostChunk& h) {
        const std::size_t m = std::min(chunk, count - c0);
        h.r.resize(m * n);
        h.e0.resize(m * n);
        h.e1.resize(m * n);
        produce(c0, m, h);
    };
    std::future<void> next = std::async(std::launch::async, make, 0, std::ref(host[0]));
    for (std::size_t c0 = 0, k = 0; c0 < count; c0 += chunk, ++k) {
        const std::size_t m = std::min(chunk, count - c0);
        next.get();  // rethrows the producer's exception (e.g. encode range checks)
        HostChunk& h = host[k & 1];
        if (c0 + chunk < count) next = std::async(std::launch::async, make, c0 + chunk, std::ref(host[(k + 1) & 1]));
        C.upload(dr.get(), h.r.data(), m * n);
        C.upload(de0.get(), h.e0.data(), m * n);
        C.upload(de1.get(), h.e1.data(), m * n);
        const u64* mres = nullptr;
        if (with_msgs) {
            if (h.small) {
                C.upload(dmi.get(), h.mi.data(), m * n * 8);
                i64_to_rns(C.dev, dmi.as<long long>(), dm.as<u64>(), static_cast<int>(level), m, L);
            } else {
                C.upload(dm.get(), h.mres.data(), m * limbs * n * 8);
            }
            mres = dm.as<u64>();
        }
        small_to_rns(C.dev, dr.as<signed char>(), rr.as<u64>(), static_cast<int>(level), m, L);
        ntt_forward(C.dev, rr.as<u64>(), static_cast<int>(level), m, L);
        u64* o = out + c0 * cw;
        mul_by_key(C.dev, rr.as<u64>(), C.pk.as<u64>(), C.top() + 1, o, static_cast<int>(level), m, L);
        ntt_inverse(C.dev, o, static_cast<int>(level), 2 * m, L);
        add_noise_msg(C.dev, o, de0.as<signed char>(), de1.as<signed char>(), mres, static_cast<int>(level), m, L);
    }
}

// make_encryption_randomness(seed) (ckks.hpp:238-244) as int8 rows
void sample_randomness(Context& C, u64 s, signed char* r, signed char* e0, signed char* e1) {
    to_int8(sample_secretish(C, 0.5, derive_seed(s, 0x0a01)), r);
    to_int8(sample_error(C, derive_seed(s, 0x0a02)), e0);
    to_int8(sample_error(C, derive_seed(s, 0x0a03)), e1);
}

// the message rows of chunk cells from encoded messages
void fill_messages(Context& C, const EncodedCoeffs* msgs, std::size_t m, std::uint32_t level, HostChunk& h) {
    const std::size_t n = C.n(), limbs = level + 1;
    h.small = true;
    for (std::size_t k = 0; k < m; ++k) h.small = h.small && msgs[k].small;
    if (h.small) {
        h.mi.resize(m * n);
        for (std::size_t k = 0; k < m; ++k) std::memcpy(&h.mi[k * n], msgs[k].coeffs.data(), n * 8);
    } else {
        h.mres.assign(m * limbs * n, 0);
        for (std::size_t k = 0; k < m; ++k) {
            const EncodedCoeffs& e = msgs[k];
            for (std::size_t i = 0; i < limbs; ++i)
                for (std::size_t j = 0; j < n; ++j)
                    h.mres[(k * limbs + i) * n + j] = e.small ? C.ring.mods[i].from_signed(e.coeffs[j]) : e.residues[i * n + j];
        }
    }
}

void encrypt_into(Context& C, std::size_t count, const u64* seeds, const std::vector<EncodedCoeffs>* msgs,
                  std::uint32_t level, u64* out) {
    const std::size_t n = C.n();
    encrypt_pipelined(C, count, level, out, msgs != nullptr, [&](std::size_t c0, std::size_t m, HostChunk& h) {
        parallel_items(m, [&](std::size_t k) { sample_randomness(C, seeds[c0 + k], &h.r[k * n], &h.e0[k * n], &h.e1[k * n]); });
        if (msgs) fill_messages(C, msgs->data() + c0, m, level, h);
    });
}

void encrypt_sampled(Context& C, std::size_t count, const signed char* r, const signed char* e0, const signed char* e1,
                     std::uint32_t level, u64* out) {
    if (!C.has_pk) throw std::invalid_argument("encrypt: no public key loaded");
    const std::size_t n = C.n(), limbs = level + 1, cw = 2 * limbs * n;
    const std::size_t chunk = std::max<std::size_t>(1, std::min<std::size_t>(count, 1024));
    Launch L = C.L();
    DevBuf dr(&C, chunk * n), de0(&C, chunk * n), de1(&C, chunk * n), rr(&C, chunk * limbs * n * 8);
    for (std::size_t c0 = 0; c0 < count; c0 += chunk) {
        const std::size_t m = std::min(chunk, count - c0);
        C.upload(dr.get(), r + c0 * n, m * n);
        C.upload(de0.get(), e0 + c0 * n, m * n);
        C.upload(de1.get(), e1 + c0 * n, m * n);
        small_to_rns(C.dev, dr.as<signed char>(), rr.as<u64>(), static_cast<int>(level), m, L);
        ntt_forward(C.dev, rr.as<u64>(), static_cast<int>(level), m, L);
        u64* o = out + c0 * cw;
        mul_by_key(C.dev, rr.as<u64>(), C.pk.as<u64>(), C.top() + 1, o, static_cast<int>(level), m, L);
        ntt_inverse(C.dev, o, static_cast<int>(level), 2 * m, L);
        add_noise_msg(C.dev, o, de0.as<signed char>(), de1.as<signed char>(), nullptr, static_cast<int>(level), m, L);
    }
}

PadNoiseMap start_pad_noise(Context& C, const Model& M, u64 seed) {
    PadNoiseMap out;
    if (!C.has_pk) return out;  // the pad layer raises the reference's error
    Shape in = M.input;
    for (std::size_t i = 0; i < M.layers.size() && i < M.shapes.size(); ++i) {
        const Layer& l = M.layers[i];
        const Shape os = M.shapes[i];
        if (l.kind == 2 && !in.flat && l.pad) {
            const u64 layer_seed = derive_seed(seed, 0x1a7e + i);
            const std::size_t pad = l.pad;
            const Shape is = in;
            out.emplace(i, std::async(std::launch::async, [&C, os, is, pad, layer_seed]() {
                                auto P = std::make_shared<PadNoise>();
                                const std::size_t cells = os.positions(), n = C.n();
                                P->border.assign(cells, -1);
                                std::vector<u64> seeds;
                                for (std::size_t p = 0; p < cells; ++p) {
                                    const std::size_t xy = p / os.c, y = xy / os.w, xx = xy % os.w;
                                    const bool inside = y >= pad && y < pad + is.h && xx >= pad && xx < pad + is.w;
                                    if (!inside) {
                                        P->border[p] = static_cast<int>(seeds.size());
                                        seeds.push_back(derive_seed(layer_seed, 0xbad0 + p));
                                    }
                                }
                                P->r.resize(seeds.size() * n);
                                P->e0.resize(seeds.size() * n);
                                P->e1.resize(seeds.size() * n);
                                parallel_items(seeds.size(), [&](std::size_t k) {
                                    const u64 s = seeds[k];
                                    to_int8(sample_secretish(C, 0.5, derive_seed(s, 0x0a01)), &P->r[k * n]);
                                    to_int8(sample_error(C, derive_seed(s, 0x0a02)), &P->e0[k * n]);
                                    to_int8(sample_error(C, derive_seed(s, 0x0a03)), &P->e1[k * n]);
                                });
                                return std::shared_ptr<const PadNoise>(P);
                            }).share());
        }
        in = os;
    }
    return out;
}

}  // namespace detail

using detail::encrypt_into;

// encrypt_tensor (tensor.hpp:77-94): the host encode (long-double FFT) and the
// randomness of cell chunk k + 1 run on host threads while chunk k encrypts
// on the device.
TensorPtr encrypt_tensor(Context& C, const double* data, std::size_t batch, std::size_t positions, u64 seed) {
    if (batch > C.n() / 2) throw std::invalid_argument("encrypt_tensor: batch exceeds slot count");
    const std::size_t top = C.top(), n = C.n();
    TensorPtr out = make_tensor(C, positions, static_cast<std::uint32_t>(top), C.scale);
    out->batch = batch;
    detail::encrypt_pipelined(C, positions, static_cast<std::uint32_t>(top), out->data(), true,
                              [&](std::size_t c0, std::size_t m, detail::HostChunk& h) {
                                  std::vector<EncodedCoeffs> part(m);
                                  std::vector<std::string> errs(m);
                                  parallel_items(m, [&](std::size_t k) {
                                      const std::size_t pos = c0 + k;
                                      try {
                                          std::vector<double> slots(batch);
                                          for (std::size_t i = 0; i < batch; ++i) slots[i] = data[i * positions + pos];
                                          C.enc->encode_real(slots.data(), batch, C.scale, top, part[k]);
                                      } catch (const std::exception& e) {
                                          errs[k] = e.what();
                                          return;
                                      }
                                      detail::sample_randomness(C, derive_seed(seed, 0xce11 + pos), &h.r[k * n],
                                                                &h.e0[k * n], &h.e1[k * n]);
                                  });
                                  for (const auto& e : errs)
                                      if (!e.empty()) throw std::invalid_argument(e);
                                  detail::fill_messages(C, part.data(), m, static_cast<std::uint32_t>(top), h);
                              });
    return out;
}

// CkksEngine::encrypt with explicit randomness (ckks.hpp:249-266)
TensorPtr encrypt_raw(Context& C, const u64* m, const long long* r, const long long* e0, const long long* e1,
                      std::size_t count, double scale) {
    if (!C.has_pk) throw std::invalid_argument("encrypt: no public key loaded");
    const std::size_t n = C.n(), top = C.top(), limbs = top + 1;
    TensorPtr out = make_tensor(C, count, static_cast<std::uint32_t>(top), scale);
    std::vector<signed char> hr(count * n), h0(count * n), h1(count * n);
    to_int8(std::vector<long long>(r, r + count * n), hr.data());
    to_int8(std::vector<long long>(e0, e0 + count * n), h0.data());
    to_int8(std::vector<long long>(e1, e1 + count * n), h1.data());
    DevBuf dr = C.upload_vec(hr), d0 = C.upload_vec(h0), d1 = C.upload_vec(h1);
    DevBuf dm(&C, count * limbs * n * 8), rr(&C, count * limbs * n * 8);
    C.upload(dm.get(), m, count * limbs * n * 8);
    Launch L = C.L();
    small_to_rns(C.dev, dr.as<signed char>(), rr.as<u64>(), static_cast<int>(top), count, L);
    ntt_forward(C.dev, rr.as<u64>(), static_cast<int>(top), count, L);
    mul_by_key(C.dev, rr.as<u64>(), C.pk.as<u64>(), limbs, out->data(), static_cast<int>(top), count, L);
    ntt_inverse(C.dev, out->data(), static_cast<int>(top), 2 * count, L);
    add_noise_msg(C.dev, out->data(), d0.as<signed char>(), d1.as<signed char>(), dm.as<u64>(), static_cast<int>(top),
                  count, L);
    return out;
}

// decrypt (ckks.hpp:273-279): c0 + c1 * s at the ciphertext level
void decrypt_raw(Context& C, const Tensor& t, u64* out_host) {
    if (!C.has_secret) throw std::invalid_argument("decrypt: no secret key loaded");
    const std::size_t n = C.n(), limbs = t.level + 1, pw = limbs * n;
    DevBuf tmp(&C, t.cells * pw * 8);
    Launch L = C.L();
    cuda_check(cudaMemcpy2DAsync(tmp.get(), pw * 8, t.data() + pw, 2 * pw * 8, pw * 8, t.cells,
                                 cudaMemcpyDeviceToDevice, C.stream),
               "copy c1");
    ntt_forward(C.dev, tmp.as<u64>(), static_cast<int>(t.level), t.cells, L);
    mul_secret(C.dev, tmp.as<u64>(), C.s_ntt.as<u64>(), static_cast<int>(t.level), t.cells, L);
    ntt_inverse(C.dev, tmp.as<u64>(), static_cast<int>(t.level), t.cells, L);
    add_c0(C.dev, t.data(), tmp.as<u64>(), static_cast<int>(t.level), t.cells, L);
    C.download(out_host, tmp.get(), t.cells * pw * 8);
}

// decrypt_tensor (tensor.hpp:96-106): out [batch][positions]
void decrypt_tensor(Context& C, const Tensor& t, std::size_t batch, double* out) {
    if (batch > C.n() / 2) throw std::invalid_argument("decrypt_tensor: batch exceeds slot count");
    const std::size_t pw = (t.level + 1) * C.n();
    std::vector<u64> plain(t.cells * pw);
    decrypt_raw(C, t, plain.data());
    parallel_items(t.cells, [&](std::size_t pos) {
        std::vector<double> v(batch);
        C.enc->decode_real(&plain[pos * pw], t.level, t.scale, v.data(), batch);
        for (std::size_t i = 0; i < batch; ++i) out[i * t.cells + pos] = v[i];
    });
}

// ---------------------------------------------------------------- network

const char* Layer::kind_name() const {
    switch (kind) {
        case 0: return "conv2d";
        case 1: return "avg_pool2d";
        case 2: return "zero_pad2d";
        case 3: return "dense";
        case 4: return "activation";
        case 5: return "sigmoid";
    }
    return "?";
}

// shape_infer / infer_layer_shape (model.hpp:116-157)
void Model::infer_shapes() {
    shapes.clear();
    Shape cur = input;
    for (std::size_t i = 0; i < layers.size(); ++i) {
        const Layer& l = layers[i];
        if (l.kind == 5 && i + 1 != layers.size())
            throw std::invalid_argument("shape_infer: sigmoid allowed only as final layer");
        if (l.kind == 3 && !cur.flat) cur = cur.as_flat();
        switch (l.kind) {
            case 0: {
                if (cur.flat) throw std::invalid_argument("shape_infer: conv2d on flattened input");
                if (l.filters == 0 || l.kh == 0 || l.kw == 0 || l.stride == 0)
                    throw std::invalid_argument("shape_infer: conv2d parameters must be positive");
                auto dim = [&](std::size_t in, std::size_t k) -> std::size_t {
                    if (!l.valid) return (in + l.stride - 1) / l.stride;
                    if (in < k) throw std::invalid_argument("shape_infer: conv kernel larger than input (valid padding)");
                    return (in - k) / l.stride + 1;
                };
                std::size_t oh = dim(cur.h, l.kh);
                std::size_t ow = dim(cur.w, l.kw);
                cur = Shape::spatial(oh, ow, l.filters);
                break;
            }
            case 1:
                if (cur.flat) throw std::invalid_argument("shape_infer: avg_pool2d on flattened input");
                if (l.pool == 0) throw std::invalid_argument("shape_infer: pool size must be positive");
                if (cur.h < l.pool || cur.w < l.pool)
                    throw std::invalid_argument("shape_infer: spatial dims smaller than pool size");
                cur = Shape::spatial(cur.h / l.pool, cur.w / l.pool, cur.c);
                break;
            case 2:
                if (cur.flat) throw std::invalid_argument("shape_infer: zero_pad2d on flattened input");
                cur = Shape::spatial(cur.h + 2 * l.pad, cur.w + 2 * l.pad, cur.c);
                break;
            case 3:
                if (l.units == 0) throw std::invalid_argument("shape_infer: dense units must be positive");
                cur = Shape::flattened(l.units);
                break;
            case 4:
                if (l.act < 0 || static_cast<std::size_t>(l.act) >= acts.size())
                    throw std::invalid_argument("model: activation layer references unregistered surrogate 'act" +
                                                std::to_string(l.act) + "'");
                break;
            case 5: break;
            default: throw std::invalid_argument("shape_infer: unknown layer kind");
        }
        shapes.push_back(cur);
    }
}

std::size_t Model::depth_cost() const {
    std::size_t cost = 0;
    for (const auto& l : layers) {
        if (l.kind == 0 || l.kind == 1 || l.kind == 3) cost += 1;
        else if (l.kind == 4) cost += acts.at(static_cast<std::size_t>(l.act)).encrypted_depth();
    }
    return cost;
}

namespace {

// Limbs whose residues fit five bytes run the linear layers on the integer
// tensor cores (conv_imma.cu); HECNN_NO_IMMA=1 keeps every limb on the
// FP64 / integer gather-MAC (linear.cu) for A/B comparisons.
bool imma_limb(const Context& C, std::size_t i) { return C.ring.primes[i] < (1ull << 40); }

bool imma_enabled(const Context& C, std::size_t K) {
    const char* e = std::getenv("HECNN_NO_IMMA");  // read per layer build (cached per model and level)
    const bool off = e && *e && *e != '0';
    return !off && imma_mac_supported(C.dev, K);
}

// Calls f(l0, l1, tc) for maximal runs of limbs [l0, l1) of equal kind.
template <class F>
void for_limb_runs(const Context& C, std::size_t limbs, F f) {
    std::size_t l0 = 0;
    while (l0 < limbs) {
        const bool tc = imma_limb(C, l0);
        std::size_t l1 = l0 + 1;
        while (l1 < limbs && imma_limb(C, l1) == tc) ++l1;
        f(l0, l1, tc);
        l0 = l1;
    }
}

// A fragments of mma.m16n8k32 (row-major 16 x 32): lane (g, t) holds
// reg0 = row g, k 4t..4t+3; reg1 = row g+8, same k; reg2/reg3 = the same rows
// at k + 16; byte u of a register is k + u. Row = output channel in the tile.
void build_imma_cache(Context& C, Model::LinearCache& lc, const std::vector<u64>& w, std::size_t rows,
                      std::size_t limbs) {
    const std::size_t K = rows, oc = static_cast<std::size_t>(lc.oc), oc_pad = static_cast<std::size_t>(lc.oc_pad);
    const std::size_t ksteps = (K + 31) / 32, kpad = ksteps * 32;
    std::size_t tiles = (oc + 15) / 16;
    if (tiles >= 2) tiles = (tiles + 1) / 2 * 2;  // the kernel pairs tiles
    std::vector<std::uint32_t> frag(limbs * tiles * ksteps * 5 * 32 * 4, 0u);
    parallel_items(limbs * tiles, [&](std::size_t it) {
        const std::size_t i = it / tiles, t = it % tiles;
        if (!imma_limb(C, i)) return;
        {
            for (std::size_t ks = 0; ks < ksteps; ++ks)
                for (std::size_t lane = 0; lane < 32; ++lane) {
                    const std::size_t g = lane >> 2, tq = lane & 3;
                    for (int r = 0; r < 4; ++r) {
                        const std::size_t o = t * 16 + g + ((r & 1) ? 8 : 0);
                        const std::size_t k0 = ks * 32 + 4 * tq + ((r & 2) ? 16 : 0);
                        std::uint64_t wv[4] = {0, 0, 0, 0};
                        for (int u = 0; u < 4; ++u)
                            if (o < oc && k0 + u < K) wv[u] = w[(i * rows + k0 + u) * oc_pad + o];
                        for (int b = 0; b < 5; ++b) {
                            std::uint32_t reg = 0;
                            for (int u = 0; u < 4; ++u) reg |= static_cast<std::uint32_t>((wv[u] >> (8 * b)) & 0xFF) << (8 * u);
                            frag[((((i * tiles + t) * ksteps + ks) * 5 + b) * 32 + lane) * 4 + r] = reg;
                        }
                    }
                }
        }
    });
    // signed weight integers W (|W| < 2^47) recovered from the widest limb and
    // checked against every limb's residue; their balanced base-256 digits
    // feed the wide-limb kernel
    std::size_t wl = 0;
    for (std::size_t i = 1; i < limbs; ++i)
        if (C.ring.primes[i] > C.ring.primes[wl]) wl = i;
    const std::int64_t wmax = 127LL * ((1LL << 48) - 1) / 255;  // 6 balanced digits
    std::vector<std::int64_t> W(K * oc, 0);
    std::vector<char> row_ok(K, 1);
    parallel_items(K, [&](std::size_t k) {
        for (std::size_t o = 0; o < oc && row_ok[k]; ++o) {
            const u64 qw = C.ring.primes[wl], r = w[(wl * rows + k) * oc_pad + o];
            const std::int64_t v = r > qw / 2 ? -static_cast<std::int64_t>(qw - r) : static_cast<std::int64_t>(r);
            if (v > wmax || v < -wmax) row_ok[k] = 0;
            for (std::size_t i = 0; i < limbs && row_ok[k]; ++i) {
                const u64 qi = C.ring.primes[i];
                const u64 ri = v >= 0 ? static_cast<u64>(v) % qi : (qi - static_cast<u64>(-v) % qi) % qi;
                if (ri != w[(i * rows + k) * oc_pad + o]) row_ok[k] = 0;
            }
            W[k * oc + o] = v;
        }
    });
    const bool wide_ok = std::all_of(row_ok.begin(), row_ok.end(), [](char c) { return c != 0; });
    if (wide_ok) {
        std::vector<std::uint32_t> fw(tiles * ksteps * 6 * 32 * 4, 0u);
        parallel_items(tiles, [&](std::size_t t) {
            for (std::size_t ks = 0; ks < ksteps; ++ks)
                for (std::size_t lane = 0; lane < 32; ++lane) {
                    const std::size_t g = lane >> 2, tq = lane & 3;
                    for (int r = 0; r < 4; ++r) {
                        const std::size_t o = t * 16 + g + ((r & 1) ? 8 : 0);
                        const std::size_t k0 = ks * 32 + 4 * tq + ((r & 2) ? 16 : 0);
                        std::int8_t dig[4][6] = {};
                        for (int u = 0; u < 4; ++u) {
                            if (o >= oc || k0 + u >= K) continue;
                            std::int64_t v = W[(k0 + u) * oc + o];
                            for (int b = 0; b < 6; ++b) {
                                const std::int8_t d = static_cast<std::int8_t>(v & 0xFF);  // balanced digit
                                dig[u][b] = d;
                                v = (v - d) / 256;
                            }
                        }
                        for (int b = 0; b < 6; ++b) {
                            std::uint32_t reg = 0;
                            for (int u = 0; u < 4; ++u) reg |= static_cast<std::uint32_t>(static_cast<std::uint8_t>(dig[u][b])) << (8 * u);
                            fw[(((t * ksteps + ks) * 6 + b) * 32 + lane) * 4 + r] = reg;
                        }
                    }
                }
        });
        std::vector<ulonglong2> shw(limbs * 16, make_ulonglong2(0, 0));
        for (std::size_t i = 0; i < limbs; ++i)
            for (int s = 0; s < 13; ++s) {
                const u64 c = C.ring.mods[i].pow(2, 8 * s);
                shw[i * 16 + s] = make_ulonglong2(c, shoup_of(c, C.ring.primes[i]));
            }
        lc.wfrag_wide = C.upload_vec(fw);
        lc.shift_wide = C.upload_vec(shw);
    }
    lc.wide_ok = wide_ok;
    std::vector<double> sh(limbs * 9);
    for (std::size_t i = 0; i < limbs; ++i)
        for (int s = 0; s < 9; ++s) sh[i * 9 + s] = static_cast<double>(C.ring.mods[i].pow(2, 8 * s));
    // tcgen05 weight tiles: per (limb, 48-channel tile, 32-tap step) the B
    // operand of conv_tc.cu, rows n = b * 48 + o (weight byte b of channel o),
    // in the UMMA K-major core-matrix layout (8 rows x 16 taps per 128 B)
    const std::size_t TOC = static_cast<std::size_t>(tc_oc_tile(false)), ttiles = (oc + TOC - 1) / TOC;
    const std::size_t tile_bytes = 5 * TOC * 32, wtc_bytes = limbs * ttiles * ksteps * tile_bytes;
    const char* no_tc = std::getenv("HECNN_NO_TCGEN05");
    if (!(no_tc && *no_tc == '1') && lc.conv && ksteps <= 192 && C.n() % 128 == 0 && wtc_bytes <= (std::size_t(1) << 30)) {
        std::vector<std::uint8_t> t(wtc_bytes, 0);
        parallel_items(limbs * ttiles, [&](std::size_t it) {
            const std::size_t i = it / ttiles, ot = it % ttiles;
            if (!imma_limb(C, i)) return;
            {
                for (std::size_t ks = 0; ks < ksteps; ++ks) {
                    std::uint8_t* tile = t.data() + ((i * ttiles + ot) * ksteps + ks) * tile_bytes;
                    for (std::size_t o = 0; o < TOC; ++o) {
                        const std::size_t oo = ot * TOC + o;
                        if (oo >= oc) continue;
                        for (std::size_t k = 0; k < 32; ++k) {
                            const std::size_t kk = ks * 32 + k;
                            if (kk >= K) continue;
                            const u64 v = w[(i * rows + kk) * oc_pad + oo];
                            for (std::size_t b = 0; b < 5; ++b) {
                                const std::size_t n = b * TOC + o;
                                tile[(n >> 3) * 256 + (k >> 4) * 128 + (n & 7) * 16 + (k & 15)] =
                                    static_cast<std::uint8_t>(v >> (8 * b));
                            }
                        }
                    }
                }
            }
        });
        lc.wtc = C.upload_vec(t);
        if (wide_ok) {
            // the 60-bit limb: the balanced signed base-256 digits of W (one copy for all
            // limbs), rows n = b * 32 + o of 192 per 32-tap step
            const std::size_t WOC = static_cast<std::size_t>(tc_oc_tile(true)), wtiles = (oc + WOC - 1) / WOC;
            const std::size_t wtile_bytes = 6 * WOC * 32;
            std::vector<std::uint8_t> tw(wtiles * ksteps * wtile_bytes, 0);
            for (std::size_t ot = 0; ot < wtiles; ++ot)
                for (std::size_t ks = 0; ks < ksteps; ++ks) {
                    std::uint8_t* tile = tw.data() + (ot * ksteps + ks) * wtile_bytes;
                    for (std::size_t o = 0; o < WOC; ++o) {
                        const std::size_t oo = ot * WOC + o;
                        if (oo >= oc) continue;
                        for (std::size_t k = 0; k < 32; ++k) {
                            const std::size_t kk = ks * 32 + k;
                            if (kk >= K) continue;
                            std::int64_t v = W[kk * oc + oo];
                            for (std::size_t b = 0; b < 6; ++b) {
                                const std::int8_t dgt = static_cast<std::int8_t>(v & 0xFF);  // balanced digit
                                v = (v - dgt) / 256;
                                const std::size_t n = b * WOC + o;
                                tile[(n >> 3) * 256 + (k >> 4) * 128 + (n & 7) * 16 + (k & 15)] = static_cast<std::uint8_t>(dgt);
                            }
                        }
                    }
                }
            lc.wtc_wide = C.upload_vec(tw);
        }
    }
    lc.wfrag = C.upload_vec(frag);
    lc.shift = C.upload_vec(sh);
    lc.kpad = static_cast<int>(kpad);
    lc.ksteps = static_cast<int>(ksteps);
    lc.oc_tiles = static_cast<int>(tiles);
}

}  // namespace

namespace detail {

// Integer weight residues of a conv / dense layer at `level`, with the
// tensor-core layouts (layers.hpp:185-188 encodes each weight once per layer
// call; here once per model and level).
Model::LinearCache& linear_weights(Context& C, Model& M, std::size_t li, std::uint32_t level, std::size_t rows) {
    const Layer& l = M.layers[li];
    const bool conv = l.kind == 0;
    const std::size_t oc = conv ? l.filters : l.units;
    if (l.w.size() != rows * oc || l.b.size() != oc)
        throw std::invalid_argument(conv ? "conv2d: weight/bias shape mismatch" : "dense: weight/bias shape mismatch");
    if (level == 0) throw std::invalid_argument(conv ? "conv2d: no level headroom" : "dense: no level headroom");
    auto key = std::make_pair(li, level);
    auto it = M.linear.find(key);
    if (it != M.linear.end()) return it->second;
    const std::size_t limbs = level + 1;
    Model::LinearCache lc;
    lc.conv = conv;
    lc.K = static_cast<int>(rows);
    lc.oc = static_cast<int>(oc);
    lc.oc_pad = static_cast<int>((oc + 15) / 16 * 16);
    // make_scalar_plain per weight (host roundl / fmod), rows in parallel; the
    // first failing range check is rethrown in row order
    std::vector<u64> w(rows * lc.oc_pad * limbs, 0);  // [limbs][rows][oc_pad]: OCT channels contiguous
    std::vector<std::string> errs(rows);
    parallel_items(rows, [&](std::size_t r) {
        try {
            for (std::size_t o = 0; o < oc; ++o) {
                std::vector<u64> res = C.enc->scalar_residues(l.w[r * oc + o], C.scale, level);
                for (std::size_t i = 0; i < limbs; ++i) w[(i * rows + r) * lc.oc_pad + o] = res[i];
            }
        } catch (const std::exception& e) {
            errs[r] = e.what();
        }
    });
    for (const auto& e : errs)
        if (!e.empty()) throw std::invalid_argument(e);
    std::vector<ulonglong2> rc(2 * limbs);
    for (std::size_t i = 0; i < limbs; ++i) {
        const HostMod& m = C.ring.mods[i];
        const u64 a = m.pow(2, 21), b = m.pow(2, 42);
        rc[2 * i] = make_ulonglong2(a, shoup_of(a, m.q));
        rc[2 * i + 1] = make_ulonglong2(b, shoup_of(b, m.q));
    }
    lc.recomb = C.upload_vec(rc);
    if (imma_enabled(C, rows)) build_imma_cache(C, lc, w, rows, limbs);
    if (!lc.ksteps || !lc.wide_ok) {
        // gather-MAC operands (some limb is not on the tensor cores): Shoup pairs
        // and the 21-bit split of each residue
        std::vector<ulonglong2> wp(w.size());
        std::vector<uint2> ws(w.size());
        parallel_items(limbs, [&](std::size_t i) {
            for (std::size_t at = i * rows * lc.oc_pad; at < (i + 1) * rows * lc.oc_pad; ++at) {
                wp[at] = make_ulonglong2(w[at], shoup_of(w[at], C.ring.primes[i]));
                ws[at] = make_uint2(static_cast<unsigned>(w[at] & 0x1FFFFFu), static_cast<unsigned>(w[at] >> 21));
            }
        });
        lc.weights = C.upload_vec(wp);
        lc.wsplit = C.upload_vec(ws);
    }
    return M.linear.emplace(key, std::move(lc)).first->second;
}

Model::Taps make_taps(Context& C, const Model::LinearCache& lc, const std::vector<int>& src) {
    Model::Taps t;
    const std::size_t K = static_cast<std::size_t>(lc.K);
    t.pixels = src.size() / K;
    t.src = C.upload_vec(src);
    if (lc.ksteps) {
        const std::size_t kpad = static_cast<std::size_t>(lc.kpad);
        std::vector<int> sp(t.pixels * kpad, -1);
        for (std::size_t p = 0; p < t.pixels; ++p)
            for (std::size_t k = 0; k < K; ++k) sp[p * kpad + k] = src[p * K + k];
        t.src_pad = C.upload_vec(sp);
    }
    return t;
}

// ConvGeom (layers.hpp:24-50): same padding offsets of a conv from its input dims
void conv_offsets(const Layer& l, std::size_t in_h, std::size_t in_w, std::size_t out_h, std::size_t out_w,
                  long long& pad_top, long long& pad_left) {
    pad_top = pad_left = 0;
    if (l.valid) return;
    const std::size_t need_h = (out_h - 1) * l.stride + l.kh, need_w = (out_w - 1) * l.stride + l.kw;
    pad_top = need_h > in_h ? static_cast<long long>((need_h - in_h) / 2) : 0;
    pad_left = need_w > in_w ? static_cast<long long>((need_w - in_w) / 2) : 0;
}

// bias residues at the accumulator scale (add_scalar_inplace, ckks.hpp:468-472)
const u64* linear_bias(Context& C, Model& M, std::size_t li, std::uint32_t level, double acc_scale) {
    const Layer& l = M.layers[li];
    const std::size_t oc = l.kind == 0 ? l.filters : l.units, limbs = level + 1;
    auto bkey = std::make_tuple(li, level, acc_scale);
    auto bit = M.bias.find(bkey);
    if (bit == M.bias.end()) {
        std::vector<u64> b(oc * limbs);
        for (std::size_t o = 0; o < oc; ++o) {
            std::vector<u64> res = C.enc->scalar_residues(l.b[o], acc_scale, level);
            std::copy(res.begin(), res.end(), b.begin() + o * limbs);
        }
        bit = M.bias.emplace(bkey, C.upload_vec(b)).first;
    }
    return bit->second.as<u64>();
}

// Output cells [m][oc] at `out` (level - 1) for pixels [p0, p0 + m) of a tap
// table over the input cells at `x`: MAC over the taps (mul_scalar_mac,
// ckks.hpp:448-465), bias, rescale (ckks.hpp:474-482). Chunked so the
// pre-rescale scratch stays within kScratchBytes.
void linear_apply(Context& C, Model::LinearCache& lc, const Model::Taps& taps, const u64* bias, const u64* x,
                  std::uint32_t level, std::size_t p0, std::size_t m, u64* out) {
    const std::size_t limbs = level + 1, oc = static_cast<std::size_t>(lc.oc);
    const std::size_t cw = 2 * limbs * C.n();
    const std::size_t per_pixel = oc * cw * 8;
    const std::size_t pix_chunk = std::max<std::size_t>(1, std::min<std::size_t>(m, kScratchBytes / per_pixel));
    DevBuf pre(&C, pix_chunk * per_pixel);
    Launch L = C.L();
    for (std::size_t q0 = 0; q0 < m; q0 += pix_chunk) {
        const std::size_t mm = std::min(pix_chunk, m - q0), pp = p0 + q0;
        GatherMac g{taps.src.as<int>() + pp * lc.K, lc.weights.as<ulonglong2>(), bias, lc.wsplit.as<uint2>(),
                    lc.recomb.as<ulonglong2>(), static_cast<int>(mm), lc.K, lc.oc, lc.oc_pad, lc.oc};
        if (lc.ksteps) {
            ImmaMac im{taps.src_pad.as<int>() + pp * lc.kpad, lc.wfrag.as<uint4>(), bias, lc.shift.as<double>(),
                       static_cast<int>(mm), lc.K, lc.kpad, lc.ksteps, lc.oc, lc.oc_tiles, lc.oc,
                       lc.wfrag_wide.as<uint4>(), lc.shift_wide.as<ulonglong2>(), lc.wtc.as<uint4>(),
                       lc.wtc_wide.as<uint4>()};
            for_limb_runs(C, limbs, [&](std::size_t l0, std::size_t l1, bool tc) {
                if ((tc || lc.wide_ok) && tc_mac_supported(C.dev, im, !tc))
                    tc_mac(C.dev, im, x, pre.as<u64>(), static_cast<int>(level), static_cast<int>(l0),
                           static_cast<int>(l1), !tc, L);
                else if (tc || lc.wide_ok)
                    imma_mac(C.dev, im, x, pre.as<u64>(), static_cast<int>(level), static_cast<int>(l0),
                             static_cast<int>(l1), !tc, L);
                else gather_mac(C.dev, g, x, pre.as<u64>(), static_cast<int>(level), static_cast<int>(l0),
                                static_cast<int>(l1), L);
            });
        } else {
            gather_mac(C.dev, g, x, pre.as<u64>(), static_cast<int>(level), 0, static_cast<int>(limbs), L);
        }
        rescale(C.dev, pre.as<u64>(), out + q0 * oc * 2 * level * C.n(), static_cast<int>(level), 2 * mm * oc, L);
    }
}

}  // namespace detail

namespace {

using detail::linear_weights;

// conv2d / dense as a gather-MAC (layers.hpp:174-211, 269-293)
TensorPtr linear_layer(Context& C, Model& M, std::size_t li, const Tensor& x, const Shape& out_shape) {
    Trace tr("linear_layer");
    const Layer& l = M.layers[li];
    const bool conv = l.kind == 0;
    const Shape& in = x.shape;
    const std::size_t rows = conv ? l.kh * l.kw * in.c : in.positions();
    const std::uint32_t level = x.level;
    Model::LinearCache& lc = linear_weights(C, M, li, level, rows);
    if (!lc.taps.pixels) {
        std::vector<int> src;  // tap k of every pixel uses weight row k (ky, kx, ic order)
        if (conv) {
            long long pad_top = 0, pad_left = 0;
            detail::conv_offsets(l, in.h, in.w, out_shape.h, out_shape.w, pad_top, pad_left);
            for (std::size_t oy = 0; oy < out_shape.h; ++oy)
                for (std::size_t ox = 0; ox < out_shape.w; ++ox)
                    for (std::size_t ky = 0; ky < l.kh; ++ky)
                        for (std::size_t kx = 0; kx < l.kw; ++kx)
                            for (std::size_t ic = 0; ic < in.c; ++ic) {
                                long long y = static_cast<long long>(oy * l.stride + ky) - pad_top;
                                long long xx = static_cast<long long>(ox * l.stride + kx) - pad_left;
                                bool ok = y >= 0 && xx >= 0 && y < static_cast<long long>(in.h) &&
                                          xx < static_cast<long long>(in.w);
                                src.push_back(ok ? static_cast<int>((y * in.w + xx) * in.c + ic) : -1);
                            }
        } else {
            for (std::size_t k = 0; k < rows; ++k) src.push_back(static_cast<int>(k));
        }
        lc.taps = detail::make_taps(C, lc, src);
    }
    const double acc_scale = x.scale * C.scale;
    const u64* bias = detail::linear_bias(C, M, li, level, acc_scale);
    TensorPtr out = make_tensor(C, out_shape.positions(), level - 1, acc_scale / static_cast<double>(C.ring.primes[level]));
    out->shape = out_shape;
    out->batch = x.batch;
    detail::linear_apply(C, lc, lc.taps, bias, x.data(), level, 0, lc.taps.pixels, out->data());
    return out;
}

// avg_pool2d_encrypted (layers.hpp:213-239)
TensorPtr pool_layer(Context& C, Model& M, std::size_t li, const Tensor& x, const Shape& out_shape) {
    const Layer& l = M.layers[li];
    if (x.level == 0) throw std::invalid_argument("avg_pool2d: no level headroom");
    const std::uint32_t level = x.level;
    const double inv_area = 1.0 / static_cast<double>(l.pool * l.pool);
    std::vector<u64> res = C.enc->scalar_residues(inv_area, C.scale, level);
    DevBuf wres = C.upload_vec(with_shoup(C.ring, res));
    auto key = std::make_pair(li, level);
    auto it = M.pool_srcs.find(key);
    const std::size_t taps = l.pool * l.pool;
    if (it == M.pool_srcs.end()) {
        std::vector<int> srcs;
        const Shape& in = x.shape;
        for (std::size_t p = 0; p < out_shape.positions(); ++p) {
            std::size_t ch = p % out_shape.c, oxy = p / out_shape.c;
            std::size_t oy = oxy / out_shape.w, ox = oxy % out_shape.w;
            for (std::size_t dy = 0; dy < l.pool; ++dy)
                for (std::size_t dx = 0; dx < l.pool; ++dx)
                    srcs.push_back(static_cast<int>(((oy * l.pool + dy) * in.w + (ox * l.pool + dx)) * in.c + ch));
        }
        it = M.pool_srcs.emplace(key, C.upload_vec(srcs)).first;
    }
    const std::size_t cells = out_shape.positions();
    DevBuf pre(&C, cells * x.cell_words() * 8);
    Launch L = C.L();
    pool_sum_scale(C.dev, x.data(), it->second.as<int>(), static_cast<int>(taps), wres.as<ulonglong2>(), pre.as<u64>(),
                   static_cast<int>(level), cells, L);
    TensorPtr out = make_tensor(C, cells, level - 1, x.scale * C.scale / static_cast<double>(C.ring.primes[level]));
    out->shape = out_shape;
    out->batch = x.batch;
    rescale(C.dev, pre.as<u64>(), out->data(), static_cast<int>(level), 2 * cells, L);
    return out;
}

// zero_pad2d_encrypted (layers.hpp:241-267): inner cells copied, border cells
// are fresh encryptions of zero (host randomness, device arithmetic).
TensorPtr pad_layer(Context& C, Model& M, std::size_t li, const Tensor& x, const Shape& out_shape, u64 layer_seed,
                    const detail::PadNoiseMap& pads) {
    const Layer& l = M.layers[li];
    const std::size_t cells = out_shape.positions();
    std::vector<int> idx_in(cells, -1), idx_border(cells, -1);
    std::vector<u64> seeds;
    for (std::size_t p = 0; p < cells; ++p) {
        std::size_t ch = p % out_shape.c, xy = p / out_shape.c;
        std::size_t y = xy / out_shape.w, xx = xy % out_shape.w;
        bool inside = y >= l.pad && y < l.pad + x.shape.h && xx >= l.pad && xx < l.pad + x.shape.w;
        if (inside) {
            idx_in[p] = static_cast<int>(((y - l.pad) * x.shape.w + (xx - l.pad)) * x.shape.c + ch);
        } else {
            idx_border[p] = static_cast<int>(seeds.size());
            seeds.push_back(derive_seed(layer_seed, 0xbad0 + p));
        }
    }
    if (!seeds.empty()) C.enc->check_encode(1, 0.0, x.scale, C.top());  // encode_const(0, scale, top)
    TensorPtr out = make_tensor(C, cells, x.level, x.scale);
    out->shape = out_shape;
    out->batch = x.batch;
    Launch L = C.L();
    DevBuf din = C.upload_vec(idx_in);
    gather_cells(x.data(), din.as<int>(), out->data(), x.cell_words(), cells, L);
    if (!seeds.empty()) {
        DevBuf fresh(&C, seeds.size() * x.cell_words() * 8);
        auto it = pads.find(li);
        if (it != pads.end()) {  // sampled on host threads while earlier layers ran
            const detail::PadNoise& P = *it->second.get();
            detail::encrypt_sampled(C, seeds.size(), P.r.data(), P.e0.data(), P.e1.data(), x.level, fresh.as<u64>());
        } else {
            encrypt_into(C, seeds.size(), seeds.data(), nullptr, x.level, fresh.as<u64>());
        }
        DevBuf db = C.upload_vec(idx_border);
        gather_cells(fresh.as<u64>(), db.as<int>(), out->data(), x.cell_words(), cells, L);
    }
    return out;
}

}  // namespace

// forward_encrypted (layers.hpp:299-368)
TensorPtr forward_encrypted(Context& C, Model& M, const Tensor& x, u64 seed, double* layer_seconds) {
    if (!(x.shape == M.input))
        throw std::invalid_argument("forward_encrypted: input shape " + x.shape.str() + " != model input " +
                                    M.input.str());
    M.infer_shapes();
    long long level = static_cast<long long>(x.level);
    for (std::size_t i = 0; i < M.layers.size(); ++i) {
        const Layer& l = M.layers[i];
        std::size_t cost = 0;
        if (l.kind == 0 || l.kind == 1 || l.kind == 3) cost = 1;
        else if (l.kind == 4) cost = M.acts[static_cast<std::size_t>(l.act)].encrypted_depth();
        level -= static_cast<long long>(cost);
        if (level < 0)
            throw std::invalid_argument("forward_encrypted: depth budget exhausted at layer " + std::to_string(i) + " (" +
                                        l.kind_name() + ")");
    }
    std::vector<cudaEvent_t> ev(M.layers.size() + 1);
    if (layer_seconds)
        for (auto& e : ev) cudaEventCreate(&e);
    if (layer_seconds) cudaEventRecord(ev[0], C.stream);

    TensorPtr cur;
    auto current = [&]() -> const Tensor& { return cur ? *cur : x; };
    std::vector<double> stream_ms(M.layers.size(), 0.0);
    const detail::PadNoiseMap pads = detail::start_pad_noise(C, M, seed);
    std::vector<bool> streamed(M.layers.size(), false);
    for (std::size_t i = 0; i < M.layers.size(); ++i) {
        // layers whose tensors do not fit in device memory run row-streamed (stream.cpp)
        std::size_t end = i;
        TensorPtr seg =
            detail::forward_streamed(C, M, current(), i, end, seed, layer_seconds ? &stream_ms : nullptr, pads);
        if (seg) {
            cur = std::move(seg);
            for (std::size_t j = i; j < end; ++j) {
                streamed[j] = true;
                if (layer_seconds) cudaEventRecord(ev[j + 1], C.stream);
            }
            i = end - 1;
            continue;
        }
        const Layer& l = M.layers[i];
        const u64 layer_seed = derive_seed(seed, 0x1a7e + i);
        Shape in_shape = current().shape;
        if (l.kind == 3 && !in_shape.flat) {
            if (!cur) {  // flatten the caller's tensor: metadata only, take a view-copy
                cur = make_tensor(C, x.cells, x.level, x.scale);
                cuda_check(cudaMemcpyAsync(cur->data(), x.data(), x.cells * x.cell_words() * 8,
                                           cudaMemcpyDeviceToDevice, C.stream), "copy");
                cur->batch = x.batch;
            }
            cur->shape = in_shape.as_flat();
        }
        TensorPtr next;
        switch (l.kind) {
            case 0:
            case 3: next = linear_layer(C, M, i, current(), M.shapes[i]); break;
            case 1: next = pool_layer(C, M, i, current(), M.shapes[i]); break;
            case 2: next = pad_layer(C, M, i, current(), M.shapes[i], layer_seed, pads); break;
            case 4:
                next = eval_activation(C, M.acts[static_cast<std::size_t>(l.act)], current());
                break;
            case 5: break;  // the client thresholds the decrypted logit (layers.hpp:360-362)
        }
        if (next) cur = std::move(next);
        if (layer_seconds) cudaEventRecord(ev[i + 1], C.stream);
    }
    if (!cur) {
        cur = make_tensor(C, x.cells, x.level, x.scale);
        cuda_check(cudaMemcpyAsync(cur->data(), x.data(), x.cells * x.cell_words() * 8, cudaMemcpyDeviceToDevice,
                                   C.stream), "copy");
        cur->shape = x.shape;
        cur->batch = x.batch;
    }
    if (layer_seconds) {
        C.sync();
        for (std::size_t i = 0; i < M.layers.size(); ++i) {
            float ms = 0;
            if (!streamed[i]) cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
            layer_seconds[i] = (streamed[i] ? stream_ms[i] : ms) / 1000.0;
        }
        for (auto& e : ev) cudaEventDestroy(e);
    }
    return cur;
}

}  // namespace hecnn_b200
