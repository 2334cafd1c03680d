// extern "C" boundary (include/hecnn_b200.h). Each entry converts C++
// exceptions into status codes + a thread-local message, mirroring the
// reference's exception types: std::invalid_argument -> HECNN_EINVAL,
// std::runtime_error (and anything else) -> HECNN_ERUNTIME.
#include <cstdio>
#include <cstring>
#include <string>

#include "blob.hpp"
#include "engine.hpp"
#include "hecnn_b200.h"

using namespace hecnn_b200;

// Tensors and models share ownership of their context: destroying the
// context handle only drops one reference, so handles released in any order
// (e.g. by a garbage collector) never touch a dead context.
struct hecnn_context {
    std::shared_ptr<Context> ctx;
};
struct hecnn_tensor {
    std::shared_ptr<Context> keep;  // destroyed after t (reverse member order)
    TensorPtr t;
};
struct hecnn_model {
    std::shared_ptr<Context> keep;
    Model m;
};

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return HECNN_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return HECNN_EINVAL;
    } catch (const std::exception& e) {
        g_err = e.what();
        return HECNN_ERUNTIME;
    } catch (...) {
        g_err = "unknown error";
        return HECNN_ERUNTIME;
    }
}

Context& C(hecnn_context* c) {
    if (!c || !c->ctx) throw std::invalid_argument("null context");
    cudaSetDevice(c->ctx->device);
    return *c->ctx;
}
const Context& C(const hecnn_context* c) {
    if (!c || !c->ctx) throw std::invalid_argument("null context");
    return *c->ctx;
}
const Tensor& T(const hecnn_tensor* t) {
    if (!t || !t->t) throw std::invalid_argument("null tensor");
    return *t->t;
}
// a tensor modified in place must live in the context the call names
Tensor& TM(hecnn_context* c, hecnn_tensor* t) {
    if (!t || !t->t) throw std::invalid_argument("null tensor");
    if (!c || t->t->ctx != c->ctx.get()) throw std::invalid_argument("tensor belongs to another context");
    return *t->t;
}
std::shared_ptr<Context> owner(hecnn_context* c) { return c->ctx; }

hecnn_tensor* wrap(hecnn_context* c, TensorPtr t) {
    auto* h = new hecnn_tensor;
    h->keep = owner(c);
    h->t = std::move(t);
    return h;
}

}  // namespace

extern "C" {

const char* hecnn_last_error(void) { return g_err.c_str(); }
int hecnn_abi_version(void) { return 1; }

int hecnn_find_chain(size_t n, const int* prime_bits, size_t count, uint64_t* primes_out) {
    return guard([&] {
        std::vector<u64> c = make_chain(n, std::vector<int>(prime_bits, prime_bits + count));
        std::memcpy(primes_out, c.data(), c.size() * 8);
    });
}

int hecnn_host_encode_real(size_t n, const uint64_t* primes, size_t nprimes, const double* values, size_t len,
                           double scale, size_t level, uint64_t* out) {
    return guard([&] {
        RingTables R;
        R.build(n, std::vector<u64>(primes, primes + nprimes));
        Encoder enc(R, scale);
        EncodedCoeffs e;
        enc.encode_real(values, len, scale, level, e);
        for (size_t i = 0; i <= level; ++i)
            for (size_t j = 0; j < n; ++j)
                out[i * n + j] = e.small ? R.mods[i].from_signed(e.coeffs[j]) : e.residues[i * n + j];
    });
}

int hecnn_host_decode_real(size_t n, const uint64_t* primes, size_t nprimes, const uint64_t* poly, size_t level,
                           double scale, double* out, size_t count) {
    return guard([&] {
        RingTables R;
        R.build(n, std::vector<u64>(primes, primes + nprimes));
        Encoder enc(R, scale);
        enc.decode_real(poly, level, scale, out, count);
    });
}

int hecnn_host_encryption_randomness(size_t n, double sigma, int degenerate, uint64_t seed, int64_t* r, int64_t* e0,
                                     int64_t* e1) {
    return guard([&] {
        auto put = [&](const std::vector<long long>& v, int64_t* dst) {
            for (size_t j = 0; j < n; ++j) dst[j] = v[j];
        };
        std::vector<long long> zero(n, 0);
        put(degenerate ? zero : sample_ternary(n, 0.5, derive_seed(seed, 0x0a01)), r);
        const bool no_err = degenerate || sigma == 0.0;
        put(no_err ? zero : sample_gaussian(n, sigma, derive_seed(seed, 0x0a02)), e0);
        put(no_err ? zero : sample_gaussian(n, sigma, derive_seed(seed, 0x0a03)), e1);
    });
}

int hecnn_context_create(size_t n, const uint64_t* primes, size_t nprimes, double scale, double sigma,
                         int degenerate_noise, int device, hecnn_context** out) {
    return guard([&] {
        auto h = std::make_unique<hecnn_context>();
        h->ctx = std::make_shared<Context>(n, std::vector<u64>(primes, primes + nprimes), scale, sigma,
                                           degenerate_noise != 0, device);
        *out = h.release();
    });
}

int hecnn_context_destroy(hecnn_context* ctx) {
    return guard([&] { delete ctx; });
}

int hecnn_context_set_stream(hecnn_context* ctx, void* stream) {
    return guard([&] {
        Context& c = C(ctx);
        c.sync();
        if (c.own_stream) cudaStreamDestroy(c.stream);
        c.own_stream = false;
        c.stream = static_cast<cudaStream_t>(stream);
    });
}

int hecnn_context_trim(hecnn_context* ctx, size_t* freed) {
    return guard([&] {
        Context& c = C(ctx);
        c.sync();
        const std::size_t f = c.arena.trim();
        if (freed) *freed = f;
    });
}

int hecnn_context_synchronize(hecnn_context* ctx) {
    return guard([&] { C(ctx).sync(); });
}

int hecnn_context_info(const hecnn_context* ctx, size_t* n, size_t* top_level, double* scale) {
    return guard([&] {
        const Context& c = C(ctx);
        if (n) *n = c.n();
        if (top_level) *top_level = c.top();
        if (scale) *scale = c.scale;
    });
}

int hecnn_relin_digits(const hecnn_context* ctx, size_t level, size_t* digits) {
    return guard([&] {
        const Context& c = C(ctx);
        if (level > c.top()) throw std::invalid_argument("relin_digits: level out of range");
        *digits = c.ring.relin_digits(level);
    });
}

int hecnn_launch_count(const hecnn_context* ctx, uint64_t* launches) {
    return guard([&] { *launches = C(ctx).launches; });
}

int hecnn_profile_enable(hecnn_context* ctx, int on) {
    return guard([&] {
        Context& c = C(ctx);
        c.sync();
        c.prof.collect();
        c.prof.enabled = on != 0;
    });
}

int hecnn_profile_reset(hecnn_context* ctx) {
    return guard([&] {
        Context& c = C(ctx);
        c.sync();
        c.prof.reset();
    });
}

int hecnn_profile_read(hecnn_context* ctx, char* buf, size_t len) {
    return guard([&] {
        Context& c = C(ctx);
        c.sync();
        c.prof.collect();
        std::string js = "{";
        bool first = true;
        for (const auto& kv : c.prof.stats) {
            if (!first) js += ",";
            first = false;
            char num[160];
            std::snprintf(num, sizeof num, "{\"ms\":%.6f,\"launches\":%llu,\"ops\":%.6e,\"bytes\":%.6e}",
                          kv.second.ms, kv.second.launches, kv.second.ops, kv.second.bytes);
            js += "\"" + kv.first + "\":" + num;
        }
        js += "}";
        if (js.size() + 1 > len) throw std::invalid_argument("profile_read: buffer too small");
        std::memcpy(buf, js.c_str(), js.size() + 1);
    });
}

int hecnn_modmul_peak(hecnn_context* ctx, double* modmul_per_s) {
    return guard([&] { *modmul_per_s = measure_modmul_peak(C(ctx)); });
}

int hecnn_fp64_modmul_peak(hecnn_context* ctx, double* modmul_per_s) {
    return guard([&] { *modmul_per_s = measure_modmul_peak(C(ctx), true); });
}

int hecnn_tensor_copy_to_device(hecnn_context* ctx, const hecnn_tensor* t, void* dst) {
    return guard([&] {
        Context& c = C(ctx);
        const Tensor& x = T(t);
        if (cudaMemcpyAsync(dst, x.data(), x.cells * x.cell_words() * 8, cudaMemcpyDeviceToDevice, c.stream) !=
            cudaSuccess)
            throw std::runtime_error("tensor_copy_to_device failed");
        c.sync();
    });
}

int hecnn_keygen(hecnn_context* ctx, uint64_t seed) {
    return guard([&] { keygen(C(ctx), seed); });
}

int hecnn_import_keys(hecnn_context* ctx, const uint64_t* secret, const uint64_t* pk_b, const uint64_t* pk_a,
                      const uint64_t* evk, size_t evk_digits) {
    return guard([&] { import_keys(C(ctx), secret, pk_b, pk_a, evk, evk_digits); });
}

int hecnn_export_secret_key(const hecnn_context* ctx, uint64_t* secret) {
    return guard([&] {
        const Context& c = C(ctx);
        if (!c.has_secret) throw std::invalid_argument("no secret key");
        std::memcpy(secret, c.secret_host.data(), c.secret_host.size() * 8);
    });
}

int hecnn_export_public_key(const hecnn_context* ctx, uint64_t* pk_b, uint64_t* pk_a) {
    return guard([&] {
        Context& c = *const_cast<hecnn_context*>(ctx)->ctx;
        if (!c.has_pk) throw std::invalid_argument("no public key");
        const std::size_t poly = (c.top() + 1) * c.n() * 8;
        c.download(pk_b, c.pk.get(), poly);
        c.download(pk_a, c.pk.as<u64>() + poly / 8, poly);
    });
}

int hecnn_eval_key_digits(const hecnn_context* ctx, size_t* digits) {
    return guard([&] { *digits = C(ctx).evk_digits; });
}

int hecnn_export_eval_key(const hecnn_context* ctx, uint64_t* evk) {
    return guard([&] {
        Context& c = *const_cast<hecnn_context*>(ctx)->ctx;
        if (!c.evk_digits) throw std::invalid_argument("no evaluation key");
        c.download(evk, c.evk.get(), c.evk.bytes());
    });
}

int hecnn_device_alloc(hecnn_context* ctx, size_t bytes, void** dptr) {
    return guard([&] {
        Context& c = C(ctx);
        void* p = nullptr;
        if (cudaMalloc(&p, bytes) != cudaSuccess) throw std::runtime_error("cudaMalloc failed");
        (void)c;
        *dptr = p;
    });
}

int hecnn_device_free(hecnn_context* ctx, void* dptr) {
    return guard([&] {
        C(ctx).sync();
        cudaFree(dptr);
    });
}

int hecnn_memcpy_h2d(hecnn_context* ctx, void* dst, const void* src, size_t bytes) {
    return guard([&] { C(ctx).upload(dst, src, bytes); });
}

int hecnn_memcpy_d2h(hecnn_context* ctx, void* dst, const void* src, size_t bytes) {
    return guard([&] { C(ctx).download(dst, src, bytes); });
}

int hecnn_ntt_forward(hecnn_context* ctx, uint64_t* polys, size_t level, size_t count) {
    return guard([&] {
        Context& c = C(ctx);
        if (level > c.top()) throw std::invalid_argument("ntt_transform: level out of range");
        ntt_forward(c.dev, polys, static_cast<int>(level), count, c.L());
    });
}

int hecnn_ntt_inverse(hecnn_context* ctx, uint64_t* polys, size_t level, size_t count) {
    return guard([&] {
        Context& c = C(ctx);
        if (level > c.top()) throw std::invalid_argument("ntt_transform: level out of range");
        ntt_inverse(c.dev, polys, static_cast<int>(level), count, c.L());
    });
}

static int ew(hecnn_context* ctx, EwOp op, const uint64_t* a, const uint64_t* b, uint64_t* out, size_t level,
              size_t count) {
    return guard([&] {
        Context& c = C(ctx);
        if (level > c.top()) throw std::invalid_argument("ring op: level out of range");
        poly_elementwise(c.dev, op, a, b, out, static_cast<int>(level), count, c.L());
    });
}

int hecnn_poly_add(hecnn_context* ctx, const uint64_t* a, const uint64_t* b, uint64_t* out, size_t level, size_t count) {
    return ew(ctx, EwOp::Add, a, b, out, level, count);
}
int hecnn_poly_sub(hecnn_context* ctx, const uint64_t* a, const uint64_t* b, uint64_t* out, size_t level, size_t count) {
    return ew(ctx, EwOp::Sub, a, b, out, level, count);
}
int hecnn_poly_neg(hecnn_context* ctx, const uint64_t* a, uint64_t* out, size_t level, size_t count) {
    return ew(ctx, EwOp::Neg, a, nullptr, out, level, count);
}
int hecnn_poly_pointwise_mul(hecnn_context* ctx, const uint64_t* a, const uint64_t* b, uint64_t* out, size_t level,
                             size_t count) {
    return ew(ctx, EwOp::Mul, a, b, out, level, count);
}
int hecnn_poly_pointwise_mac(hecnn_context* ctx, uint64_t* acc, const uint64_t* a, const uint64_t* b, size_t level,
                             size_t count) {
    return ew(ctx, EwOp::Mac, a, b, acc, level, count);
}

int hecnn_rescale_poly(hecnn_context* ctx, const uint64_t* in, uint64_t* out, size_t level, size_t count) {
    return guard([&] {
        Context& c = C(ctx);
        if (level == 0) throw std::invalid_argument("rescale_poly: already at last level");
        if (level > c.top()) throw std::invalid_argument("rescale_poly: level out of range");
        rescale(c.dev, in, out, static_cast<int>(level), count, c.L());
    });
}

int hecnn_key_switch(hecnn_context* ctx, const uint64_t* d2, uint64_t* out, size_t level, size_t count) {
    return guard([&] {
        Context& c = C(ctx);
        if (level > c.top()) throw std::invalid_argument("key_switch: level out of range");
        key_switch_raw(c, d2, out, level, count);
    });
}

int hecnn_tensor_create(hecnn_context* ctx, size_t cells, uint32_t level, double scale, hecnn_tensor** out) {
    return guard([&] {
        Context& c = C(ctx);
        if (level > c.top()) throw std::invalid_argument("tensor: level out of range");
        *out = wrap(ctx, make_tensor(c, cells, level, scale));
    });
}

int hecnn_tensor_destroy(hecnn_tensor* t) {
    return guard([&] {
        if (t && t->t) cudaSetDevice(t->t->ctx->device);
        delete t;
    });
}

int hecnn_tensor_info(const hecnn_tensor* t, size_t* cells, uint32_t* level, double* scale) {
    return guard([&] {
        const Tensor& x = T(t);
        if (cells) *cells = x.cells;
        if (level) *level = x.level;
        if (scale) *scale = x.scale;
    });
}

int hecnn_tensor_set_shape(hecnn_tensor* t, int flat, size_t h, size_t w, size_t c, size_t batch) {
    return guard([&] {
        Tensor& x = *t->t;
        Shape s = flat ? Shape::flattened(h) : Shape::spatial(h, w, c);
        if (s.positions() != x.cells) throw std::invalid_argument("tensor: shape does not match the cell count");
        x.shape = s;
        x.batch = batch;
    });
}

int hecnn_tensor_shape(const hecnn_tensor* t, int* flat, size_t* h, size_t* w, size_t* c, size_t* batch) {
    return guard([&] {
        const Tensor& x = T(t);
        *flat = x.shape.flat ? 1 : 0;
        *h = x.shape.flat ? x.shape.feat : x.shape.h;
        *w = x.shape.w;
        *c = x.shape.c;
        *batch = x.batch;
    });
}

int hecnn_tensor_data(const hecnn_tensor* t, uint64_t** dptr) {
    return guard([&] { *dptr = T(t).data(); });
}

int hecnn_tensor_upload(hecnn_context* ctx, hecnn_tensor* t, const uint64_t* host) {
    return guard([&] { C(ctx).upload(t->t->data(), host, t->t->cells * t->t->cell_words() * 8); });
}

int hecnn_tensor_download(hecnn_context* ctx, const hecnn_tensor* t, uint64_t* host) {
    return guard([&] { C(ctx).download(host, T(t).data(), T(t).cells * T(t).cell_words() * 8); });
}

int hecnn_tensor_upload_async(hecnn_context* ctx, hecnn_tensor* t, const uint64_t* host, void* stream) {
    return guard([&] {
        if (!host) throw std::invalid_argument("tensor_upload_async: null host buffer");
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : C(ctx).stream;
        cuda_check(cudaMemcpyAsync(t->t->data(), host, t->t->cells * t->t->cell_words() * 8, cudaMemcpyHostToDevice, st),
                   "cudaMemcpyAsync H2D");
    });
}

int hecnn_tensor_download_async(hecnn_context* ctx, const hecnn_tensor* t, uint64_t* host, void* stream) {
    return guard([&] {
        if (!host) throw std::invalid_argument("tensor_download_async: null host buffer");
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : C(ctx).stream;
        cuda_check(cudaMemcpyAsync(host, T(t).data(), T(t).cells * T(t).cell_words() * 8, cudaMemcpyDeviceToHost, st),
                   "cudaMemcpyAsync D2H");
    });
}

int hecnn_encrypt_tensor(hecnn_context* ctx, const double* data, size_t batch, size_t positions, uint64_t seed,
                         hecnn_tensor** out) {
    return guard([&] { *out = wrap(ctx, encrypt_tensor(C(ctx), data, batch, positions, seed)); });
}

int hecnn_encrypt_raw(hecnn_context* ctx, const uint64_t* m, const int64_t* r, const int64_t* e0, const int64_t* e1,
                      size_t count, double scale, hecnn_tensor** out) {
    return guard([&] {
        *out = wrap(ctx, encrypt_raw(C(ctx), m, reinterpret_cast<const long long*>(r),
                                reinterpret_cast<const long long*>(e0), reinterpret_cast<const long long*>(e1), count,
                                scale));
    });
}

int hecnn_decrypt_raw(hecnn_context* ctx, const hecnn_tensor* t, uint64_t* out_host) {
    return guard([&] { decrypt_raw(C(ctx), T(t), out_host); });
}

int hecnn_decrypt_tensor(hecnn_context* ctx, const hecnn_tensor* t, size_t batch, double* out) {
    return guard([&] { decrypt_tensor(C(ctx), T(t), batch, out); });
}

int hecnn_ct_add(hecnn_context* ctx, const hecnn_tensor* x, const hecnn_tensor* y, hecnn_tensor** out) {
    return guard([&] { *out = wrap(ctx, ct_add(C(ctx), T(x), T(y), false)); });
}
int hecnn_ct_sub(hecnn_context* ctx, const hecnn_tensor* x, const hecnn_tensor* y, hecnn_tensor** out) {
    return guard([&] { *out = wrap(ctx, ct_add(C(ctx), T(x), T(y), true)); });
}
int hecnn_ct_mul(hecnn_context* ctx, const hecnn_tensor* x, const hecnn_tensor* y, hecnn_tensor** out) {
    return guard([&] { *out = wrap(ctx, ct_mul(C(ctx), T(x), T(y))); });
}
int hecnn_ct_square(hecnn_context* ctx, const hecnn_tensor* x, hecnn_tensor** out) {
    return guard([&] { *out = wrap(ctx, ct_square(C(ctx), T(x))); });
}
int hecnn_ct_rescale(hecnn_context* ctx, const hecnn_tensor* x, hecnn_tensor** out) {
    return guard([&] { *out = wrap(ctx, ct_rescale(C(ctx), T(x))); });
}
int hecnn_ct_mod_switch(hecnn_context* ctx, const hecnn_tensor* x, uint32_t to_level, hecnn_tensor** out) {
    return guard([&] { *out = wrap(ctx, ct_mod_switch(C(ctx), T(x), to_level)); });
}
int hecnn_ct_mul_const(hecnn_context* ctx, const hecnn_tensor* x, double c, double scale, hecnn_tensor** out) {
    return guard([&] { *out = wrap(ctx, ct_mul_const(C(ctx), T(x), c, scale)); });
}
int hecnn_ct_add_const(hecnn_context* ctx, const hecnn_tensor* x, double c, hecnn_tensor** out) {
    return guard([&] { *out = wrap(ctx, ct_add_const(C(ctx), T(x), c)); });
}

int hecnn_make_scalar_plain(hecnn_context* ctx, double c, double scale, size_t level, uint64_t* residues_out) {
    return guard([&] {
        Context& cx = C(ctx);
        if (level > cx.top()) throw std::invalid_argument("make_scalar_plain: level above the chain");
        if (!residues_out) throw std::invalid_argument("make_scalar_plain: null output");
        const ScalarPlain sp = make_scalar_plain(cx, c, scale, level);
        std::copy(sp.residues.begin(), sp.residues.end(), residues_out);
    });
}
int hecnn_ct_zero(hecnn_context* ctx, size_t cells, uint32_t level, double scale, hecnn_tensor** out) {
    return guard([&] { *out = wrap(ctx, ct_zero(C(ctx), cells, level, scale)); });
}
int hecnn_ct_add_inplace(hecnn_context* ctx, hecnn_tensor* acc, const hecnn_tensor* x) {
    return guard([&] { ct_add_inplace(C(ctx), TM(ctx, acc), T(x)); });
}
int hecnn_ct_scalar_mac(hecnn_context* ctx, hecnn_tensor* acc, const hecnn_tensor* x, const uint64_t* residues,
                        size_t ncs, double sp_scale, uint32_t sp_level) {
    return guard([&] {
        if (!residues) throw std::invalid_argument("mul_scalar_mac: null residues");
        ct_scalar_mac(C(ctx), TM(ctx, acc), T(x), residues, ncs, sp_scale, sp_level);
    });
}
int hecnn_ct_add_scalar(hecnn_context* ctx, hecnn_tensor* ct, double c) {
    return guard([&] { ct_add_scalar(C(ctx), TM(ctx, ct), c); });
}
int hecnn_ct_add_plain(hecnn_context* ctx, const hecnn_tensor* x, const uint64_t* pt, uint32_t pt_level,
                       double pt_scale, hecnn_tensor** out) {
    return guard([&] {
        if (!pt) throw std::invalid_argument("add_plain: null plaintext");
        *out = wrap(ctx, ct_add_plain(C(ctx), T(x), pt, pt_level, pt_scale));
    });
}
int hecnn_ct_mul_plain(hecnn_context* ctx, const hecnn_tensor* x, const uint64_t* pt, uint32_t pt_level,
                       double pt_scale, int is_constant, int rescale, hecnn_tensor** out) {
    return guard([&] {
        if (!pt) throw std::invalid_argument("mul_plain: null plaintext");
        *out = wrap(ctx, ct_mul_plain(C(ctx), T(x), pt, pt_level, pt_scale, is_constant != 0, rescale != 0));
    });
}

int hecnn_eval_activation(hecnn_context* ctx, const double* coefficients, size_t n_coefficients, double interval_bound,
                          const hecnn_tensor* x, hecnn_tensor** out) {
    return guard([&] {
        Activation a{std::vector<double>(coefficients, coefficients + n_coefficients), interval_bound};
        *out = wrap(ctx, eval_activation(C(ctx), a, T(x)));
    });
}

int hecnn_model_create(hecnn_context* ctx, const hecnn_model_desc* d, hecnn_model** out) {
    return guard([&] {
        (void)C(ctx);
        auto h = std::make_unique<hecnn_model>();
        h->keep = owner(ctx);
        Model& m = h->m;
        m.input = d->input_flat ? Shape::flattened(d->input_features)
                                : Shape::spatial(d->input_h, d->input_w, d->input_c);
        for (size_t a = 0; a < d->n_activations; ++a) {
            Activation act;
            act.coefficients.assign(d->activations[a].coefficients,
                                    d->activations[a].coefficients + d->activations[a].n_coefficients);
            act.interval_bound = d->activations[a].interval_bound;
            m.acts.push_back(act);
        }
        for (size_t i = 0; i < d->n_layers; ++i) {
            const hecnn_layer_desc& L = d->layers[i];
            Layer l;
            l.kind = L.kind;
            if (l.kind < 0 || l.kind > 5) throw std::invalid_argument("model: unknown layer kind");
            l.filters = static_cast<size_t>(L.filters);
            l.kh = static_cast<size_t>(L.kernel_h);
            l.kw = static_cast<size_t>(L.kernel_w);
            l.stride = static_cast<size_t>(L.stride);
            l.valid = L.padding_valid != 0;
            l.pool = static_cast<size_t>(L.pool);
            l.pad = static_cast<size_t>(L.pad);
            l.units = static_cast<size_t>(L.units);
            l.act = L.activation;
            if (L.weights) l.w.assign(L.weights, L.weights + L.n_weights);
            if (L.biases) l.b.assign(L.biases, L.biases + L.n_biases);
            m.layers.push_back(std::move(l));
        }
        *out = h.release();
    });
}

int hecnn_model_destroy(hecnn_model* m) {
    return guard([&] { delete m; });
}

int hecnn_model_depth_cost(const hecnn_model* m, size_t* cost) {
    return guard([&] {
        const_cast<hecnn_model*>(m)->m.infer_shapes();
        *cost = m->m.depth_cost();
    });
}

int hecnn_model_set_streaming(hecnn_model* m, int mode, size_t tile, size_t mem_budget) {
    return guard([&] {
        if (!m) throw std::invalid_argument("model: null handle");
        if (mode < 0 || mode > 2) throw std::invalid_argument("model: streaming mode must be 0, 1 or 2");
        m->m.stream_mode = mode;
        m->m.stream_tile = tile;
        m->m.mem_budget = mem_budget;
        m->m.plans.clear();
    });
}

int hecnn_forward_encrypted(hecnn_context* ctx, const hecnn_model* m, const hecnn_tensor* x, uint64_t seed,
                            hecnn_tensor** out, double* layer_seconds) {
    return guard([&] {
        *out = wrap(ctx, forward_encrypted(C(ctx), const_cast<hecnn_model*>(m)->m, T(x), seed, layer_seconds));
    });
}


// ---------------------------------------------------------------- CKKS blob v1

namespace {

blob::Params ctx_params(const Context& c) {
    blob::Params p;
    p.n = c.n();
    p.primes = c.ring.primes;
    p.scale = c.scale;
    p.sigma = c.sigma;
    p.degenerate = c.degenerate;
    return p;
}

void emit(const std::vector<uint8_t>& b, uint8_t* buf, size_t cap, size_t* len) {
    if (!len) throw std::invalid_argument("blob: null length pointer");
    *len = b.size();
    if (!buf) return;
    if (cap < b.size()) throw std::invalid_argument("blob: buffer too small");
    std::memcpy(buf, b.data(), b.size());
}

void require_same(const blob::Params& p, const Context& c) {
    if (!blob::same(p, ctx_params(c))) throw std::invalid_argument("ckks blob: parameters differ from the context");
}

}  // namespace

int hecnn_blob_params(const uint8_t* blob, size_t len, int* kind, size_t* n, uint64_t* primes, size_t* nprimes,
                      double* scale, double* sigma, int* degenerate) {
    return guard([&] {
        uint16_t k = 0;  // peeked so the header check accepts any kind; a short blob fails in the reader
        if (blob && len >= 8) std::memcpy(&k, blob + 6, 2);
        blob::Reader r(blob, len);
        const blob::Params p = r.header(static_cast<blob::Kind>(k));
        if (kind) *kind = k;
        if (n) *n = p.n;
        if (nprimes) {
            if (primes && *nprimes < p.primes.size()) throw std::invalid_argument("blob: primes buffer too small");
            if (primes) std::memcpy(primes, p.primes.data(), p.primes.size() * 8);
            *nprimes = p.primes.size();
        }
        if (scale) *scale = p.scale;
        if (sigma) *sigma = p.sigma;
        if (degenerate) *degenerate = p.degenerate ? 1 : 0;
    });
}

int hecnn_blob_save_key(const hecnn_context* ctx, int kind, uint8_t* buf, size_t cap, size_t* len) {
    return guard([&] {
        Context& c = *const_cast<hecnn_context*>(ctx)->ctx;
        const std::size_t L = c.top(), n = c.n(), poly = (L + 1) * n;
        blob::Writer w;
        if (kind == HECNN_BLOB_SECRET_KEY) {
            if (!c.has_secret) throw std::invalid_argument("no secret key");
            w.header(blob::kSecret, ctx_params(c));
            w.poly(static_cast<uint16_t>(L), 0, c.secret_host.data(), n);  // Coeff
        } else if (kind == HECNN_BLOB_PUBLIC_KEY) {
            if (!c.has_pk) throw std::invalid_argument("no public key");
            std::vector<u64> ba(2 * poly);
            c.download(ba.data(), c.pk.get(), 2 * poly * 8);
            w.header(blob::kPublic, ctx_params(c));
            w.poly(static_cast<uint16_t>(L), 1, ba.data(), n);  // b, NTT
            w.poly(static_cast<uint16_t>(L), 1, ba.data() + poly, n);
        } else if (kind == HECNN_BLOB_EVAL_KEY) {
            if (!c.evk_digits) throw std::invalid_argument("no evaluation key");
            std::vector<u64> evk(c.evk_digits * 2 * poly);
            c.download(evk.data(), c.evk.get(), evk.size() * 8);
            w.header(blob::kEval, ctx_params(c));
            w.le<uint16_t>(20);  // base_bits (kRelinBaseBits)
            w.le<uint16_t>(static_cast<uint16_t>(c.evk_digits));
            for (std::size_t t = 0; t < 2 * c.evk_digits; ++t) w.poly(static_cast<uint16_t>(L), 1, evk.data() + t * poly, n);
        } else {
            throw std::invalid_argument("blob: unknown key kind");
        }
        emit(w.bytes(), buf, cap, len);
    });
}

int hecnn_blob_load_key(hecnn_context* ctx, int kind, const uint8_t* data, size_t len) {
    return guard([&] {
        Context& c = C(ctx);
        const std::size_t L = c.top(), n = c.n(), poly = (L + 1) * n;
        if (kind < HECNN_BLOB_SECRET_KEY || kind > HECNN_BLOB_EVAL_KEY) throw std::invalid_argument("blob: unknown key kind");
        blob::Reader r(data, len);
        require_same(r.header(static_cast<blob::Kind>(kind)), c);
        auto top_poly = [&](u64* dst, uint8_t want_rep, const char* what) {
            const auto [level, rep] = r.poly(dst, n, poly, c.ring.primes.data());
            if (level != L || rep != want_rep)
                throw std::invalid_argument(std::string("ckks blob: ") + what + " must be a top-level " +
                                            (want_rep ? "NTT" : "coefficient") + "-domain polynomial");
        };
        if (kind == HECNN_BLOB_SECRET_KEY) {
            std::vector<u64> s(poly);
            top_poly(s.data(), 0, "secret key");
            import_keys(c, s.data(), nullptr, nullptr, nullptr, 0);
        } else if (kind == HECNN_BLOB_PUBLIC_KEY) {
            std::vector<u64> b(poly), a(poly);
            top_poly(b.data(), 1, "public key");
            top_poly(a.data(), 1, "public key");
            import_keys(c, nullptr, b.data(), a.data(), nullptr, 0);
        } else {
            if (r.le<uint16_t>() != 20) throw std::invalid_argument("mul: unexpected evk digit base");
            const std::size_t D = r.le<uint16_t>();
            std::vector<u64> evk(D * 2 * poly);
            for (std::size_t t = 0; t < 2 * D; ++t) top_poly(evk.data() + t * poly, 1, "evaluation key");
            import_keys(c, nullptr, nullptr, nullptr, evk.data(), D);
        }
    });
}

int hecnn_blob_save_ciphertext(hecnn_context* ctx, const hecnn_tensor* t, size_t cell, uint8_t* buf, size_t cap,
                               size_t* len) {
    return guard([&] {
        Context& c = C(ctx);
        const Tensor& x = T(t);
        if (cell >= x.cells) throw std::invalid_argument("blob: cell index out of range");
        const std::size_t n = c.n(), rows = (x.level + 1) * n;
        std::vector<u64> words(2 * rows);
        c.download(words.data(), x.cell(cell), words.size() * 8);
        blob::Writer w;
        w.header(blob::kCipher, ctx_params(c));
        w.le<double>(x.scale);
        w.le<uint16_t>(static_cast<uint16_t>(x.level));
        w.poly(static_cast<uint16_t>(x.level), 0, words.data(), n);  // c0, Coeff
        w.poly(static_cast<uint16_t>(x.level), 0, words.data() + rows, n);
        emit(w.bytes(), buf, cap, len);
    });
}

int hecnn_blob_load_ciphertexts(hecnn_context* ctx, const uint8_t* const* blobs, const size_t* lens, size_t count,
                                hecnn_tensor** out) {
    return guard([&] {
        Context& c = C(ctx);
        if (!count) throw std::invalid_argument("blob: no ciphertexts");
        const std::size_t n = c.n();
        std::vector<u64> host;
        uint32_t level = 0;
        double scale = 0.0;
        for (std::size_t k = 0; k < count; ++k) {
            blob::Reader r(blobs[k], lens[k]);
            require_same(r.header(blob::kCipher), c);
            const double s = r.le<double>();
            const uint32_t l = r.le<uint16_t>();
            if (l > c.top()) throw std::invalid_argument("ckks blob: ciphertext level exceeds the context's chain");
            if (k == 0) {
                level = l, scale = s;
                host.resize(count * 2 * (level + 1) * n);
            } else if (l != level || s != scale) {
                // TensorEncrypted keeps one (scale, level) for all cells (tensor.hpp:52-62)
                throw std::invalid_argument("blob: ciphertexts of one tensor must share level and scale");
            }
            u64* dst = host.data() + k * 2 * (level + 1) * n;
            for (int comp = 0; comp < 2; ++comp) {
                // storage for this cell is sized by the header level: a polynomial
                // declaring a higher level is rejected before any word is copied
                const auto [pl, rep] = r.poly(dst + comp * (level + 1) * n, n, (level + 1) * n, c.ring.primes.data());
                if (pl != level || rep != 0)
                    throw std::invalid_argument("ckks blob: ciphertext polynomials must be coefficient-domain at the ciphertext level");
            }
        }
        TensorPtr t = make_tensor(c, count, level, scale);
        c.upload(t->data(), host.data(), host.size() * 8);
        *out = wrap(ctx, std::move(t));
    });
}

}  // extern "C"
