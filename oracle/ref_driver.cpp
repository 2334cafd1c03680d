// TEST INFRASTRUCTURE ONLY -- the parity checker, never the product.
//
// C-ABI driver around the UNMODIFIED reference library (hecnn, header-only
// C++20, /root/reference/proj/include/hecnn). Built by oracle/Makefile into
// oracle/_ref/libhecnn_ref.so from the reference's own headers, with the
// reference's CMake Release flags (-O3 -DNDEBUG, no -march; proj/CMakeLists.txt:6-8).
// Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
// --impl reference) load it. Every function forwards to the reference API
// named beside it; no arithmetic of its own.

#include <chrono>
#include <cstring>
#include <memory>
#include <string>

#include <sstream>

#include "hecnn/ckks_serialize.hpp"
#include "hecnn/layers.hpp"
#include "hecnn/model_io.hpp"
#include "hecnn/presets.hpp"
#include "hecnn/synthetic.hpp"
#include "hecnn_b200.h"

using namespace hecnn;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

struct RefEngine {
    CkksEngine eng;
    explicit RefEngine(CkksParams p) : eng(std::move(p)) {}
};

struct RefTensor {
    TensorEncrypted t;
};

RingPoly poly_from(const RingContext& ctx, const uint64_t* src, std::size_t level, Rep rep) {
    RingPoly p = make_zero_poly(ctx, level, rep);
    std::size_t n = ctx.degree();
    for (std::size_t i = 0; i <= level; ++i) std::memcpy(p.rns[i].data(), src + i * n, n * 8);
    return p;
}

void poly_to(const RingPoly& p, uint64_t* dst) {
    std::size_t n = p.degree();
    for (std::size_t i = 0; i < p.rns.size(); ++i) std::memcpy(dst + i * n, p.rns[i].data(), n * 8);
}

Ciphertext ct_from(const CkksEngine& e, const uint64_t* src, std::size_t level, double scale) {
    std::size_t n = e.ring().degree();
    Ciphertext ct;
    ct.c0 = poly_from(e.ring(), src, level, Rep::Coeff);
    ct.c1 = poly_from(e.ring(), src + (level + 1) * n, level, Rep::Coeff);
    ct.scale = scale;
    ct.level = static_cast<u32>(level);
    return ct;
}

void ct_to(const CkksEngine& e, const Ciphertext& ct, uint64_t* dst) {
    std::size_t n = e.ring().degree();
    poly_to(ct.c0, dst);
    poly_to(ct.c1, dst + (ct.level + 1) * n);
}

ModelSpec model_from(const hecnn_model_desc* d) {
    ModelSpec m;
    m.input = d->input_flat ? Shape::flattened(d->input_features)
                            : Shape::spatial(d->input_h, d->input_w, d->input_c);
    for (std::size_t a = 0; a < d->n_activations; ++a) {
        PolyActivation act;
        act.coefficients.assign(d->activations[a].coefficients,
                                d->activations[a].coefficients + d->activations[a].n_coefficients);
        act.interval_bound = d->activations[a].interval_bound;
        act.source = "relu";
        m.activations["act" + std::to_string(a)] = act;
    }
    for (std::size_t i = 0; i < d->n_layers; ++i) {
        const hecnn_layer_desc& L = d->layers[i];
        LayerSpec l;
        switch (L.kind) {
            case HECNN_LAYER_CONV2D:
                l = LayerSpec::conv2d(L.filters, L.kernel_h, L.kernel_w, L.stride,
                                      L.padding_valid ? LayerSpec::Padding::Valid : LayerSpec::Padding::Same);
                break;
            case HECNN_LAYER_AVG_POOL2D: l = LayerSpec::avg_pool2d(L.pool); break;
            case HECNN_LAYER_ZERO_PAD2D: l = LayerSpec::zero_pad2d(L.pad); break;
            case HECNN_LAYER_DENSE: l = LayerSpec::dense(L.units); break;
            case HECNN_LAYER_ACTIVATION: l = LayerSpec::activation("act" + std::to_string(L.activation)); break;
            case HECNN_LAYER_SIGMOID: l = LayerSpec::sigmoid(); break;
            default: throw std::invalid_argument("ref: unknown layer kind");
        }
        m.layers.push_back(l);
    }
    m.ensure_param_slots();
    for (std::size_t i = 0; i < d->n_layers; ++i) {
        const hecnn_layer_desc& L = d->layers[i];
        if (L.weights) m.weights[i].assign(L.weights, L.weights + L.n_weights);
        if (L.biases) m.biases[i].assign(L.biases, L.biases + L.n_biases);
    }
    return m;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// RingParams::create (ring.hpp:20-30)
int ref_find_chain(size_t n, const int* bits, size_t count, uint64_t* out) {
    return guard([&] {
        RingParams p = RingParams::create(n, std::vector<int>(bits, bits + count));
        for (size_t i = 0; i < count; ++i) out[i] = p.primes[i];
    });
}

// CkksEngine(CkksParams) (ckks.hpp:79-93)
int ref_engine_create(size_t n, const uint64_t* primes, size_t nprimes, double scale, double sigma, int degenerate,
                      void** out) {
    return guard([&] {
        CkksParams p;
        p.ring.n = n;
        p.ring.primes.assign(primes, primes + nprimes);
        p.ring.finalize();
        p.scale = scale;
        p.sigma = sigma;
        p.degenerate_noise = degenerate != 0;
        *out = new RefEngine(p);
    });
}

void ref_engine_destroy(void* e) { delete static_cast<RefEngine*>(e); }

int ref_relin_digits(void* e, size_t level, size_t* out) {
    return guard([&] { *out = static_cast<RefEngine*>(e)->eng.relin_digits(level); });
}

// NttTables::forward / inverse (ring.hpp:83-137), one limb in place
int ref_ntt_forward(void* e, size_t limb, uint64_t* a) {
    return guard([&] { static_cast<RefEngine*>(e)->eng.ring().ntt(limb).forward(a); });
}
int ref_ntt_inverse(void* e, size_t limb, uint64_t* a) {
    return guard([&] { static_cast<RefEngine*>(e)->eng.ring().ntt(limb).inverse(a); });
}

// sample_poly Uniform (ring.hpp:461-470)
int ref_sample_uniform(void* e, size_t level, uint64_t seed, uint64_t* out) {
    return guard([&] {
        const CkksEngine& eng = static_cast<RefEngine*>(e)->eng;
        poly_to(sample_poly(eng.ring(), SampleKind::Uniform, {.level = level}, seed), out);
    });
}

// rescale_poly (ring.hpp:419-442)
int ref_rescale_poly(void* e, const uint64_t* in, size_t level, uint64_t* out) {
    return guard([&] {
        const CkksEngine& eng = static_cast<RefEngine*>(e)->eng;
        poly_to(rescale_poly(eng.ring(), poly_from(eng.ring(), in, level, Rep::Coeff)), out);
    });
}

// reconstruct_mod_q (ring.hpp:529-538): words little-endian, `words` per coefficient
int ref_reconstruct(void* e, const uint64_t* in, size_t level, size_t words, uint64_t* out) {
    return guard([&] {
        const CkksEngine& eng = static_cast<RefEngine*>(e)->eng;
        RingPoly p = poly_from(eng.ring(), in, level, Rep::Coeff);
        for (size_t j = 0; j < eng.ring().degree(); ++j) {
            BigUInt v = reconstruct_mod_q(eng.ring(), p, j);
            for (size_t w = 0; w < words; ++w) out[j * words + w] = v.limb(w);
        }
    });
}

// CkksEngine::keygen (ckks.hpp:200-236)
int ref_keygen(void* e, uint64_t seed, void** out) {
    return guard([&] { *out = new KeySet(static_cast<RefEngine*>(e)->eng.keygen(seed)); });
}
void ref_keys_destroy(void* k) { delete static_cast<KeySet*>(k); }
size_t ref_eval_key_digits(void* k) { return static_cast<KeySet*>(k)->eval.pairs.size(); }
void ref_export_keys(void* k, uint64_t* s, uint64_t* pk_b, uint64_t* pk_a, uint64_t* evk) {
    KeySet* ks = static_cast<KeySet*>(k);
    if (s) poly_to(ks->secret.s, s);
    if (pk_b) poly_to(ks->public_key.b, pk_b);
    if (pk_a) poly_to(ks->public_key.a, pk_a);
    if (evk) {
        std::size_t per = ks->eval.pairs[0].first.rns.size() * ks->eval.pairs[0].first.degree();
        for (std::size_t t = 0; t < ks->eval.pairs.size(); ++t) {
            poly_to(ks->eval.pairs[t].first, evk + (2 * t) * per);
            poly_to(ks->eval.pairs[t].second, evk + (2 * t + 1) * per);
        }
    }
}

// encode_real + encrypt(pk, m, seed) (ckks.hpp:125-129, 268-270)
int ref_encrypt(void* e, void* k, const double* slots, size_t nslots, double scale, uint64_t seed, uint64_t* out) {
    return guard([&] {
        const CkksEngine& eng = static_cast<RefEngine*>(e)->eng;
        EncodedPlaintext m = eng.encode_real(std::vector<double>(slots, slots + nslots), scale, eng.top_level());
        ct_to(eng, eng.encrypt(static_cast<KeySet*>(k)->public_key, m, seed), out);
    });
}

// encode_real only (ckks.hpp:105-129): out [(level+1)][n]
int ref_encode(void* e, const double* slots, size_t nslots, double scale, size_t level, uint64_t* out) {
    return guard([&] {
        const CkksEngine& eng = static_cast<RefEngine*>(e)->eng;
        poly_to(eng.encode_real(std::vector<double>(slots, slots + nslots), scale, level).poly, out);
    });
}

// decode (ckks.hpp:142-154) of a plaintext poly: real parts of the slots
int ref_decode(void* e, const uint64_t* poly, size_t level, double scale, double* out) {
    return guard([&] {
        const CkksEngine& eng = static_cast<RefEngine*>(e)->eng;
        EncodedPlaintext m{poly_from(eng.ring(), poly, level, Rep::Coeff), scale, false};
        PlaintextVector v = eng.decode(m);
        for (size_t i = 0; i < v.size(); ++i) out[i] = v[i].real();
    });
}

// make_encryption_randomness (ckks.hpp:238-244): signed coefficients
int ref_encryption_randomness(void* e, uint64_t seed, int64_t* r, int64_t* e0, int64_t* e1) {
    return guard([&] {
        const CkksEngine& eng = static_cast<RefEngine*>(e)->eng;
        EncryptionRandomness rr = eng.make_encryption_randomness(seed);
        const RingContext& ctx = eng.ring();
        u64 q = ctx.prime(0);
        auto signed_of = [&](const RingPoly& p, int64_t* dst) {
            for (size_t j = 0; j < ctx.degree(); ++j) {
                u64 v = p.rns[0][j];
                dst[j] = v > q / 2 ? -static_cast<int64_t>(q - v) : static_cast<int64_t>(v);
            }
        };
        signed_of(rr.r, r);
        signed_of(rr.e0, e0);
        signed_of(rr.e1, e1);
    });
}

// decrypt + decode (ckks.hpp:273-279, 142-154)
int ref_decrypt(void* e, void* k, const uint64_t* ct, size_t level, double scale, double* slots_out) {
    return guard([&] {
        const CkksEngine& eng = static_cast<RefEngine*>(e)->eng;
        PlaintextVector v = eng.decode(eng.decrypt(static_cast<KeySet*>(k)->secret, ct_from(eng, ct, level, scale)));
        for (size_t i = 0; i < v.size(); ++i) slots_out[i] = v[i].real();
    });
}

// decrypt only: plaintext poly [(level+1)][n]
int ref_decrypt_raw(void* e, void* k, const uint64_t* ct, size_t level, double scale, uint64_t* out) {
    return guard([&] {
        const CkksEngine& eng = static_cast<RefEngine*>(e)->eng;
        poly_to(eng.decrypt(static_cast<KeySet*>(k)->secret, ct_from(eng, ct, level, scale)).poly, out);
    });
}

// CkksEngine::mul (ckks.hpp:315-342)
int ref_mul(void* e, void* k, const uint64_t* x, const uint64_t* y, size_t level, double sx, double sy,
            uint64_t* out, double* out_scale) {
    return guard([&] {
        const CkksEngine& eng = static_cast<RefEngine*>(e)->eng;
        Ciphertext r = eng.mul(ct_from(eng, x, level, sx), ct_from(eng, y, level, sy), static_cast<KeySet*>(k)->eval);
        ct_to(eng, r, out);
        *out_scale = r.scale;
    });
}

// CkksEngine::square (ckks.hpp:345-369)
int ref_square(void* e, void* k, const uint64_t* x, size_t level, double sx, uint64_t* out, double* out_scale) {
    return guard([&] {
        const CkksEngine& eng = static_cast<RefEngine*>(e)->eng;
        Ciphertext r = eng.square(ct_from(eng, x, level, sx), static_cast<KeySet*>(k)->eval);
        ct_to(eng, r, out);
        *out_scale = r.scale;
    });
}

// CkksEngine::rescale (ckks.hpp:474-482)
int ref_rescale(void* e, const uint64_t* x, size_t level, double sx, uint64_t* out, double* out_scale) {
    return guard([&] {
        const CkksEngine& eng = static_cast<RefEngine*>(e)->eng;
        Ciphertext r = eng.rescale(ct_from(eng, x, level, sx));
        ct_to(eng, r, out);
        *out_scale = r.scale;
    });
}

// mul_plain(x, encode_const(c, scale, level)) (ckks.hpp:395-398)
int ref_mul_const(void* e, const uint64_t* x, size_t level, double sx, double c, double cscale, uint64_t* out,
                  double* out_scale) {
    return guard([&] {
        const CkksEngine& eng = static_cast<RefEngine*>(e)->eng;
        Ciphertext r = eng.mul_plain(ct_from(eng, x, level, sx), eng.encode_const(c, cscale, level));
        ct_to(eng, r, out);
        *out_scale = r.scale;
    });
}

// make_scalar_plain (ckks.hpp:407-423): residues of round(c * scale)
int ref_scalar_plain(void* e, double c, double scale, size_t level, uint64_t* out) {
    return guard([&] {
        const CkksEngine& eng = static_cast<RefEngine*>(e)->eng;
        CkksEngine::ScalarPlain sp = eng.make_scalar_plain(c, scale, level);
        std::memcpy(out, sp.residues.data(), sp.residues.size() * 8);
    });
}

// acc' = acc + x * make_scalar_plain(c, cscale) (mul_scalar_mac, ckks.hpp:448-465),
// then add_scalar_inplace(acc', b) when add_b != 0 (:468-472)
int ref_scalar_mac(void* e, const uint64_t* acc, const uint64_t* x, size_t level, double acc_scale, double sx,
                   double c, double cscale, int add_b, double b, uint64_t* out) {
    return guard([&] {
        const CkksEngine& eng = static_cast<RefEngine*>(e)->eng;
        Ciphertext a = ct_from(eng, acc, level, acc_scale);
        eng.mul_scalar_mac(a, ct_from(eng, x, level, sx), eng.make_scalar_plain(c, cscale, level));
        if (add_b) eng.add_scalar_inplace(a, b);
        ct_to(eng, a, out);
    });
}

// add_plain / mul_plain_raw / mul_plain of an encode_real plaintext (or
// encode_const(slots[0]) when constant) (ckks.hpp:305-311, 372-398)
int ref_plain_op(void* e, int op, const uint64_t* x, size_t level, double sx, const double* slots, size_t nslots,
                 double pscale, int constant, uint64_t* out, uint32_t* out_level, double* out_scale) {
    return guard([&] {
        const CkksEngine& eng = static_cast<RefEngine*>(e)->eng;
        EncodedPlaintext m = constant ? eng.encode_const(slots[0], pscale, level)
                                      : eng.encode_real(std::vector<double>(slots, slots + nslots), pscale, level);
        Ciphertext in = ct_from(eng, x, level, sx);
        Ciphertext r = op == 0 ? eng.add_plain(in, m) : (op == 1 ? eng.mul_plain_raw(in, m) : eng.mul_plain(in, m));
        ct_to(eng, r, out);
        *out_level = r.level;
        *out_scale = r.scale;
    });
}

// eval_encrypted (activation.hpp:228-265)
int ref_eval_activation(void* e, void* k, const double* coeffs, size_t ncoeffs, double bound, const uint64_t* x,
                        size_t level, double sx, uint64_t* out, uint32_t* out_level, double* out_scale) {
    return guard([&] {
        const CkksEngine& eng = static_cast<RefEngine*>(e)->eng;
        PolyActivation act{std::vector<double>(coeffs, coeffs + ncoeffs), bound, "relu"};
        Ciphertext r = eval_encrypted(act, ct_from(eng, x, level, sx), eng, static_cast<KeySet*>(k)->eval);
        ct_to(eng, r, out);
        *out_level = r.level;
        *out_scale = r.scale;
    });
}

// ---- tensors / network ----------------------------------------------------

// encrypt_tensor (tensor.hpp:77-94); data [batch][positions]
int ref_encrypt_tensor(void* e, void* k, const double* data, size_t batch, int flat, size_t h, size_t w, size_t c,
                       size_t feat, uint64_t seed, unsigned threads, void** out) {
    return guard([&] {
        const CkksEngine& eng = static_cast<RefEngine*>(e)->eng;
        TensorPlain x;
        x.shape = flat ? Shape::flattened(feat) : Shape::spatial(h, w, c);
        x.batch = batch;
        x.data.assign(data, data + batch * x.shape.positions());
        auto* t = new RefTensor{encrypt_tensor(eng, static_cast<KeySet*>(k)->public_key, x, seed, threads)};
        *out = t;
    });
}

// wrap raw ciphertext words as a TensorEncrypted
int ref_tensor_from(void* e, const uint64_t* cts, size_t cells, size_t level, double scale, int flat, size_t h,
                    size_t w, size_t c, size_t feat, size_t batch, void** out) {
    return guard([&] {
        const CkksEngine& eng = static_cast<RefEngine*>(e)->eng;
        auto* t = new RefTensor;
        t->t.shape = flat ? Shape::flattened(feat) : Shape::spatial(h, w, c);
        t->t.batch = batch;
        std::size_t per = 2 * (level + 1) * eng.ring().degree();
        for (size_t i = 0; i < cells; ++i) t->t.cells.push_back(ct_from(eng, cts + i * per, level, scale));
        *out = t;
    });
}

void ref_tensor_destroy(void* t) { delete static_cast<RefTensor*>(t); }

void ref_tensor_info(void* t, size_t* cells, uint32_t* level, double* scale) {
    RefTensor* r = static_cast<RefTensor*>(t);
    *cells = r->t.cells.size();
    *level = r->t.cells.empty() ? 0 : r->t.level();
    *scale = r->t.cells.empty() ? 0.0 : r->t.scale();
}

void ref_tensor_export(void* e, void* t, uint64_t* out) {
    const CkksEngine& eng = static_cast<RefEngine*>(e)->eng;
    RefTensor* r = static_cast<RefTensor*>(t);
    std::size_t n = eng.ring().degree();
    for (size_t i = 0; i < r->t.cells.size(); ++i) {
        const Ciphertext& ct = r->t.cells[i];
        ct_to(eng, ct, out + i * 2 * (ct.level + 1) * n);
    }
}

// decrypt_tensor (tensor.hpp:96-106): out [batch][positions]
int ref_decrypt_tensor(void* e, void* k, void* t, unsigned threads, double* out) {
    return guard([&] {
        const CkksEngine& eng = static_cast<RefEngine*>(e)->eng;
        TensorPlain p = decrypt_tensor(eng, static_cast<KeySet*>(k)->secret, static_cast<RefTensor*>(t)->t, threads);
        std::memcpy(out, p.data.data(), p.data.size() * sizeof(double));
    });
}

// forward_encrypted (layers.hpp:299-368)
int ref_forward_encrypted(void* e, void* k, const hecnn_model_desc* desc, void* x, uint64_t seed, unsigned threads,
                          void** out, double* layer_seconds) {
    return guard([&] {
        const CkksEngine& eng = static_cast<RefEngine*>(e)->eng;
        KeySet* ks = static_cast<KeySet*>(k);
        ModelSpec m = model_from(desc);
        EvalKeys keys{ks->public_key, ks->eval};
        std::vector<double> secs;
        auto* t = new RefTensor{forward_encrypted(m, static_cast<RefTensor*>(x)->t, eng, keys, seed, threads, &secs)};
        if (layer_seconds)
            for (size_t i = 0; i < secs.size(); ++i) layer_seconds[i] = secs[i];
        *out = t;
    });
}

// forward_plain (layers.hpp:141-168): data [batch][positions] -> out [batch][out positions]
int ref_forward_plain(const hecnn_model_desc* desc, const double* data, size_t batch, double* out) {
    return guard([&] {
        ModelSpec m = model_from(desc);
        TensorPlain x;
        x.shape = m.input;
        x.batch = batch;
        x.data.assign(data, data + batch * m.input.positions());
        TensorPlain y = forward_plain(m, x);
        std::memcpy(out, y.data.data(), y.data.size() * sizeof(double));
    });
}

// init_random_weights (model_io.hpp:183-203): fills the desc's weight/bias
// buffers (caller sizes them via shape inference).
int ref_init_random_weights(const hecnn_model_desc* desc, uint64_t seed, double* const* weights,
                            double* const* biases) {
    return guard([&] {
        ModelSpec m = model_from(desc);
        init_random_weights(m, seed);
        for (size_t i = 0; i < desc->n_layers; ++i) {
            if (weights[i]) std::memcpy(weights[i], m.weights[i].data(), m.weights[i].size() * sizeof(double));
            if (biases[i]) std::memcpy(biases[i], m.biases[i].data(), m.biases[i].size() * sizeof(double));
        }
    });
}

// save_model (model_io.hpp:61-103): manifest + weight blob at `base`
int ref_save_model(const hecnn_model_desc* desc, const char* base) {
    return guard([&] { save_model(base, model_from(desc)); });
}

// load_model (model_io.hpp:105-181) round trip: loads `base` and writes its
// weights / biases into the caller's buffers (sized by shape inference); the
// reference's errors for a malformed file come back as the status + message
int ref_load_model_weights(const char* base, double* const* weights, double* const* biases, size_t n_layers) {
    return guard([&] {
        ModelSpec m = load_model(base);
        if (!n_layers) return;  // validation only
        if (m.layers.size() != n_layers) throw std::invalid_argument("ref: layer count differs");
        for (size_t i = 0; i < n_layers; ++i) {
            if (weights[i]) std::memcpy(weights[i], m.weights[i].data(), m.weights[i].size() * sizeof(double));
            if (biases[i]) std::memcpy(biases[i], m.biases[i].data(), m.biases[i].size() * sizeof(double));
        }
    });
}

// gen_synthetic + save_dataset (synthetic.hpp:24-99): an HDTS file
int ref_save_dataset(size_t count, size_t image, size_t channels, uint64_t seed, const char* path) {
    return guard([&] {
        save_dataset(path, gen_synthetic({.count = count, .image = image, .channels = channels, .seed = seed}));
    });
}

// Rng::uniform01 stream (common.hpp:173-179): `count` draws from Rng(seed)
int ref_rng_uniform(uint64_t seed, size_t count, double* out) {
    return guard([&] {
        Rng rng(seed);
        for (size_t i = 0; i < count; ++i) out[i] = rng.uniform01();
    });
}

// gen_synthetic (synthetic.hpp:24-86): images [count][positions], labels
int ref_gen_synthetic(size_t count, size_t image, size_t channels, uint64_t seed, double* images, uint8_t* labels) {
    return guard([&] {
        Dataset ds = gen_synthetic({.count = count, .image = image, .channels = channels, .seed = seed});
        std::memcpy(images, ds.images.data.data(), ds.images.data.size() * sizeof(double));
        if (labels) std::memcpy(labels, ds.labels.data(), ds.labels.size());
    });
}

// ---- timing helpers for the CPU baseline (reference code path, parallel_for
// over independent ciphertexts exactly as its own call sites do) -------------

// `count` independent ntt forward+inverse passes over all limbs of a
// (level+1)-limb poly; returns seconds.
int ref_time_ntt(void* e, size_t level, size_t count, unsigned threads, double* secs) {
    return guard([&] {
        const CkksEngine& eng = static_cast<RefEngine*>(e)->eng;
        const RingContext& ctx = eng.ring();
        std::vector<RingPoly> polys(count);
        for (size_t i = 0; i < count; ++i)
            polys[i] = sample_poly(ctx, SampleKind::Uniform, {.level = level}, 1000 + i);
        auto t0 = std::chrono::steady_clock::now();
        parallel_for(count, threads, [&](std::size_t b, std::size_t en) {
            for (std::size_t i = b; i < en; ++i) {
                ntt_transform_inplace(ctx, polys[i], NttDirection::Forward);
                ntt_transform_inplace(ctx, polys[i], NttDirection::Inverse);
            }
        });
        *secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

// `count` independent mul(x_i, y_i, evk) at `level`; returns seconds.
int ref_time_mul(void* e, void* k, size_t level, size_t count, unsigned threads, double* secs) {
    return guard([&] {
        const CkksEngine& eng = static_cast<RefEngine*>(e)->eng;
        const RingContext& ctx = eng.ring();
        KeySet* ks = static_cast<KeySet*>(k);
        std::vector<Ciphertext> xs(count), ys(count);
        for (size_t i = 0; i < count; ++i) {
            xs[i].c0 = sample_poly(ctx, SampleKind::Uniform, {.level = level}, 1000 + 4 * i);
            xs[i].c1 = sample_poly(ctx, SampleKind::Uniform, {.level = level}, 1001 + 4 * i);
            ys[i].c0 = sample_poly(ctx, SampleKind::Uniform, {.level = level}, 1002 + 4 * i);
            ys[i].c1 = sample_poly(ctx, SampleKind::Uniform, {.level = level}, 1003 + 4 * i);
            xs[i].level = ys[i].level = static_cast<u32>(level);
            xs[i].scale = ys[i].scale = eng.params().scale;
        }
        std::vector<Ciphertext> out(count);
        auto t0 = std::chrono::steady_clock::now();
        parallel_for(count, threads, [&](std::size_t b, std::size_t en) {
            for (std::size_t i = b; i < en; ++i) out[i] = eng.mul(xs[i], ys[i], ks->eval);
        });
        *secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

// Per-op costs of the reference's layer kernels (layers.hpp:174-293,
// activation.hpp:228-265), `count` independent items over its parallel_for;
// returns seconds. op 0: eval_encrypted(relu_default_surrogate) at `level`;
// op 1: make_zero_ciphertext + `inner` mul_scalar_mac + add_scalar_inplace +
// rescale (one conv / dense output with `inner` taps); op 2: a zero-pad border
// cell (encode_const(0) at the top, encrypt with a seed, mod_switch to `level`).
int ref_time_layer_op(void* e, void* k, int op, size_t level, size_t count, size_t inner, unsigned threads,
                      double* secs) {
    return guard([&] {
        const CkksEngine& eng = static_cast<RefEngine*>(e)->eng;
        const RingContext& ctx = eng.ring();
        const KeySet* ks = static_cast<KeySet*>(k);
        const double sc = eng.params().scale;
        std::vector<Ciphertext> xs(op == 2 ? 0 : count);
        for (size_t i = 0; i < xs.size(); ++i) {
            xs[i].c0 = sample_poly(ctx, SampleKind::Uniform, {.level = level}, 2000 + 2 * i);
            xs[i].c1 = sample_poly(ctx, SampleKind::Uniform, {.level = level}, 2001 + 2 * i);
            xs[i].level = static_cast<u32>(level);
            xs[i].scale = sc;
        }
        const PolyActivation act = relu_default_surrogate();
        const CkksEngine::ScalarPlain sp = eng.make_scalar_plain(0.125, sc, level);
        std::vector<Ciphertext> out(count);
        auto t0 = std::chrono::steady_clock::now();
        parallel_for(count, threads, [&](std::size_t b, std::size_t en) {
            for (std::size_t i = b; i < en; ++i) {
                if (op == 0) {
                    out[i] = eval_encrypted(act, xs[i], eng, ks->eval);
                } else if (op == 1) {
                    Ciphertext acc = eng.make_zero_ciphertext(level, sc * sp.scale);
                    for (size_t m = 0; m < inner; ++m) eng.mul_scalar_mac(acc, xs[i], sp);
                    eng.add_scalar_inplace(acc, 0.25);
                    out[i] = eng.rescale(acc);
                } else {
                    EncodedPlaintext zero = eng.encode_const(0.0, sc, eng.top_level());
                    Ciphertext ct = eng.encrypt(ks->public_key, zero, CkksEngine::derive_seed(77, 0xbad0 + i));
                    out[i] = eng.mod_switch(ct, level);
                }
            }
        });
        *secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

// ---- ckks_serialize.hpp (blob v1): the reference's own save_* / load_*
// Writes the blob into `buf` (cap bytes); *len = blob size (buf may be null
// to query it).
static int blob_out(const std::string& b, uint8_t* buf, size_t cap, size_t* len) {
    *len = b.size();
    if (buf) {
        if (cap < b.size()) throw std::invalid_argument("ref: blob buffer too small");
        std::memcpy(buf, b.data(), b.size());
    }
    return 0;
}

// kind 1 secret, 2 public, 3 evaluation (BlobKind, ckks_serialize.hpp:17-22)
int ref_save_key(void* e, void* k, int kind, uint8_t* buf, size_t cap, size_t* len) {
    return guard([&] {
        const CkksEngine& eng = static_cast<RefEngine*>(e)->eng;
        KeySet* ks = static_cast<KeySet*>(k);
        std::ostringstream os;
        if (kind == 1) save_secret_key(os, eng.params(), ks->secret);
        else if (kind == 2) save_public_key(os, eng.params(), ks->public_key);
        else save_evaluation_key(os, eng.params(), ks->eval);
        blob_out(os.str(), buf, cap, len);
    });
}

int ref_save_ciphertext(void* e, const uint64_t* ct, size_t level, double scale, uint8_t* buf, size_t cap, size_t* len) {
    return guard([&] {
        const CkksEngine& eng = static_cast<RefEngine*>(e)->eng;
        std::ostringstream os;
        save_ciphertext(os, eng.params(), ct_from(eng, ct, level, scale));
        blob_out(os.str(), buf, cap, len);
    });
}

// load_ciphertext (ckks_serialize.hpp:133-141): words [2][level+1][n] out
int ref_load_ciphertext(const uint8_t* blob, size_t len, uint64_t* out, size_t cap_words, uint32_t* level,
                        double* scale) {
    return guard([&] {
        std::istringstream is(std::string(reinterpret_cast<const char*>(blob), len));
        auto [p, ct] = load_ciphertext(is);
        const std::size_t n = p.ring.n, words = 2 * (ct.level + 1) * n;
        if (cap_words < words) throw std::invalid_argument("ref: output too small");
        poly_to(ct.c0, out);
        poly_to(ct.c1, out + (ct.level + 1) * n);
        *level = ct.level;
        *scale = ct.scale;
    });
}

// load_secret_key / load_public_key / load_evaluation_key by kind; returns
// the error text of a rejected blob through ref_last_error()
int ref_load_key_check(const uint8_t* blob, size_t len, int kind) {
    return guard([&] {
        std::istringstream is(std::string(reinterpret_cast<const char*>(blob), len));
        if (kind == 1) (void)load_secret_key(is);
        else if (kind == 2) (void)load_public_key(is);
        else (void)load_evaluation_key(is);
    });
}

}  // extern "C"
