// hecnn_b200/hecnn.hpp -- C++ drop-in for the reference's encrypted-CNN API.
//
// Mirrors the names, value semantics and exceptions of the reference library
// (proj/include/hecnn: ckks.hpp, tensor.hpp, activation.hpp, model.hpp,
// layers.hpp) on top of the C-ABI in hecnn_b200.h. A reference call site
// switches by replacing its hecnn includes with this header and linking
// libhecnn_b200.so; see INTEGRATION.md. Ciphertexts stay host values here
// (RingPoly owns vector<vector<u64>> exactly as ring.hpp:239-253) and every
// operation uploads, runs on the B200 and downloads -- the drop-in shim. The
// throughput path is forward_encrypted(), which uploads the tensor once and
// keeps every intermediate in HBM.
#pragma once

#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <istream>
#include <ostream>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "hecnn_b200.h"

namespace hecnn {

using u32 = std::uint32_t;
using u64 = std::uint64_t;

namespace b200_detail {
inline u64 splitmix64(u64 x) {  // common.hpp:164-169
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
inline u64 derive_seed(u64 seed, u64 domain) { return splitmix64(seed ^ splitmix64(domain)); }
inline void check(int st) {
    if (st == HECNN_OK) return;
    if (st == HECNN_EINVAL) throw std::invalid_argument(hecnn_last_error());
    throw std::runtime_error(hecnn_last_error());
}
struct TensorHandle {
    hecnn_tensor* h = nullptr;
    explicit TensorHandle(hecnn_tensor* t) : h(t) {}
    ~TensorHandle() { if (h) hecnn_tensor_destroy(h); }
    TensorHandle(const TensorHandle&) = delete;
    TensorHandle& operator=(const TensorHandle&) = delete;
};
}  // namespace b200_detail

// ---- ring.hpp ----------------------------------------------------------------
enum class Rep : std::uint8_t { Coeff = 0, Ntt = 1 };

struct RingParams {  // ring.hpp:20-55
    std::size_t n = 0;
    std::vector<u64> primes;
    static RingParams create(std::size_t n, const std::vector<int>& prime_bits) {
        RingParams p;
        p.n = n;
        p.primes.resize(prime_bits.size());
        b200_detail::check(hecnn_find_chain(n, prime_bits.data(), prime_bits.size(), p.primes.data()));
        return p;
    }
    std::size_t chain_length() const { return primes.size(); }
    std::size_t top_level() const { return primes.size() - 1; }
};

struct RingPoly {  // ring.hpp:239-253
    u32 level = 0;
    Rep rep = Rep::Coeff;
    std::vector<std::vector<u64>> rns;
    std::size_t degree() const { return rns.empty() ? 0 : rns[0].size(); }
};

// ---- ckks.hpp ------------------------------------------------------------------
struct CkksParams {  // ckks.hpp:21-34
    RingParams ring;
    double scale = 0.0;
    double sigma = 3.2;
    bool degenerate_noise = false;
    std::size_t slot_count() const { return ring.n / 2; }
};

using PlaintextVector = std::vector<std::complex<double>>;

struct EncodedPlaintext {
    RingPoly poly;
    double scale = 0.0;
    bool is_constant = false;
};

struct Ciphertext {  // ckks.hpp:68-72
    RingPoly c0, c1;
    double scale = 0.0;
    u32 level = 0;
};

// Keys live on the device inside the engine's context; the structs carry the
// exported words so they can be saved or compared like the reference's.
struct SecretKey { RingPoly s; };
struct PublicKey { RingPoly b, a; };
struct EvaluationKey {
    u32 base_bits = 20;
    std::vector<std::pair<RingPoly, RingPoly>> pairs;
};
struct KeySet {
    SecretKey secret;
    PublicKey public_key;
    EvaluationKey eval;
};

class CkksEngine {  // ckks.hpp:77-636 (device-backed)
public:
    explicit CkksEngine(CkksParams params, int device = 0) : par_(std::move(params)) {
        b200_detail::check(hecnn_context_create(par_.ring.n, par_.ring.primes.data(), par_.ring.primes.size(),
                                                par_.scale, par_.sigma, par_.degenerate_noise ? 1 : 0, device, &ctx_));
    }
    ~CkksEngine() { if (ctx_) hecnn_context_destroy(ctx_); }
    CkksEngine(const CkksEngine&) = delete;
    CkksEngine& operator=(const CkksEngine&) = delete;

    const CkksParams& params() const { return par_; }
    std::size_t slot_count() const { return par_.slot_count(); }
    std::size_t top_level() const { return par_.ring.top_level(); }
    std::size_t depth_budget() const { return par_.ring.chain_length() - 1; }
    std::size_t relin_digits(std::size_t level) const {
        std::size_t d = 0;
        b200_detail::check(hecnn_relin_digits(ctx_, level, &d));
        return d;
    }
    hecnn_context* context() const { return ctx_; }

    // keygen (ckks.hpp:200-236): keys generated and kept on the device.
    KeySet keygen(u64 seed) const {
        b200_detail::check(hecnn_keygen(ctx_, seed));
        KeySet ks;
        const std::size_t L = top_level() + 1, n = par_.ring.n;
        std::vector<u64> s(L * n), b(L * n), a(L * n);
        b200_detail::check(hecnn_export_secret_key(ctx_, s.data()));
        b200_detail::check(hecnn_export_public_key(ctx_, b.data(), a.data()));
        ks.secret.s = to_poly(s.data(), top_level(), Rep::Coeff);
        ks.public_key.b = to_poly(b.data(), top_level(), Rep::Ntt);
        ks.public_key.a = to_poly(a.data(), top_level(), Rep::Ntt);
        std::size_t D = 0;
        b200_detail::check(hecnn_eval_key_digits(ctx_, &D));
        std::vector<u64> evk(D * 2 * L * n);
        b200_detail::check(hecnn_export_eval_key(ctx_, evk.data()));
        for (std::size_t t = 0; t < D; ++t)
            ks.eval.pairs.emplace_back(to_poly(&evk[(2 * t) * L * n], top_level(), Rep::Ntt),
                                       to_poly(&evk[(2 * t + 1) * L * n], top_level(), Rep::Ntt));
        return ks;
    }

    // encode_real / decode (ckks.hpp:105-154), host numerics bit-identical to the reference
    EncodedPlaintext encode_real(const std::vector<double>& v, double scale, std::size_t level) const {
        std::vector<u64> out((level + 1) * par_.ring.n);
        b200_detail::check(hecnn_host_encode_real(par_.ring.n, par_.ring.primes.data(), par_.ring.primes.size(),
                                                  v.data(), v.size(), scale, level, out.data()));
        return EncodedPlaintext{to_poly(out.data(), level, Rep::Coeff), scale, false};
    }
    PlaintextVector decode(const EncodedPlaintext& m) const {
        std::vector<u64> flat = from_poly(m.poly);
        std::vector<double> re(slot_count());
        b200_detail::check(hecnn_host_decode_real(par_.ring.n, par_.ring.primes.data(), par_.ring.primes.size(),
                                                  flat.data(), m.poly.level, m.scale, re.data(), re.size()));
        PlaintextVector out(re.size());
        for (std::size_t i = 0; i < re.size(); ++i) out[i] = {re[i], 0.0};
        return out;
    }

    // encrypt(pk, m, seed) (ckks.hpp:249-270): host randomness from `seed`
    // (make_encryption_randomness), device encryption with this engine's pk.
    Ciphertext encrypt(const PublicKey&, const EncodedPlaintext& m, u64 seed) const {
        if (m.poly.level != top_level()) throw std::invalid_argument("encrypt: plaintext must be at top level");
        if (m.poly.rep != Rep::Coeff) throw std::invalid_argument("encrypt: plaintext must be in coefficient domain");
        const std::size_t n = par_.ring.n;
        std::vector<std::int64_t> r(n), e0(n), e1(n);
        b200_detail::check(hecnn_host_encryption_randomness(n, par_.sigma, par_.degenerate_noise ? 1 : 0, seed,
                                                            r.data(), e0.data(), e1.data()));
        std::vector<u64> flat = from_poly(m.poly);
        hecnn_tensor* t = nullptr;
        b200_detail::check(hecnn_encrypt_raw(ctx_, flat.data(), r.data(), e0.data(), e1.data(), 1, m.scale, &t));
        b200_detail::TensorHandle h(t);
        return download(t)[0];
    }

    EncodedPlaintext decrypt(const SecretKey&, const Ciphertext& ct) const {
        b200_detail::TensorHandle h(upload({ct}));
        std::vector<u64> out((ct.level + 1) * par_.ring.n);
        b200_detail::check(hecnn_decrypt_raw(ctx_, h.h, out.data()));
        return EncodedPlaintext{to_poly(out.data(), ct.level, Rep::Coeff), ct.scale, false};
    }

    Ciphertext add(const Ciphertext& x, const Ciphertext& y) const { return binary(hecnn_ct_add, x, y); }
    Ciphertext sub(const Ciphertext& x, const Ciphertext& y) const { return binary(hecnn_ct_sub, x, y); }
    Ciphertext mul(const Ciphertext& x, const Ciphertext& y, const EvaluationKey&) const {
        return binary(hecnn_ct_mul, x, y);
    }
    Ciphertext square(const Ciphertext& x, const EvaluationKey&) const {
        b200_detail::TensorHandle a(upload({x}));
        hecnn_tensor* o = nullptr;
        b200_detail::check(hecnn_ct_square(ctx_, a.h, &o));
        b200_detail::TensorHandle r(o);
        return download(o)[0];
    }
    Ciphertext rescale(const Ciphertext& x) const {
        b200_detail::TensorHandle a(upload({x}));
        hecnn_tensor* o = nullptr;
        b200_detail::check(hecnn_ct_rescale(ctx_, a.h, &o));
        b200_detail::TensorHandle r(o);
        return download(o)[0];
    }
    Ciphertext mod_switch(const Ciphertext& x, std::size_t to_level) const {
        b200_detail::TensorHandle a(upload({x}));
        hecnn_tensor* o = nullptr;
        b200_detail::check(hecnn_ct_mod_switch(ctx_, a.h, static_cast<u32>(to_level), &o));
        b200_detail::TensorHandle r(o);
        return download(o)[0];
    }
    // mul_plain(x, encode_const(c, scale, x.level)) (ckks.hpp:395-398)
    Ciphertext mul_const(const Ciphertext& x, double c, double scale) const {
        b200_detail::TensorHandle a(upload({x}));
        hecnn_tensor* o = nullptr;
        b200_detail::check(hecnn_ct_mul_const(ctx_, a.h, c, scale, &o));
        b200_detail::TensorHandle r(o);
        return download(o)[0];
    }

    // ---- plaintext operands and the scalar fast path (ckks.hpp:132-140, 305-311, 372-472)
    EncodedPlaintext encode_const(double c, double scale, std::size_t level) const {
        std::vector<u64> r(level + 1);
        b200_detail::check(hecnn_make_scalar_plain(ctx_, c, scale, level, r.data()));
        RingPoly p;
        p.level = static_cast<u32>(level);
        p.rns.assign(level + 1, std::vector<u64>(par_.ring.n, 0));
        for (std::size_t i = 0; i <= level; ++i) p.rns[i][0] = r[i];
        return EncodedPlaintext{std::move(p), scale, true};
    }
    Ciphertext add_plain(const Ciphertext& x, const EncodedPlaintext& m) const {
        b200_detail::TensorHandle a(upload({x}));
        std::vector<u64> flat = from_poly(m.poly);
        hecnn_tensor* o = nullptr;
        b200_detail::check(hecnn_ct_add_plain(ctx_, a.h, flat.data(), m.poly.level, m.scale, &o));
        b200_detail::TensorHandle r(o);
        return download(o)[0];
    }
    Ciphertext mul_plain_raw(const Ciphertext& x, const EncodedPlaintext& m) const { return plain_mul(x, m, 0); }
    Ciphertext mul_plain(const Ciphertext& x, const EncodedPlaintext& m) const { return plain_mul(x, m, 1); }

    struct ScalarPlain {  // ckks.hpp:400-405
        std::vector<u64> residues, residues_shoup;
        double scale = 0.0;
        u32 level = 0;
    };
    ScalarPlain make_scalar_plain(double c, double scale, std::size_t level) const {
        ScalarPlain sp;
        sp.residues.resize(level + 1);
        b200_detail::check(hecnn_make_scalar_plain(ctx_, c, scale, level, sp.residues.data()));
        for (std::size_t i = 0; i <= level; ++i)
            sp.residues_shoup.push_back(static_cast<u64>((static_cast<unsigned __int128>(sp.residues[i]) << 64) /
                                                         par_.ring.primes[i]));
        sp.scale = scale;
        sp.level = static_cast<u32>(level);
        return sp;
    }
    Ciphertext make_zero_ciphertext(std::size_t level, double scale) const {
        Ciphertext ct;
        ct.c0.level = ct.c1.level = static_cast<u32>(level);
        ct.c0.rns.assign(level + 1, std::vector<u64>(par_.ring.n, 0));
        ct.c1.rns = ct.c0.rns;
        ct.scale = scale;
        ct.level = static_cast<u32>(level);
        return ct;
    }
    void add_inplace(Ciphertext& acc, const Ciphertext& x) const {
        b200_detail::TensorHandle a(upload({acc})), b(upload({x}));
        b200_detail::check(hecnn_ct_add_inplace(ctx_, a.h, b.h));
        acc = download(a.h)[0];
    }
    // acc += x * sp; on device tensors prefer hecnn_ct_scalar_mac over a whole
    // tensor of cells (one launch) -- this per-ciphertext form round-trips
    void mul_scalar_mac(Ciphertext& acc, const Ciphertext& x, const ScalarPlain& sp) const {
        b200_detail::TensorHandle a(upload({acc})), b(upload({x}));
        b200_detail::check(hecnn_ct_scalar_mac(ctx_, a.h, b.h, sp.residues.data(), 1, sp.scale, sp.level));
        acc = download(a.h)[0];
    }
    void add_scalar_inplace(Ciphertext& ct, double c) const {
        b200_detail::TensorHandle a(upload({ct}));
        b200_detail::check(hecnn_ct_add_scalar(ctx_, a.h, c));
        ct = download(a.h)[0];
    }
    static u64 derive_seed(u64 seed, u64 domain) {  // ckks.hpp:507
        return b200_detail::derive_seed(seed, domain);
    }

    // ---- host <-> device conversion of value-semantic ciphertexts
    hecnn_tensor* upload(const std::vector<Ciphertext>& cts) const {
        if (cts.empty()) throw std::invalid_argument("upload: empty ciphertext list");
        const u32 level = cts.front().level;
        const std::size_t n = par_.ring.n, cw = 2 * (level + 1) * n;
        std::vector<u64> words(cts.size() * cw);
        for (std::size_t c = 0; c < cts.size(); ++c) {
            if (cts[c].level != level || cts[c].scale != cts.front().scale)
                throw std::runtime_error("TensorEncrypted: cells disagree on scale/level");
            for (std::size_t i = 0; i <= level; ++i) {
                std::copy(cts[c].c0.rns[i].begin(), cts[c].c0.rns[i].end(), &words[c * cw + i * n]);
                std::copy(cts[c].c1.rns[i].begin(), cts[c].c1.rns[i].end(), &words[c * cw + (level + 1 + i) * n]);
            }
        }
        hecnn_tensor* t = nullptr;
        b200_detail::check(hecnn_tensor_create(ctx_, cts.size(), level, cts.front().scale, &t));
        b200_detail::TensorHandle guard(t);
        b200_detail::check(hecnn_tensor_upload(ctx_, t, words.data()));
        guard.h = nullptr;
        return t;
    }

    std::vector<Ciphertext> download(const hecnn_tensor* t) const {
        std::size_t cells = 0;
        u32 level = 0;
        double scale = 0;
        b200_detail::check(hecnn_tensor_info(t, &cells, &level, &scale));
        const std::size_t n = par_.ring.n, cw = 2 * (level + 1) * n;
        std::vector<u64> words(cells * cw);
        b200_detail::check(hecnn_tensor_download(ctx_, t, words.data()));
        std::vector<Ciphertext> out(cells);
        for (std::size_t c = 0; c < cells; ++c) {
            out[c].c0 = to_poly(&words[c * cw], level, Rep::Coeff);
            out[c].c1 = to_poly(&words[c * cw + (level + 1) * n], level, Rep::Coeff);
            out[c].scale = scale;
            out[c].level = level;
        }
        return out;
    }

private:
    Ciphertext plain_mul(const Ciphertext& x, const EncodedPlaintext& m, int rescale) const {
        b200_detail::TensorHandle a(upload({x}));
        std::vector<u64> flat = from_poly(m.poly);
        hecnn_tensor* o = nullptr;
        b200_detail::check(hecnn_ct_mul_plain(ctx_, a.h, flat.data(), m.poly.level, m.scale, m.is_constant ? 1 : 0,
                                              rescale, &o));
        b200_detail::TensorHandle r(o);
        return download(o)[0];
    }
    template <class F>
    Ciphertext binary(F fn, const Ciphertext& x, const Ciphertext& y) const {
        b200_detail::TensorHandle a(upload({x})), b(upload({y}));
        hecnn_tensor* o = nullptr;
        b200_detail::check(fn(ctx_, a.h, b.h, &o));
        b200_detail::TensorHandle r(o);
        return download(o)[0];
    }
    RingPoly to_poly(const u64* src, std::size_t level, Rep rep) const {
        RingPoly p;
        p.level = static_cast<u32>(level);
        p.rep = rep;
        const std::size_t n = par_.ring.n;
        p.rns.resize(level + 1);
        for (std::size_t i = 0; i <= level; ++i) p.rns[i].assign(src + i * n, src + (i + 1) * n);
        return p;
    }
    std::vector<u64> from_poly(const RingPoly& p) const {
        std::vector<u64> flat;
        for (const auto& row : p.rns) flat.insert(flat.end(), row.begin(), row.end());
        return flat;
    }

    CkksParams par_;
    hecnn_context* ctx_ = nullptr;
};

// ---- ckks_serialize.hpp (CKKS blob v1) -----------------------------------------
// Same byte layout as the reference and as the device codec behind
// hecnn_blob_* (include/hecnn_b200.h): blobs written here load in the
// reference and vice versa.
enum class BlobKind : std::uint16_t { SecretKey = 1, PublicKey = 2, EvaluationKey = 3, Ciphertext = 4 };

namespace b200_detail {
template <class T>
void put(std::ostream& os, T v) {
    char b[sizeof(T)];
    std::memcpy(b, &v, sizeof(T));
    os.write(b, sizeof(T));
}
template <class T>
T get(std::istream& is) {
    char b[sizeof(T)];
    is.read(b, sizeof(T));
    if (is.gcount() != static_cast<std::streamsize>(sizeof(T))) throw std::runtime_error("io: unexpected end of file");
    T v;
    std::memcpy(&v, b, sizeof(T));
    return v;
}
inline void put_header(std::ostream& os, BlobKind kind, const CkksParams& p) {
    os.write("CKKS", 4);
    put<std::uint16_t>(os, 1);
    put<std::uint16_t>(os, static_cast<std::uint16_t>(kind));
    put<std::uint32_t>(os, static_cast<std::uint32_t>(p.ring.n));
    put<std::uint16_t>(os, static_cast<std::uint16_t>(p.ring.primes.size()));
    for (u64 q : p.ring.primes) put<u64>(os, q);
    put<double>(os, p.scale);
    put<double>(os, p.sigma);
    put<std::uint8_t>(os, p.degenerate_noise ? 1 : 0);
}
inline CkksParams get_header(std::istream& is, BlobKind want) {
    char magic[4];
    is.read(magic, 4);
    if (is.gcount() != 4) throw std::runtime_error("io: unexpected end of file");
    if (std::memcmp(magic, "CKKS", 4) != 0) throw std::runtime_error("ckks blob: bad magic");
    if (get<std::uint16_t>(is) != 1) throw std::runtime_error("ckks blob: unsupported version");
    if (get<std::uint16_t>(is) != static_cast<std::uint16_t>(want)) throw std::runtime_error("ckks blob: wrong object kind");
    CkksParams p;
    p.ring.n = get<std::uint32_t>(is);
    p.ring.primes.resize(get<std::uint16_t>(is));
    for (u64& q : p.ring.primes) q = get<u64>(is);
    p.scale = get<double>(is);
    p.sigma = get<double>(is);
    p.degenerate_noise = get<std::uint8_t>(is) != 0;
    return p;
}
inline void put_poly(std::ostream& os, const RingPoly& r) {
    put<std::uint16_t>(os, static_cast<std::uint16_t>(r.level));
    put<std::uint8_t>(os, static_cast<std::uint8_t>(r.rep));
    for (const auto& row : r.rns) os.write(reinterpret_cast<const char*>(row.data()), static_cast<std::streamsize>(row.size() * 8));
}
inline RingPoly get_poly(std::istream& is, std::size_t n) {
    RingPoly r;
    r.level = get<std::uint16_t>(is);
    r.rep = static_cast<Rep>(get<std::uint8_t>(is));
    r.rns.assign(r.level + 1, std::vector<u64>(n));
    for (auto& row : r.rns) {
        is.read(reinterpret_cast<char*>(row.data()), static_cast<std::streamsize>(n * 8));
        if (is.gcount() != static_cast<std::streamsize>(n * 8)) throw std::runtime_error("io: unexpected end of file");
    }
    return r;
}
}  // namespace b200_detail

inline void save_secret_key(std::ostream& os, const CkksParams& p, const SecretKey& sk) {
    b200_detail::put_header(os, BlobKind::SecretKey, p);
    b200_detail::put_poly(os, sk.s);
}
inline std::pair<CkksParams, SecretKey> load_secret_key(std::istream& is) {
    CkksParams p = b200_detail::get_header(is, BlobKind::SecretKey);
    SecretKey sk{b200_detail::get_poly(is, p.ring.n)};
    return {std::move(p), std::move(sk)};
}
inline void save_public_key(std::ostream& os, const CkksParams& p, const PublicKey& pk) {
    b200_detail::put_header(os, BlobKind::PublicKey, p);
    b200_detail::put_poly(os, pk.b);
    b200_detail::put_poly(os, pk.a);
}
inline std::pair<CkksParams, PublicKey> load_public_key(std::istream& is) {
    CkksParams p = b200_detail::get_header(is, BlobKind::PublicKey);
    PublicKey pk;
    pk.b = b200_detail::get_poly(is, p.ring.n);
    pk.a = b200_detail::get_poly(is, p.ring.n);
    return {std::move(p), std::move(pk)};
}
inline void save_evaluation_key(std::ostream& os, const CkksParams& p, const EvaluationKey& evk) {
    b200_detail::put_header(os, BlobKind::EvaluationKey, p);
    b200_detail::put<std::uint16_t>(os, static_cast<std::uint16_t>(evk.base_bits));
    b200_detail::put<std::uint16_t>(os, static_cast<std::uint16_t>(evk.pairs.size()));
    for (const auto& pr : evk.pairs) {
        b200_detail::put_poly(os, pr.first);
        b200_detail::put_poly(os, pr.second);
    }
}
inline std::pair<CkksParams, EvaluationKey> load_evaluation_key(std::istream& is) {
    CkksParams p = b200_detail::get_header(is, BlobKind::EvaluationKey);
    EvaluationKey evk;
    evk.base_bits = b200_detail::get<std::uint16_t>(is);
    const std::size_t count = b200_detail::get<std::uint16_t>(is);
    for (std::size_t t = 0; t < count; ++t) {
        RingPoly b = b200_detail::get_poly(is, p.ring.n);
        evk.pairs.emplace_back(std::move(b), b200_detail::get_poly(is, p.ring.n));
    }
    return {std::move(p), std::move(evk)};
}
inline void save_ciphertext(std::ostream& os, const CkksParams& p, const Ciphertext& ct) {
    b200_detail::put_header(os, BlobKind::Ciphertext, p);
    b200_detail::put<double>(os, ct.scale);
    b200_detail::put<std::uint16_t>(os, static_cast<std::uint16_t>(ct.level));
    b200_detail::put_poly(os, ct.c0);
    b200_detail::put_poly(os, ct.c1);
}
inline std::pair<CkksParams, Ciphertext> load_ciphertext(std::istream& is) {
    CkksParams p = b200_detail::get_header(is, BlobKind::Ciphertext);
    Ciphertext ct;
    ct.scale = b200_detail::get<double>(is);
    ct.level = b200_detail::get<std::uint16_t>(is);
    ct.c0 = b200_detail::get_poly(is, p.ring.n);
    ct.c1 = b200_detail::get_poly(is, p.ring.n);
    return {std::move(p), std::move(ct)};
}
inline bool same_params(const CkksParams& a, const CkksParams& b) {
    return a.ring.n == b.ring.n && a.ring.primes == b.ring.primes && a.scale == b.scale && a.sigma == b.sigma &&
           a.degenerate_noise == b.degenerate_noise;
}

// ---- presets.hpp (built-ins, presets.hpp:33-49) ------------------------------------
inline CkksParams preset_params(const std::string& name, bool degenerate_noise = false) {
    struct Def { const char* name; std::size_t n; std::vector<int> bits; int log2_scale; };
    std::vector<int> large{60};
    large.insert(large.end(), 24, 40);
    const Def defs[] = {{"toy-n16", 16, {40, 21, 21, 21}, 20},
                        {"test-n4096-d4", 4096, {60, 40, 40, 40, 40}, 40},
                        {"nn-n4096-d8", 4096, {60, 40, 40, 40, 40, 40, 40, 40, 40}, 40},
                        {"net-n8192-d8", 8192, {60, 40, 40, 40, 40, 40, 40, 40, 40}, 40},
                        {"large-n16384-d24", 16384, large, 40}};
    for (const auto& d : defs)
        if (name == d.name) {
            CkksParams p;
            p.ring = RingParams::create(d.n, d.bits);
            p.scale = std::ldexp(1.0, d.log2_scale);
            p.degenerate_noise = degenerate_noise;
            return p;
        }
    throw std::invalid_argument("unknown parameter preset: " + name);
}

// ---- tensor.hpp -------------------------------------------------------------------
struct Shape {  // tensor.hpp:16-39
    bool flat = false;
    std::size_t h = 0, w = 0, c = 0, feat = 0;
    static Shape spatial(std::size_t h, std::size_t w, std::size_t c) { return {false, h, w, c, 0}; }
    static Shape flattened(std::size_t f) { return {true, 0, 0, 0, f}; }
    std::size_t positions() const { return flat ? feat : h * w * c; }
};

struct TensorPlain {
    Shape shape;
    std::size_t batch = 0;
    std::vector<double> data;  // [batch][position]
    double at(std::size_t b, std::size_t pos) const { return data[b * shape.positions() + pos]; }
};

struct TensorEncrypted {  // tensor.hpp:61-75
    Shape shape;
    std::size_t batch = 0;
    std::vector<Ciphertext> cells;
};

// encrypt_tensor (tensor.hpp:77-94); `threads` is accepted for signature parity
inline TensorEncrypted encrypt_tensor(const CkksEngine& eng, const PublicKey&, const TensorPlain& x, u64 seed,
                                      unsigned threads = 1) {
    (void)threads;
    hecnn_tensor* t = nullptr;
    b200_detail::check(hecnn_encrypt_tensor(eng.context(), x.data.data(), x.batch, x.shape.positions(), seed, &t));
    b200_detail::TensorHandle h(t);
    return TensorEncrypted{x.shape, x.batch, eng.download(t)};
}

// decrypt_tensor (tensor.hpp:96-106)
inline TensorPlain decrypt_tensor(const CkksEngine& eng, const SecretKey&, const TensorEncrypted& x,
                                  unsigned threads = 1) {
    (void)threads;
    b200_detail::TensorHandle h(eng.upload(x.cells));
    TensorPlain out{x.shape, x.batch, std::vector<double>(x.batch * x.cells.size())};
    b200_detail::check(hecnn_decrypt_tensor(eng.context(), h.h, x.batch, out.data.data()));
    return out;
}

// ---- activation.hpp / model.hpp --------------------------------------------------
struct PolyActivation {  // activation.hpp:24-45
    std::vector<double> coefficients;
    double interval_bound = 0.0;
    std::string source;
};
inline constexpr double kReluQuadCoeff = 0.000469841857369822;
inline PolyActivation relu_default_surrogate() {
    return PolyActivation{{0.0, 0.5, kReluQuadCoeff}, 3.0 / (8.0 * kReluQuadCoeff), "relu"};
}

struct LayerSpec {  // model.hpp:12-76
    enum class Kind { Conv2d, AvgPool2d, ZeroPad2d, Dense, Activation, Sigmoid };
    enum class Padding { Same, Valid };
    Kind kind = Kind::Conv2d;
    std::size_t filters = 0, kernel_h = 0, kernel_w = 0, stride = 1;
    Padding padding = Padding::Same;
    std::size_t pool = 0, pad = 0, units = 0;
    std::string surrogate;
    static LayerSpec conv2d(std::size_t f, std::size_t kh, std::size_t kw, std::size_t s = 1,
                            Padding p = Padding::Same) {
        LayerSpec l;
        l.kind = Kind::Conv2d;
        l.filters = f;
        l.kernel_h = kh;
        l.kernel_w = kw;
        l.stride = s;
        l.padding = p;
        return l;
    }
    static LayerSpec avg_pool2d(std::size_t p) { LayerSpec l; l.kind = Kind::AvgPool2d; l.pool = p; return l; }
    static LayerSpec zero_pad2d(std::size_t p) { LayerSpec l; l.kind = Kind::ZeroPad2d; l.pad = p; return l; }
    static LayerSpec dense(std::size_t u) { LayerSpec l; l.kind = Kind::Dense; l.units = u; return l; }
    static LayerSpec activation(std::string s) { LayerSpec l; l.kind = Kind::Activation; l.surrogate = std::move(s); return l; }
    static LayerSpec sigmoid() { LayerSpec l; l.kind = Kind::Sigmoid; return l; }
};

struct ModelSpec {  // model.hpp:78-97
    Shape input;
    std::vector<LayerSpec> layers;
    std::map<std::string, PolyActivation> activations;
    std::vector<std::vector<double>> weights, biases;
    void ensure_param_slots() {
        weights.resize(layers.size());
        biases.resize(layers.size());
    }
};

inline ModelSpec tiny_preset() {  // model.hpp:223-235
    ModelSpec m;
    m.input = Shape::spatial(8, 8, 3);
    m.activations["relu-poly2"] = relu_default_surrogate();
    m.layers = {LayerSpec::conv2d(4, 3, 3), LayerSpec::activation("relu-poly2"), LayerSpec::avg_pool2d(2),
                LayerSpec::dense(1)};
    m.ensure_param_slots();
    return m;
}

struct EvalKeys {  // layers.hpp:17-20
    PublicKey pk;
    EvaluationKey evk;
};

// forward_encrypted (layers.hpp:299-368): one upload, all layers in HBM, one download.
inline TensorEncrypted forward_encrypted(const ModelSpec& model, const TensorEncrypted& x, const CkksEngine& eng,
                                         const EvalKeys&, u64 seed = 1, unsigned threads = 1,
                                         std::vector<double>* layer_seconds = nullptr) {
    (void)threads;
    std::vector<std::string> names;
    std::vector<hecnn_activation_desc> acts;
    for (const auto& kv : model.activations) {
        names.push_back(kv.first);
        acts.push_back({kv.second.coefficients.data(), kv.second.coefficients.size(), kv.second.interval_bound});
    }
    std::vector<hecnn_layer_desc> layers;
    for (std::size_t i = 0; i < model.layers.size(); ++i) {
        const LayerSpec& l = model.layers[i];
        hecnn_layer_desc d{};
        d.kind = static_cast<int32_t>(l.kind);
        d.filters = static_cast<int32_t>(l.filters);
        d.kernel_h = static_cast<int32_t>(l.kernel_h);
        d.kernel_w = static_cast<int32_t>(l.kernel_w);
        d.stride = static_cast<int32_t>(l.stride);
        d.padding_valid = l.padding == LayerSpec::Padding::Valid;
        d.pool = static_cast<int32_t>(l.pool);
        d.pad = static_cast<int32_t>(l.pad);
        d.units = static_cast<int32_t>(l.units);
        d.activation = -1;
        for (std::size_t a = 0; a < names.size(); ++a)
            if (names[a] == l.surrogate) d.activation = static_cast<int32_t>(a);
        if (l.kind == LayerSpec::Kind::Activation && d.activation < 0)
            throw std::invalid_argument("model: activation layer references unregistered surrogate '" + l.surrogate + "'");
        if (i < model.weights.size() && !model.weights[i].empty()) {
            d.weights = model.weights[i].data();
            d.n_weights = model.weights[i].size();
        }
        if (i < model.biases.size() && !model.biases[i].empty()) {
            d.biases = model.biases[i].data();
            d.n_biases = model.biases[i].size();
        }
        layers.push_back(d);
    }
    hecnn_model_desc desc{model.input.flat ? 1 : 0, model.input.h, model.input.w, model.input.c, model.input.feat,
                          layers.data(), layers.size(), acts.data(), acts.size()};
    hecnn_model* m = nullptr;
    b200_detail::check(hecnn_model_create(eng.context(), &desc, &m));
    struct ModelGuard { hecnn_model* m; ~ModelGuard() { hecnn_model_destroy(m); } } mg{m};
    b200_detail::TensorHandle in(eng.upload(x.cells));
    b200_detail::check(hecnn_tensor_set_shape(in.h, x.shape.flat ? 1 : 0, x.shape.flat ? x.shape.feat : x.shape.h,
                                              x.shape.w, x.shape.c, x.batch));
    std::vector<double> secs(model.layers.size() + 1);
    hecnn_tensor* out = nullptr;
    b200_detail::check(hecnn_forward_encrypted(eng.context(), m, in.h, seed, &out, secs.data()));
    b200_detail::TensorHandle oh(out);
    if (layer_seconds) layer_seconds->assign(secs.begin(), secs.begin() + model.layers.size());
    int flat = 0;
    std::size_t h = 0, w = 0, c = 0, batch = 0;
    b200_detail::check(hecnn_tensor_shape(out, &flat, &h, &w, &c, &batch));
    TensorEncrypted res;
    res.shape = flat ? Shape::flattened(h) : Shape::spatial(h, w, c);
    res.batch = x.batch;
    res.cells = eng.download(out);
    return res;
}

}  // namespace hecnn
