// Host-side CKKS numerics (see host_ckks.hpp). Compiled with the same
// floating-point contract as the reference's Release build (g++ -O3, no
// -march, so no FMA contraction) to keep libm/long-double results identical.
#include "host_ckks.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <stdexcept>

namespace hecnn_b200 {

u64 splitmix64(u64 x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

u64 HostRng::below(u64 bound) {
    if (bound == 0) throw std::invalid_argument("Rng::below: zero bound");
    const u64 top = std::numeric_limits<u64>::max();
    const u64 accept = top - (top - bound + 1) % bound;
    for (;;) {
        u64 r = next();
        if (r <= accept) return r % bound;
    }
}

// Box-Muller pair; the sine half is kept for the next call (common.hpp:191-204).
double HostRng::gaussian() {
    if (cached_valid_) {
        cached_valid_ = false;
        return cached_;
    }
    double u1 = uniform01();
    if (u1 < 1e-300) u1 = 1e-300;
    double u2 = uniform01();
    double radius = std::sqrt(-2.0 * std::log(u1));
    constexpr double tau = 6.283185307179586476925286766559;
    cached_ = radius * std::sin(tau * u2);
    cached_valid_ = true;
    return radius * std::cos(tau * u2);
}

std::vector<long long> sample_ternary(std::size_t n, double density, u64 seed) {
    if (density < 0.0 || density > 1.0) throw std::invalid_argument("sample_poly: ternary density out of range");
    HostRng rng(seed);
    std::vector<long long> c(n);
    for (auto& v : c) {
        double u = rng.uniform01();
        v = u < density / 2 ? 1 : (u < density ? -1 : 0);
    }
    return c;
}

std::vector<long long> sample_gaussian(std::size_t n, double sigma, u64 seed) {
    if (!(sigma > 0.0)) throw std::invalid_argument("sample_poly: gaussian requires sigma > 0");
    HostRng rng(seed);
    const long long bound = std::llround(6.0 * sigma);
    std::vector<long long> c(n);
    for (auto& v : c) {
        long long z = std::llround(rng.gaussian() * sigma);
        v = std::clamp(z, -bound, bound);
    }
    return c;
}

std::vector<u64> sample_uniform(const RingTables& R, std::size_t level, u64 seed) {
    HostRng rng(seed);
    std::vector<u64> out((level + 1) * R.n);
    for (std::size_t i = 0; i <= level; ++i)
        for (std::size_t j = 0; j < R.n; ++j) out[i * R.n + j] = rng.below(R.primes[i]);
    return out;
}

Encoder::Encoder(const RingTables& R, double) : R_(R) {
    const std::size_t n = R.n;
    twiddle_.resize(n);
    twist_.resize(n);
    const long double pi = 3.14159265358979323846264338327950288L;
    for (std::size_t k = 0; k < n; ++k) {
        long double t = 2.0L * pi * static_cast<long double>(k) / static_cast<long double>(n);
        twiddle_[k] = {static_cast<double>(std::cos(t)), static_cast<double>(std::sin(t))};
        long double u = pi * static_cast<long double>(k) / static_cast<long double>(n);
        twist_[k] = {static_cast<double>(std::cos(u)), static_cast<double>(std::sin(u))};
    }
}

void Encoder::check_encode(std::size_t len, double maxval, double scale, std::size_t level) const {
    if (len > R_.n / 2) throw std::invalid_argument("encode: vector longer than slot count");
    if (!(scale > 1.0)) throw std::invalid_argument("encode: scale must be > 1");
    if (level >= R_.limbs) throw std::invalid_argument("encode: level out of range");
    double bits = std::log2(scale) + std::log2(maxval + 1.0) + 2.0;
    if (bits >= R_.log2_mod[level] - 1.0)
        throw std::invalid_argument("encode: scaled coefficients overflow the active modulus");
}

// Radix-2 in-place FFT with the reference's exact operation order
// (bit-reversal permutation, then butterflies with e^{+-2 pi i k / n}).
void Encoder::fft(std::vector<std::complex<double>>& a, bool invert) const {
    const std::size_t n = a.size();
    for (std::size_t i = 1, j = 0; i < n; ++i) {
        std::size_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) std::swap(a[i], a[j]);
    }
    for (std::size_t len = 2; len <= n; len <<= 1) {
        const std::size_t step = n / len, half = len / 2;
        for (std::size_t i = 0; i < n; i += len)
            for (std::size_t j = 0; j < half; ++j) {
                std::complex<double> w = twiddle_[step * j];
                if (invert) w = std::conj(w);
                std::complex<double> u = a[i + j];
                std::complex<double> v = a[i + j + half] * w;
                a[i + j] = u + v;
                a[i + j + half] = u - v;
            }
    }
    if (invert) {
        const double inv_n = 1.0 / static_cast<double>(n);
        for (auto& x : a) x *= inv_n;
    }
}

std::vector<u64> Encoder::residues_of_rounded(long double v, std::size_t level) const {
    std::vector<u64> out(level + 1);
    if (v >= -9.2e18L && v <= 9.2e18L) {
        long long iv = static_cast<long long>(v);
        for (std::size_t i = 0; i <= level; ++i) out[i] = R_.mods[i].from_signed(iv);
        return out;
    }
    for (std::size_t i = 0; i <= level; ++i) {
        long double q = static_cast<long double>(R_.primes[i]);
        long double r = std::fmod(v, q);
        if (r < 0) r += q;
        out[i] = static_cast<u64>(r);
    }
    return out;
}

std::vector<u64> Encoder::scalar_residues(double c, double scale, std::size_t level) const {
    check_encode(1, std::abs(c), scale, level);
    return residues_of_rounded(roundl(static_cast<long double>(c) * static_cast<long double>(scale)), level);
}

void Encoder::encode_real(const double* values, std::size_t len, double scale, std::size_t level,
                          EncodedCoeffs& out) const {
    double maxval = 0.0;
    for (std::size_t i = 0; i < len; ++i) maxval = std::max(maxval, std::abs(std::complex<double>{values[i], 0.0}));
    check_encode(len, maxval, scale, level);
    const std::size_t n = R_.n;
    std::vector<std::complex<double>> v(n, {0.0, 0.0});
    for (std::size_t j = 0; j < len; ++j) {
        std::complex<double> z{values[j], 0.0};
        v[j] = z;
        v[n - 1 - j] = std::conj(z);
    }
    fft(v, true);
    std::vector<long double> rounded(n);
    bool small = true;
    for (std::size_t k = 0; k < n; ++k) {
        std::complex<double> u = v[k] * std::conj(twist_[k]);
        long double c = static_cast<long double>(u.real()) * static_cast<long double>(scale);
        rounded[k] = roundl(c);
        if (!(rounded[k] >= -9.2e18L && rounded[k] <= 9.2e18L)) small = false;
    }
    out.small = small;
    if (small) {
        out.coeffs.resize(n);
        for (std::size_t k = 0; k < n; ++k) out.coeffs[k] = static_cast<long long>(rounded[k]);
        out.residues.clear();
    } else {
        out.coeffs.clear();
        out.residues.assign((level + 1) * n, 0);
        for (std::size_t k = 0; k < n; ++k) {
            std::vector<u64> r = residues_of_rounded(rounded[k], level);
            for (std::size_t i = 0; i <= level; ++i) out.residues[i * n + k] = r[i];
        }
    }
}

// reconstruct_centered (ring.hpp:509-527) of coefficient k.
long double Encoder::centred_coeff(const u64* poly, std::size_t level, std::size_t k) const {
    const std::size_t W = R_.crt_words;
    const u64* Q = R_.modulus.data() + level * W;
    std::vector<u64> acc(W + 1, 0);
    for (std::size_t i = 0; i <= level; ++i) {
        const u64* pinv = &R_.punct_inv[(level * R_.limbs + i) * 2];
        u64 w = R_.mods[i].mul(poly[i * R_.n + k], pinv[0]);
        const u64* P = &R_.punct[(level * R_.limbs + i) * W];
        u64 carry = 0;
        for (std::size_t t = 0; t < W; ++t) {
            u128 s = static_cast<u128>(P[t]) * w + acc[t] + carry;
            acc[t] = static_cast<u64>(s);
            carry = static_cast<u64>(s >> 64);
        }
        acc[W] += carry;
    }
    auto cmp = [&](const std::vector<u64>& a, const u64* b) {
        for (std::size_t t = W + 1; t-- > 0;) {
            u64 bt = t < W ? b[t] : 0;
            if (a[t] != bt) return a[t] < bt ? -1 : 1;
        }
        return 0;
    };
    auto sub = [&](std::vector<u64>& a, const u64* b) {
        u64 borrow = 0;
        for (std::size_t t = 0; t <= W; ++t) {
            u64 bt = t < W ? b[t] : 0;
            u128 d = static_cast<u128>(a[t]) - bt - borrow;
            a[t] = static_cast<u64>(d);
            borrow = (d >> 64) ? 1 : 0;
        }
    };
    while (cmp(acc, Q) >= 0) sub(acc, Q);
    std::vector<u64> twice(W + 1, 0);
    u64 c = 0;
    for (std::size_t t = 0; t <= W; ++t) {
        twice[t] = (acc[t] << 1) | c;
        c = acc[t] >> 63;
    }
    auto to_ld = [&](const std::vector<u64>& a) {
        std::size_t top = a.size();
        while (top > 0 && a[top - 1] == 0) --top;
        long double v = 0.0L;
        for (std::size_t t = top; t-- > 0;) v = v * 18446744073709551616.0L + static_cast<long double>(a[t]);
        return v;
    };
    if (cmp(twice, Q) > 0) {
        std::vector<u64> neg(W + 1, 0);
        std::copy(Q, Q + W, neg.begin());
        sub(neg, acc.data());
        return -to_ld(neg);
    }
    return to_ld(acc);
}

void Encoder::decode_real(const u64* poly, std::size_t level, double scale, double* out, std::size_t count) const {
    if (!(scale > 0.0) || !std::isfinite(scale)) throw std::invalid_argument("decode: invalid scale");
    const std::size_t n = R_.n;
    std::vector<std::complex<double>> u(n);
    for (std::size_t k = 0; k < n; ++k) {
        double c = static_cast<double>(centred_coeff(poly, level, k));
        u[k] = twist_[k] * c;
    }
    fft(u, false);
    for (std::size_t j = 0; j < count; ++j) out[j] = (u[j] / scale).real();
}

}  // namespace hecnn_b200
