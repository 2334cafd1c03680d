// Host-side ring setup (see ring_host.hpp). One-time work per context.
#include "ring_host.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>

namespace hecnn_b200 {

HostMod::HostMod(u64 modulus) : q(modulus) {
    if (q < 2 || q >= (u64(1) << 61)) throw std::invalid_argument("Modulus: need 2 <= q < 2^61");
    u128 r = (~static_cast<u128>(0)) / q;
    ratio_lo = static_cast<u64>(r);
    ratio_hi = static_cast<u64>(r >> 64);
}

u64 HostMod::mul(u64 a, u64 b) const { return static_cast<u64>((static_cast<u128>(a) * b) % q); }

u64 HostMod::pow(u64 base, u64 e) const {
    u64 acc = 1 % q, b = base % q;
    for (; e; e >>= 1) {
        if (e & 1) acc = mul(acc, b);
        b = mul(b, b);
    }
    return acc;
}

u64 HostMod::from_signed(long long v) const {
    long long m = v % static_cast<long long>(q);
    return m < 0 ? static_cast<u64>(m + static_cast<long long>(q)) : static_cast<u64>(m);
}

u64 shoup_of(u64 w, u64 q) { return static_cast<u64>((static_cast<u128>(w) << 64) / q); }

bool is_prime(u64 n) {
    static const u64 small[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return false;
    for (u64 p : small) {
        if (n == p) return true;
        if (n % p == 0) return false;
    }
    u64 d = n - 1;
    int r = 0;
    while (!(d & 1)) { d >>= 1; ++r; }
    auto mulm = [n](u64 a, u64 b) { return static_cast<u64>((static_cast<u128>(a) * b) % n); };
    for (u64 a : small) {
        u64 x = 1, b = a % n, e = d;
        for (; e; e >>= 1) {
            if (e & 1) x = mulm(x, b);
            b = mulm(b, b);
        }
        if (x == 1 || x == n - 1) continue;
        bool witness = true;
        for (int i = 1; i < r && witness; ++i) {
            x = mulm(x, x);
            if (x == n - 1) witness = false;
        }
        if (witness) return false;
    }
    return true;
}

std::vector<u64> ntt_primes(std::size_t count, int bits, u64 step, std::vector<u64> taken) {
    if (bits < 10 || bits > 60) throw std::invalid_argument("find_ntt_primes: bit_size out of range");
    const u64 top = u64(1) << bits;
    u64 cand = (top / step) * step + 1;
    while (cand + step > top) cand -= step;
    std::vector<u64> found;
    while (found.size() < count) {
        if (cand <= (u64(1) << (bits - 1))) throw std::runtime_error("find_ntt_primes: search exhausted");
        if (is_prime(cand) && std::find(taken.begin(), taken.end(), cand) == taken.end()) {
            found.push_back(cand);
            taken.push_back(cand);
        }
        cand -= step;
    }
    return found;
}

void validate_chain(std::size_t n, const std::vector<u64>& primes) {
    if (n < 8 || (n & (n - 1)) != 0) throw std::invalid_argument("RingParams: n must be a power of two >= 8");
    if (primes.empty()) throw std::invalid_argument("RingParams: empty modulus chain");
    for (std::size_t i = 0; i < primes.size(); ++i) {
        if (!is_prime(primes[i])) throw std::invalid_argument("RingParams: chain entry not prime");
        for (std::size_t j = i + 1; j < primes.size(); ++j)
            if (primes[i] == primes[j]) throw std::invalid_argument("RingParams: duplicate chain prime");
    }
}

std::vector<u64> make_chain(std::size_t n, const std::vector<int>& prime_bits) {
    std::vector<u64> chain;
    for (int b : prime_bits) chain.push_back(ntt_primes(1, b, static_cast<u64>(2 * n), chain)[0]);
    validate_chain(n, chain);
    return chain;
}

namespace {

std::size_t reverse_bits(std::size_t x, std::size_t width) {
    std::size_t r = 0;
    for (std::size_t b = 0; b < width; ++b) r |= ((x >> b) & 1) << (width - 1 - b);
    return r;
}

// First x^((q-1)/2n), x = 2, 3, ..., whose n-th power is -1 (ring.hpp:148-156).
u64 primitive_2n_root(const HostMod& m, std::size_t n) {
    const u64 e = (m.q - 1) / static_cast<u64>(2 * n);
    for (u64 x = 2; x < m.q; ++x) {
        u64 c = m.pow(x, e);
        if (m.pow(c, static_cast<u64>(n)) == m.q - 1) return c;
    }
    throw std::runtime_error("NttTables: no primitive 2n-th root found");
}

// little-endian multiword helpers for the CRT constants
void big_mul_small(std::vector<u64>& a, u64 m) {
    u64 carry = 0;
    for (auto& w : a) {
        u128 t = static_cast<u128>(w) * m + carry;
        w = static_cast<u64>(t);
        carry = static_cast<u64>(t >> 64);
    }
    if (carry) a.push_back(carry);
}

std::vector<u64> big_div_small(const std::vector<u64>& a, u64 d, u64& rem) {
    std::vector<u64> out(a.size(), 0);
    u128 r = 0;
    for (std::size_t i = a.size(); i-- > 0;) {
        u128 cur = (r << 64) | a[i];
        out[i] = static_cast<u64>(cur / d);
        r = cur % d;
    }
    rem = static_cast<u64>(r);
    return out;
}

}  // namespace

void RingTables::build(std::size_t degree, const std::vector<u64>& chain) {
    validate_chain(degree, chain);
    n = degree;
    logn = 0;
    while ((std::size_t(1) << logn) < n) ++logn;
    primes = chain;
    limbs = chain.size();
    mods.clear();
    for (u64 q : primes) mods.emplace_back(q);
    for (u64 q : primes)
        if (q % (2 * n) != 1) throw std::invalid_argument("CkksEngine: all chain primes must be NTT-friendly");

    fwd.assign(limbs * n * 2, 0);
    inv.assign(limbs * n * 2, 0);
    n_inv.assign(limbs * 2, 0);
    fwd_f.assign(limbs * n, 0.0);
    inv_f.assign(limbs * n, 0.0);
    n_inv_f.assign(limbs, 0.0);
    for (std::size_t l = 0; l < limbs; ++l) {
        const HostMod& m = mods[l];
        u64 psi = primitive_2n_root(m, n);
        u64 psi_inv = m.inv(psi);
        for (std::size_t i = 0; i < n; ++i) {
            std::size_t r = reverse_bits(i, logn);
            u64 w = m.pow(psi, r), wi = m.pow(psi_inv, r);
            fwd[(l * n + i) * 2] = w;
            fwd[(l * n + i) * 2 + 1] = shoup_of(w, m.q);
            inv[(l * n + i) * 2] = wi;
            inv[(l * n + i) * 2 + 1] = shoup_of(wi, m.q);
            fwd_f[l * n + i] = static_cast<double>(w);
            inv_f[l * n + i] = static_cast<double>(wi);
        }
        u64 ni = m.inv(static_cast<u64>(n % m.q));
        n_inv[2 * l] = ni;
        n_inv[2 * l + 1] = shoup_of(ni, m.q);
        n_inv_f[l] = static_cast<double>(ni);
    }

    inv_dropped.assign(limbs * limbs * 2, 0);
    p_mod.assign(limbs * limbs, 0);
    for (std::size_t l = 1; l < limbs; ++l)
        for (std::size_t i = 0; i < l; ++i) {
            u64 pm = primes[l] % primes[i];
            u64 v = mods[i].inv(pm);
            inv_dropped[(l * limbs + i) * 2] = v;
            inv_dropped[(l * limbs + i) * 2 + 1] = shoup_of(v, primes[i]);
            p_mod[l * limbs + i] = pm;
        }

    // CRT: Q_l, Q_l / q_i, (Q_l / q_i)^{-1} mod q_i
    std::vector<u64> q_top{1};
    for (u64 q : primes) big_mul_small(q_top, q);
    crt_words = q_top.size() + 1;  // headroom for sum_i w_i * (Q/q_i) < (l+1) Q
    punct_inv.assign(limbs * limbs * 2, 0);
    punct.assign(limbs * limbs * crt_words, 0);
    modulus.assign(limbs * crt_words, 0);
    log2_mod.assign(limbs, 0.0);
    for (std::size_t l = 0; l < limbs; ++l) {
        std::vector<u64> Q{1};
        for (std::size_t i = 0; i <= l; ++i) big_mul_small(Q, primes[i]);
        std::copy(Q.begin(), Q.end(), modulus.begin() + l * crt_words);
        for (std::size_t i = 0; i <= l; ++i) {
            u64 rem = 0;
            std::vector<u64> P = big_div_small(Q, primes[i], rem);
            u64 pmod = 0;
            big_div_small(P, primes[i], pmod);
            u64 pinv = mods[i].inv(pmod);
            punct_inv[(l * limbs + i) * 2] = pinv;
            punct_inv[(l * limbs + i) * 2 + 1] = shoup_of(pinv, primes[i]);
            std::copy(P.begin(), P.end(), punct.begin() + (l * limbs + i) * crt_words);
        }
        double b = 0;
        for (std::size_t i = 0; i <= l; ++i) b += std::log2(static_cast<double>(primes[i]));
        log2_mod[l] = b;
    }
}

std::size_t RingTables::relin_digits(std::size_t level) const {
    std::size_t bits = static_cast<std::size_t>(std::ceil(log2_mod[level]));
    return (bits + 20 - 1) / 20;
}

}  // namespace hecnn_b200
