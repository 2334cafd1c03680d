// Host-side ring setup: the chain of primes, per-limb NTT tables in the
// reference's bit-reversed order, rescale inverses and the per-level CRT
// tables. This is one-time setup (RingContext ctor, ring.hpp:171-201, and
// NttTables ctor, ring.hpp:58-79); the arrays it builds are uploaded to the
// device once and never touched by the host again.
#pragma once
#include <cstddef>
#include <cstdint>
#include <vector>

namespace hecnn_b200 {

using u64 = std::uint64_t;
using u128 = unsigned __int128;

// Scalar modulus with the reference's Barrett ratio (common.hpp:32-92).
struct HostMod {
    u64 q = 0, ratio_lo = 0, ratio_hi = 0;
    HostMod() = default;
    explicit HostMod(u64 q);
    u64 mul(u64 a, u64 b) const;
    u64 add(u64 a, u64 b) const { u64 s = a + b; return s >= q ? s - q : s; }
    u64 sub(u64 a, u64 b) const { return a >= b ? a - b : a + q - b; }
    u64 pow(u64 base, u64 e) const;
    u64 inv(u64 a) const { return pow(a, q - 2); }
    u64 from_signed(long long v) const;
};

u64 shoup_of(u64 w, u64 q);
bool is_prime(u64 n);
// Largest primes below 2^bits with p == 1 (mod step), excluding `taken`
// (find_ntt_primes, common.hpp:146-162).
std::vector<u64> ntt_primes(std::size_t count, int bits, u64 step, std::vector<u64> taken);
// RingParams::create (ring.hpp:20-30)
std::vector<u64> make_chain(std::size_t n, const std::vector<int>& prime_bits);
// RingParams::validate (ring.hpp:39-47)
void validate_chain(std::size_t n, const std::vector<u64>& primes);

// All tables for one context, laid out exactly as the device wants them.
struct RingTables {
    std::size_t n = 0, logn = 0, limbs = 0;  // limbs = chain length = L + 1
    std::vector<u64> primes;
    std::vector<HostMod> mods;
    // [limb][n] pairs (value, shoup): forward roots psi^bitrev(i), inverse roots
    std::vector<u64> fwd, inv;
    std::vector<u64> n_inv;          // [limb][2]
    std::vector<double> fwd_f, inv_f, n_inv_f;  // FP64 path: [limb][n] / [limb] residues as doubles
    std::vector<u64> inv_dropped;    // [l][i][2]: p_l^{-1} mod q_i and Shoup
    std::vector<u64> p_mod;          // [l][i]: p_l mod q_i
    // CRT per level l (ring.hpp:165-169, 185-200)
    std::size_t crt_words = 0;       // words per big value (fixed stride)
    std::vector<u64> punct_inv;      // [l][i][2]: (Q_l/q_i)^{-1} mod q_i and Shoup
    std::vector<u64> punct;          // [l][i][crt_words]: Q_l/q_i
    std::vector<u64> modulus;        // [l][crt_words]: Q_l
    std::vector<double> log2_mod;    // [l]: sum of log2(q_i), i <= l (ring.hpp:224-228)

    void build(std::size_t n, const std::vector<u64>& primes);
    std::size_t relin_digits(std::size_t level) const;  // ckks.hpp:509-512
};

}  // namespace hecnn_b200
