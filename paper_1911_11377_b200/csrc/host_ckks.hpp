// Host-side CKKS numerics that must stay on the CPU for bit-exactness with
// the reference: the mt19937_64 + libm samplers (common.hpp:173-210,
// ring.hpp:461-495), the canonical-embedding encoder/decoder with its
// long-double twiddles (ckks.hpp:79-154, 530-570), scalar-plaintext residues
// (ckks.hpp:413-429) and the encode-range checks (ckks.hpp:521-528). None of
// this is on the ciphertext hot path; it produces small integer inputs for
// the device kernels.
#pragma once
#include <complex>
#include <cstdint>
#include <random>
#include <vector>

#include "ring_host.hpp"

namespace hecnn_b200 {

u64 splitmix64(u64 x);
inline u64 derive_seed(u64 seed, u64 domain) { return splitmix64(seed ^ splitmix64(domain)); }

// Deterministic stream with the reference's distribution code.
class HostRng {
public:
    explicit HostRng(u64 seed) : gen_(seed) {}
    u64 next() { return gen_(); }
    double uniform01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    u64 below(u64 bound);
    double gaussian();

private:
    std::mt19937_64 gen_;
    bool cached_valid_ = false;
    double cached_ = 0.0;
};

// Small signed coefficient vectors (same integer under every limb).
std::vector<long long> sample_ternary(std::size_t n, double density, u64 seed);
std::vector<long long> sample_gaussian(std::size_t n, double sigma, u64 seed);
// Uniform residues [(level+1)][n] (sample_poly Uniform).
std::vector<u64> sample_uniform(const RingTables& R, std::size_t level, u64 seed);

// Result of encoding one slot vector: integer coefficients when all fit in
// i64 (the reference's fast set_coeff path), else full residues.
struct EncodedCoeffs {
    bool small = true;
    std::vector<long long> coeffs;  // [n] when small
    std::vector<u64> residues;      // [(level+1)][n] otherwise
};

class Encoder {
public:
    Encoder(const RingTables& R, double default_scale);
    // check_encode (ckks.hpp:521-528)
    void check_encode(std::size_t len, double maxval, double scale, std::size_t level) const;
    // encode_real (ckks.hpp:105-129)
    void encode_real(const double* values, std::size_t len, double scale, std::size_t level, EncodedCoeffs& out) const;
    // decode (ckks.hpp:142-154), real parts of the first `count` slots of a
    // coefficient-domain plaintext [(level+1)][n]
    void decode_real(const u64* poly, std::size_t level, double scale, double* out, std::size_t count) const;
    // residues of roundl(c * scale) per limb 0..level after check_encode:
    // make_scalar_plain (ckks.hpp:413-429) == encode_const's coefficient 0
    std::vector<u64> scalar_residues(double c, double scale, std::size_t level) const;
    // same without the range check (used when the reference does not check)
    std::vector<u64> residues_of_rounded(long double v, std::size_t level) const;

private:
    void fft(std::vector<std::complex<double>>& a, bool invert) const;
    long double centred_coeff(const u64* poly, std::size_t level, std::size_t k) const;

    const RingTables& R_;
    std::vector<std::complex<double>> twiddle_, twist_;
};

}  // namespace hecnn_b200
