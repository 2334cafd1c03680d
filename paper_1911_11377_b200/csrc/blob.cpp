#include "blob.hpp"

namespace hecnn_b200::blob {

namespace {
constexpr char kMagic[4] = {'C', 'K', 'K', 'S'};
constexpr std::uint16_t kVersion = 1;
}  // namespace

void Writer::header(Kind kind, const Params& p) {
    for (char c : kMagic) le<char>(c);
    le<std::uint16_t>(kVersion);
    le<std::uint16_t>(kind);
    le<std::uint32_t>(static_cast<std::uint32_t>(p.n));
    le<std::uint16_t>(static_cast<std::uint16_t>(p.primes.size()));
    for (u64 q : p.primes) le<u64>(q);
    le<double>(p.scale);
    le<double>(p.sigma);
    le<std::uint8_t>(p.degenerate ? 1 : 0);
}

Params Reader::header(Kind expected) {
    char magic[4];
    raw(magic, 4);
    if (std::memcmp(magic, kMagic, 4) != 0) throw std::runtime_error("ckks blob: bad magic");
    if (le<std::uint16_t>() != kVersion) throw std::runtime_error("ckks blob: unsupported version");
    if (le<std::uint16_t>() != expected) throw std::runtime_error("ckks blob: wrong object kind");
    Params p;
    p.n = le<std::uint32_t>();
    p.primes.resize(le<std::uint16_t>());
    for (u64& q : p.primes) q = le<u64>();
    p.scale = le<double>();
    p.sigma = le<double>();
    p.degenerate = le<std::uint8_t>() != 0;
    return p;
}

bool same(const Params& a, const Params& b) {
    return a.n == b.n && a.primes == b.primes && a.scale == b.scale && a.sigma == b.sigma &&
           a.degenerate == b.degenerate;
}

}  // namespace hecnn_b200::blob
