// CKKS blob v1 codec (the reference's wire format, ckks_serialize.hpp:3-10):
//
//   "CKKS" | version u16 = 1 | kind u16 | n u32 | chain_len u16 |
//   primes u64[chain_len] | scale f64 | sigma f64 | degenerate u8 | payload
//   poly payload: level u16 | rep u8 | (level+1) * n residues u64
//
// little-endian throughout. Host-only byte work: blobs are decoded straight
// into the limb-major [2][level+1][n] words the device tensors use (a
// ciphertext cell is c0's rows followed by c1's, the same order as the blob
// payload), so ingest is one pass over the bytes plus one H2D copy.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <vector>

namespace hecnn_b200::blob {

using u64 = std::uint64_t;

enum Kind : std::uint16_t { kSecret = 1, kPublic = 2, kEval = 3, kCipher = 4 };  // BlobKind, ckks_serialize.hpp:17-22

struct Params {
    std::size_t n = 0;
    std::vector<u64> primes;
    double scale = 0.0, sigma = 0.0;
    bool degenerate = false;
};

class Writer {
public:
    template <class T>
    void le(T v) {
        const std::size_t o = b_.size();
        b_.resize(o + sizeof(T));
        std::memcpy(b_.data() + o, &v, sizeof(T));  // hosts are little-endian, as the format
    }
    void words(const u64* w, std::size_t count) {
        const std::size_t o = b_.size();
        b_.resize(o + count * 8);
        std::memcpy(b_.data() + o, w, count * 8);
    }
    // write_poly (ckks_serialize.hpp:60-65)
    void poly(std::uint16_t level, std::uint8_t rep, const u64* rows, std::size_t n) {
        le<std::uint16_t>(level);
        le<std::uint8_t>(rep);
        words(rows, (static_cast<std::size_t>(level) + 1) * n);
    }
    void header(Kind kind, const Params& p);
    const std::vector<std::uint8_t>& bytes() const { return b_; }

private:
    std::vector<std::uint8_t> b_;
};

class Reader {
public:
    Reader(const std::uint8_t* p, std::size_t len) : p_(p), len_(len) {}
    void raw(void* dst, std::size_t bytes) {
        // io::read_bytes (io_util.hpp:21-24)
        if (!p_ || len_ - off_ < bytes) throw std::runtime_error("io: unexpected end of file");
        std::memcpy(dst, p_ + off_, bytes);
        off_ += bytes;
    }
    template <class T>
    T le() {
        T v;
        raw(&v, sizeof(T));
        return v;
    }
    // read_poly (ckks_serialize.hpp:67-75) into caller storage of `cap`
    // words; returns (level, rep). The level is checked against `cap` before
    // any word is copied, and every residue against its limb's prime: the
    // device kernels assume canonical words in [0, q_i) (the FP64 path needs
    // them below 2^52), so an unreduced blob is an error, not silent garbage.
    std::pair<std::uint16_t, std::uint8_t> poly(u64* dst, std::size_t n, std::size_t cap_words, const u64* primes) {
        const auto level = le<std::uint16_t>();
        const auto rep = le<std::uint8_t>();
        const std::size_t words = (static_cast<std::size_t>(level) + 1) * n;
        if (words > cap_words) throw std::invalid_argument("ckks blob: polynomial level exceeds the caller's storage");
        raw(dst, words * 8);
        for (std::size_t i = 0; i <= level; ++i)
            for (std::size_t j = 0; j < n; ++j)
                if (dst[i * n + j] >= primes[i])
                    throw std::invalid_argument("ckks blob: residue not reduced modulo its prime");
        return {level, rep};
    }
    Params header(Kind expected);  // read_header (ckks_serialize.hpp:41-58)
    std::size_t offset() const { return off_; }

private:
    const std::uint8_t* p_;
    std::size_t len_, off_ = 0;
};

// same_params (ckks_serialize.hpp:145-148) against a context's parameters
bool same(const Params& a, const Params& b);

}  // namespace hecnn_b200::blob
