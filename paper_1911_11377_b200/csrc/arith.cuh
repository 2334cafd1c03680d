// Device-side 64-bit modular arithmetic for the RNS limbs (q < 2^61).
//
// Semantics follow the reference's scalar primitives (proj/include/hecnn/
// common.hpp:32-111): Barrett reduction of a 128-bit value with the ratio
// floor((2^128-1)/q), Shoup multiplication by a fixed operand, and the lazy
// Shoup variant with results in [0, 2q). All of them produce the canonical
// residue after the final conditional subtraction, so every kernel built on
// them is bit-exact against the CPU path regardless of evaluation order.
#pragma once
#include <cstdint>

namespace hecnn_b200 {

using u32 = std::uint32_t;
using u64 = std::uint64_t;

// Per-limb modulus constants kept in one 32-byte record so a limb's constants
// come in with a single pair of vector loads.
struct ModConst {
    u64 q;
    u64 two_q;
    u64 ratio_lo;  // floor((2^128-1)/q) low word
    u64 ratio_hi;  // ... high word
};

#ifdef __CUDACC__
__device__ __forceinline__ u64 mulhi(u64 a, u64 b) { return __umul64hi(a, b); }

// x*w mod q, lazy: result in [0, 2q) for any x < 2^64 (common.hpp:108-111).
__device__ __forceinline__ u64 mul_shoup_lazy(u64 x, u64 w, u64 w_shoup, u64 q) {
    return x * w - mulhi(x, w_shoup) * q;
}

// x*w mod q, canonical (common.hpp:100-104).
__device__ __forceinline__ u64 mul_shoup(u64 x, u64 w, u64 w_shoup, u64 q) {
    u64 r = mul_shoup_lazy(x, w, w_shoup, q);
    return r >= q ? r - q : r;
}

// Barrett reduction of hi:lo (any 128-bit value) to [0, q) (common.hpp:45-58).
// The quotient estimate floor(V*ratio/2^128) is exact up to the dropped low
// word, so it is within 1 of floor(V/q) for every V < 2^128; one conditional
// subtraction finishes.
__device__ __forceinline__ u64 reduce128(u64 lo, u64 hi, const ModConst& m) {
    u64 carry = mulhi(lo, m.ratio_lo);
    u64 t_lo = lo * m.ratio_hi;
    u64 t_hi = mulhi(lo, m.ratio_hi);
    u64 tmp1 = t_lo + carry;
    u64 tmp3 = t_hi + (tmp1 < carry ? 1 : 0);
    u64 s_lo = hi * m.ratio_lo;
    u64 s_hi = mulhi(hi, m.ratio_lo);
    u64 s = tmp1 + s_lo;
    u64 carry2 = s_hi + (s < tmp1 ? 1 : 0);
    u64 quot = hi * m.ratio_hi + tmp3 + carry2;
    u64 rem = lo - quot * m.q;
    return rem >= m.q ? rem - m.q : rem;
}

// v mod q for a v that is almost always below 2q (a residue of a neighbouring
// chain prime): one conditional subtraction, Barrett only when v >= 2q.
__device__ __forceinline__ u64 reduce_near(u64 v, const ModConst& m) {
    u64 r = v >= m.q ? v - m.q : v;
    if (r >= m.q) r = reduce128(v, 0, m);
    return r;
}

__device__ __forceinline__ u64 mul_mod(u64 a, u64 b, const ModConst& m) {
    return reduce128(a * b, mulhi(a, b), m);
}

__device__ __forceinline__ u64 add_mod(u64 a, u64 b, u64 q) {
    u64 s = a + b;
    return s >= q ? s - q : s;
}

__device__ __forceinline__ u64 sub_mod(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }

__device__ __forceinline__ u64 neg_mod(u64 a, u64 q) { return a == 0 ? 0 : q - a; }

// Reduce a value in [0, 4q) to [0, q).
__device__ __forceinline__ u64 reduce_4q(u64 v, u64 q) {
    u64 two_q = q << 1;
    if (v >= two_q) v -= two_q;
    if (v >= q) v -= q;
    return v;
}

// Reduce a value in [0, 2q) to [0, q).
__device__ __forceinline__ u64 reduce_2q(u64 v, u64 q) { return v >= q ? v - q : v; }

// Signed small integer to residue (Modulus::reduce_i64, common.hpp:88-91).
__device__ __forceinline__ u64 from_signed(long long v, u64 q) {
    long long m = v % static_cast<long long>(q);
    return m < 0 ? static_cast<u64>(m + static_cast<long long>(q)) : static_cast<u64>(m);
}

#endif  // __CUDACC__

}  // namespace hecnn_b200
