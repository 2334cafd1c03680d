/*
 * TEST INFRASTRUCTURE ONLY -- the parity checker, never the product.
 * Plain-C restatement of the reference's hot-path integer arithmetic; see
 * hecnn_oracle.h for the contract and how it is pinned.
 */
#include "hecnn_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;
typedef uint64_t u64;

static u64 mulmod(u64 a, u64 b, u64 q) { return (u64)(((u128)a * b) % q); }
static u64 addmod(u64 a, u64 b, u64 q) { u64 s = a + b; return s >= q ? s - q : s; }
static u64 submod(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }

static u64 powmod(u64 b, u64 e, u64 q) {
    u64 r = 1 % q;
    b %= q;
    while (e) {
        if (e & 1) r = mulmod(r, b, q);
        b = mulmod(b, b, q);
        e >>= 1;
    }
    return r;
}

static u64 invmod(u64 a, u64 q) { return powmod(a, q - 2, q); }

static size_t bitrev(size_t x, size_t bits) {
    size_t r = 0;
    for (size_t i = 0; i < bits; ++i) r |= ((x >> i) & 1) << (bits - 1 - i);
    return r;
}

/* ring.hpp:58-79, 148-156: psi = first x^((q-1)/2n) (x = 2, 3, ...) with psi^n = -1 */
int or_ntt_tables(size_t n, uint64_t q, uint64_t* roots, uint64_t* iroots, uint64_t* n_inv) {
    if (q % (2 * n) != 1) return 1;
    size_t logn = 0;
    while (((size_t)1 << logn) < n) ++logn;
    u64 e = (q - 1) / (2 * n), psi = 0;
    for (u64 x = 2; x < q; ++x) {
        u64 c = powmod(x, e, q);
        if (powmod(c, n, q) == q - 1) { psi = c; break; }
    }
    if (!psi) return 2;
    u64 psi_inv = invmod(psi, q);
    for (size_t i = 0; i < n; ++i) {
        roots[i] = powmod(psi, bitrev(i, logn), q);
        iroots[i] = powmod(psi_inv, bitrev(i, logn), q);
    }
    *n_inv = invmod(n % q, q);
    return 0;
}

/* ring.hpp:83-108 (exact arithmetic: same linear map, canonical output) */
void or_ntt_forward(size_t n, uint64_t q, const uint64_t* roots, uint64_t* a) {
    size_t t = n;
    for (size_t m = 1; m < n; m <<= 1) {
        t >>= 1;
        for (size_t i = 0; i < m; ++i) {
            u64 s = roots[m + i];
            for (size_t j = 2 * i * t; j < 2 * i * t + t; ++j) {
                u64 u = a[j], v = mulmod(a[j + t], s, q);
                a[j] = addmod(u, v, q);
                a[j + t] = submod(u, v, q);
            }
        }
    }
}

/* ring.hpp:110-137 */
void or_ntt_inverse(size_t n, uint64_t q, const uint64_t* iroots, uint64_t n_inv, uint64_t* a) {
    size_t t = 1;
    for (size_t m = n; m > 1; m >>= 1) {
        size_t h = m >> 1, j1 = 0;
        for (size_t i = 0; i < h; ++i) {
            u64 s = iroots[h + i];
            for (size_t j = j1; j < j1 + t; ++j) {
                u64 u = a[j], v = a[j + t];
                a[j] = addmod(u, v, q);
                a[j + t] = mulmod(submod(u, v, q), s, q);
            }
            j1 += 2 * t;
        }
        t <<= 1;
    }
    for (size_t j = 0; j < n; ++j) a[j] = mulmod(a[j], n_inv, q);
}

/* tests/support/oracles.hpp:16-38 */
void or_naive_negacyclic(size_t n, uint64_t q, const uint64_t* a, const uint64_t* b, uint64_t* out) {
    for (size_t k = 0; k < n; ++k) {
        u64 acc = 0;
        for (size_t i = 0; i < n; ++i) {
            if (k >= i) acc = addmod(acc, mulmod(a[i], b[k - i], q), q);
            else acc = submod(acc, mulmod(a[i], b[k + n - i], q), q);
        }
        out[k] = acc;
    }
}

/* ring.hpp:419-442 */
void or_rescale(size_t n, const uint64_t* primes, size_t level, const uint64_t* in, uint64_t* out) {
    u64 p = primes[level];
    const u64* last = in + level * n;
    for (size_t i = 0; i < level; ++i) {
        u64 q = primes[i], pmod = p % q, pinv = invmod(pmod, q);
        for (size_t j = 0; j < n; ++j) {
            u64 v = last[j], c = v % q;
            if (v > (p >> 1)) c = submod(c, pmod, q);
            out[i * n + j] = mulmod(submod(in[i * n + j], c, q), pinv, q);
        }
    }
}

/* ckks.hpp:509-512, ring.hpp:224-228 */
size_t or_relin_digits(const uint64_t* primes, size_t level) {
    double b = 0;
    for (size_t i = 0; i <= level; ++i) b += log2((double)primes[i]);
    size_t bits = (size_t)ceil(b);
    return (bits + 19) / 20;
}

/* multiword helpers (little endian) for the exact CRT */
static void big_mul_small(u64* a, size_t w, u64 m) {
    u64 carry = 0;
    for (size_t i = 0; i < w; ++i) {
        u128 t = (u128)a[i] * m + carry;
        a[i] = (u64)t;
        carry = (u64)(t >> 64);
    }
}

static void big_add_mul(u64* acc, const u64* a, size_t w, u64 m) {
    u64 carry = 0;
    for (size_t i = 0; i < w; ++i) {
        u128 t = (u128)a[i] * m + acc[i] + carry;
        acc[i] = (u64)t;
        carry = (u64)(t >> 64);
    }
}

static int big_cmp(const u64* a, const u64* b, size_t w) {
    for (size_t i = w; i-- > 0;)
        if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    return 0;
}

static void big_sub(u64* a, const u64* b, size_t w) {
    u64 borrow = 0;
    for (size_t i = 0; i < w; ++i) {
        u128 d = (u128)a[i] - b[i] - borrow;
        a[i] = (u64)d;
        borrow = (u64)(d >> 64) ? 1 : 0;
    }
}

static u64 big_div_small(const u64* a, size_t w, u64 d, u64* quot) {
    u128 r = 0;
    for (size_t i = w; i-- > 0;) {
        u128 cur = (r << 64) | a[i];
        quot[i] = (u64)(cur / d);
        r = cur % d;
    }
    return (u64)r;
}

/* ring.hpp:185-200 (CRT tables) + 529-538 (reconstruct_mod_q) + bigint.hpp:110-114 */
void or_crt_digits(size_t n, const uint64_t* primes, size_t level, const uint64_t* d2, size_t D, uint32_t* digits) {
    size_t w = level + 3;
    u64* Q = calloc(w, 8);
    u64* P = calloc((level + 1) * w, 8);
    u64* pinv = calloc(level + 1, 8);
    u64* acc = calloc(w, 8);
    Q[0] = 1;
    for (size_t i = 0; i <= level; ++i) big_mul_small(Q, w, primes[i]);
    for (size_t i = 0; i <= level; ++i) {
        big_div_small(Q, w, primes[i], P + i * w);
        pinv[i] = invmod(big_div_small(P + i * w, w, primes[i], acc) % primes[i], primes[i]);
    }
    for (size_t j = 0; j < n; ++j) {
        memset(acc, 0, w * 8);
        for (size_t i = 0; i <= level; ++i) big_add_mul(acc, P + i * w, w, mulmod(d2[i * n + j], pinv[i], primes[i]));
        while (big_cmp(acc, Q, w) >= 0) big_sub(acc, Q, w);
        for (size_t t = 0; t < D; ++t) {
            size_t off = 20 * t, wi = off / 64, sh = off % 64;
            u64 lo = wi < w ? acc[wi] >> sh : 0;
            if (sh && sh + 20 > 64 && wi + 1 < w) lo |= acc[wi + 1] << (64 - sh);
            digits[t * n + j] = (uint32_t)(lo & 0xFFFFF);
        }
    }
    free(Q);
    free(P);
    free(pinv);
    free(acc);
}

/* ckks.hpp:601-630 */
void or_key_switch(size_t n, const uint64_t* primes, size_t top, const uint64_t* roots, size_t level,
                   const uint64_t* d2, const uint64_t* evk, uint64_t* out) {
    size_t D = or_relin_digits(primes, level);
    uint32_t* dig = malloc(D * n * sizeof(uint32_t));
    u64* dp = malloc(n * 8);
    or_crt_digits(n, primes, level, d2, D, dig);
    memset(out, 0, 2 * (level + 1) * n * 8);
    size_t key_poly = (top + 1) * n;
    for (size_t t = 0; t < D; ++t)
        for (size_t i = 0; i <= level; ++i) {
            u64 q = primes[i];
            for (size_t j = 0; j < n; ++j) dp[j] = dig[t * n + j] % q;
            or_ntt_forward(n, q, roots + i * n, dp);
            const u64* b = evk + (2 * t) * key_poly + i * n;
            const u64* a = evk + (2 * t + 1) * key_poly + i * n;
            for (size_t j = 0; j < n; ++j) {
                out[i * n + j] = addmod(out[i * n + j], mulmod(dp[j], b[j], q), q);
                out[(level + 1) * n + i * n + j] = addmod(out[(level + 1) * n + i * n + j], mulmod(dp[j], a[j], q), q);
            }
        }
    free(dig);
    free(dp);
}

/* ckks.hpp:315-369 */
void or_mul(size_t n, const uint64_t* primes, size_t top, size_t level, const uint64_t* x, const uint64_t* y,
            const uint64_t* evk, uint64_t* out) {
    size_t L = level + 1, pw = L * n;
    u64* roots = malloc((top + 1) * n * 8);
    u64* iroots = malloc((top + 1) * n * 8);
    u64* ninv = malloc((top + 1) * 8);
    for (size_t i = 0; i <= top; ++i) or_ntt_tables(n, primes[i], roots + i * n, iroots + i * n, ninv + i);
    u64* f = malloc(4 * pw * 8); /* fx0 fx1 fy0 fy1 */
    memcpy(f, x, 2 * pw * 8);
    memcpy(f + 2 * pw, y ? y : x, 2 * pw * 8);
    for (size_t c = 0; c < 4; ++c)
        for (size_t i = 0; i < L; ++i) or_ntt_forward(n, primes[i], roots + i * n, f + c * pw + i * n);
    u64* d = malloc(3 * pw * 8); /* d0 d1 d2 */
    for (size_t i = 0; i < L; ++i)
        for (size_t j = 0; j < n; ++j) {
            u64 q = primes[i], k = i * n + j;
            u64 x0 = f[k], x1 = f[pw + k], y0 = f[2 * pw + k], y1 = f[3 * pw + k];
            d[k] = mulmod(x0, y0, q);
            d[pw + k] = addmod(mulmod(x0, y1, q), mulmod(x1, y0, q), q);
            d[2 * pw + k] = mulmod(x1, y1, q);
        }
    for (size_t i = 0; i < L; ++i) or_ntt_inverse(n, primes[i], iroots + i * n, ninv[i], d + 2 * pw + i * n);
    u64* ks = malloc(2 * pw * 8);
    or_key_switch(n, primes, top, roots, level, d + 2 * pw, evk, ks);
    for (size_t k = 0; k < 2 * pw; ++k) d[k] = addmod(d[k], ks[k], primes[(k % pw) / n]);
    for (size_t c = 0; c < 2; ++c)
        for (size_t i = 0; i < L; ++i) or_ntt_inverse(n, primes[i], iroots + i * n, ninv[i], d + c * pw + i * n);
    or_rescale(n, primes, level, d, out);
    or_rescale(n, primes, level, d + pw, out + level * n);
    free(roots);
    free(iroots);
    free(ninv);
    free(f);
    free(d);
    free(ks);
}

/* ckks.hpp:372-398 + 588-597 */
void or_mul_const(size_t n, const uint64_t* primes, size_t level, const uint64_t* x, const uint64_t* residues,
                  uint64_t* out) {
    size_t pw = (level + 1) * n;
    u64* t = malloc(2 * pw * 8);
    for (size_t k = 0; k < 2 * pw; ++k) {
        size_t i = (k % pw) / n;
        t[k] = mulmod(x[k], residues[i], primes[i]);
    }
    or_rescale(n, primes, level, t, out);
    or_rescale(n, primes, level, t + pw, out + level * n);
    free(t);
}

/* ckks.hpp:431-472 (make_zero_ciphertext, mul_scalar_mac, add_scalar_inplace) + rescale */
void or_scalar_mac(size_t n, const uint64_t* primes, size_t level, const uint64_t* xs, const int* src, size_t K,
                   const uint64_t* w, const uint64_t* bias, uint64_t* out) {
    size_t pw = (level + 1) * n;
    u64* acc = calloc(2 * pw, 8);
    for (size_t k = 0; k < K; ++k) {
        if (src[k] < 0) continue;
        const u64* x = xs + (size_t)src[k] * 2 * pw;
        for (size_t e = 0; e < 2 * pw; ++e) {
            size_t i = (e % pw) / n;
            acc[e] = addmod(acc[e], mulmod(x[e], w[k * (level + 1) + i], primes[i]), primes[i]);
        }
    }
    if (bias)
        for (size_t i = 0; i <= level; ++i) acc[i * n] = addmod(acc[i * n], bias[i], primes[i]);
    or_rescale(n, primes, level, acc, out);
    or_rescale(n, primes, level, acc + pw, out + level * n);
    free(acc);
}
