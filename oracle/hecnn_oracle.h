/*
 * TEST INFRASTRUCTURE ONLY -- the parity checker, never the product.
 *
 * Plain-C restatement of the reference's integer arithmetic on the
 * encrypted-CNN hot path (hecnn, /root/reference/proj/include/hecnn): the
 * negacyclic NTT/INTT, rescale, exact CRT + base-2^20 digit decomposition,
 * key switching, HE mul/square, scalar multiply and the conv/dense/pool
 * scalar-MAC. Each function cites the reference code it restates.
 *
 * Pinning: tests/test_oracle.py checks every function here against the
 * reference itself (oracle/_ref/libhecnn_ref.so, compiled from the unmodified
 * reference headers) and against the golden vectors in tests/golden/ that
 * the reference generated (tests/golden/make_golden.py), plus the reference's
 * own known answers (toy ring n=8, q=17; test_ring.cpp:83-125).
 *
 * Layouts: polys [limb][n] u64 (limb-major, ring.hpp:239-253); a ciphertext
 * is [2][level+1][n]; evk is [digits][2][top+1][n] (NTT domain).
 */
#ifndef HECNN_ORACLE_H
#define HECNN_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* NTT tables for one prime (NttTables ctor, ring.hpp:58-79):
 * roots/iroots [n] = psi^bitrev(i) / psi^-bitrev(i). Returns 0 on success. */
int or_ntt_tables(size_t n, uint64_t q, uint64_t* roots, uint64_t* iroots, uint64_t* n_inv);
/* NttTables::forward / inverse (ring.hpp:83-137), in place, canonical output */
void or_ntt_forward(size_t n, uint64_t q, const uint64_t* roots, uint64_t* a);
void or_ntt_inverse(size_t n, uint64_t q, const uint64_t* iroots, uint64_t n_inv, uint64_t* a);
/* O(n^2) negacyclic product (test support oracle, tests/support/oracles.hpp:16-38) */
void or_naive_negacyclic(size_t n, uint64_t q, const uint64_t* a, const uint64_t* b, uint64_t* out);

/* rescale_poly (ring.hpp:419-442): in [(level+1)][n] -> out [level][n] */
void or_rescale(size_t n, const uint64_t* primes, size_t level, const uint64_t* in, uint64_t* out);

/* relin_digits (ckks.hpp:509-512) */
size_t or_relin_digits(const uint64_t* primes, size_t level);
/* reconstruct_mod_q (ring.hpp:529-538) + BigUInt::bits (bigint.hpp:110-114):
 * digits [D][n] of d2 (coefficient domain, [(level+1)][n]) */
void or_crt_digits(size_t n, const uint64_t* primes, size_t level, const uint64_t* d2, size_t D, uint32_t* digits);

/* key_switch (ckks.hpp:601-630): d2 coeff [(level+1)][n] -> out [2][(level+1)][n] NTT domain.
 * tables: roots [(top+1)][n] of every prime. */
void or_key_switch(size_t n, const uint64_t* primes, size_t top, const uint64_t* roots, size_t level,
                   const uint64_t* d2, const uint64_t* evk, uint64_t* out);
/* CkksEngine::mul / square (ckks.hpp:315-369) on one ciphertext pair at `level`:
 * out [2][level][n]. y == NULL means square. */
void or_mul(size_t n, const uint64_t* primes, size_t top, size_t level, const uint64_t* x, const uint64_t* y,
            const uint64_t* evk, uint64_t* out);

/* scalar_mul + rescale = mul_plain with a constant (ckks.hpp:372-398, 588-597):
 * residues[i] is the constant's residue mod q_i; out [2][level][n] */
void or_mul_const(size_t n, const uint64_t* primes, size_t level, const uint64_t* x, const uint64_t* residues,
                  uint64_t* out);

/* conv/dense scalar MAC of one output ciphertext (ckks.hpp:448-472 + rescale):
 * out = rescale( sum_k w[k] * x[src[k]] + bias on c0 coefficient 0 ).
 * xs [cells][2][level+1][n]; w [K][level+1] residues; bias [level+1]. */
void or_scalar_mac(size_t n, const uint64_t* primes, size_t level, const uint64_t* xs, const int* src, size_t K,
                   const uint64_t* w, const uint64_t* bias, uint64_t* out);

#ifdef __cplusplus
}
#endif
#endif
