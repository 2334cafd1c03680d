// Device tables and kernel launchers shared by the CUDA translation units and
// the host engine. Launchers take plain device pointers and a stream; every
// launcher bumps the context's launch counter through `Launch`.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "arith.cuh"

namespace hecnn_b200 {

// Read-only ring tables resident on the device (built by RingTables, ring_host.hpp).
struct DevRing {
    int n = 0, logn = 0, limbs = 0, crt_words = 0;
    const ModConst* mod = nullptr;           // [limbs]
    const ulonglong2* fwd = nullptr;         // [limbs][n] (psi^bitrev(i), shoup)
    const ulonglong2* inv = nullptr;         // [limbs][n] (psi^-bitrev(i), shoup)
    const ulonglong2* n_inv = nullptr;       // [limbs]
    const ulonglong2* inv_dropped = nullptr; // [limbs][limbs] (p_l^-1 mod q_i, shoup) at [l][i]
    const u64* p_mod = nullptr;              // [limbs][limbs] p_l mod q_i at [l][i]
    const ulonglong2* punct_inv = nullptr;   // [limbs][limbs] ((Q_l/q_i)^-1 mod q_i, shoup)
    const u64* punct = nullptr;              // [limbs][limbs][crt_words] Q_l/q_i
    const u64* modulus = nullptr;            // [limbs][crt_words] Q_l
    const double* garner_inv = nullptr;      // [i][j] q_j^-1 mod q_i (j < i, FP64 limbs i), exact doubles
    const double* garner_c30 = nullptr;      // [i] 2^30 mod q_i
    const double* inv_q = nullptr;           // [limbs] 1/q_i
    // FP64-path tables (limbs with q < 2^42): residues as exact doubles
    const double* fwd_f = nullptr;           // [limbs][n]
    const double* inv_f = nullptr;           // [limbs][n]
    const double* n_inv_f = nullptr;         // [limbs]
    // key-switch block-local twiddle tables (keyswitch.cu): for blocks of
    // B = 2^min(logn, 13) words, [limb][block][j] = fwd[2^(s+C) + block 2^s + m]
    // with j = 2^s + m, C = logn - log2 B (== fwd / fwd_f when N <= 2^13)
    const ulonglong2* ks_tw = nullptr;       // [limbs][n]
    const double* ks_tw_f = nullptr;         // [limbs][n]
    unsigned long long int_limbs = 0;        // bit i: q_i >= 2^42 (integer-pipe path), for i < 64
    // Key switch of the 60-bit limb 0 through limbs 1..3 (keyswitch.cu, "aux"):
    // aux_tab [Dtop][2][4][n] = NTT_{q_s}(INTT_{q0}(evk[t][c][0]) mod q_s) as
    // doubles in slots s = 1..3; CRT constants of P = q1 q2 q3.
    const double* aux_tab = nullptr;
    ulonglong2 aux_inv[3] = {};              // ((P / q_s) mod q_s)^-1 mod q_s, Shoup
    ulonglong2 aux_Mq0[3] = {};              // (P / q_s) mod q0, Shoup
    u64 aux_kPq0[4] = {};                    // k P mod q0, k = 0..3
    double aux_log2P = 0.0;
    bool small_primes = false;               // some q_i <= 2^20: key-switch digits need v mod q_i
};

// Optional per-kernel timing: CUDA events recorded on the launching stream
// around every kernel launch while enabled (see Context::profile).
struct Profiler {
    bool enabled = false;
    struct Pending {
        const char* name;
        cudaEvent_t start, stop;
        double ops, bytes;
    };
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> pool;
    const char* open_name = nullptr;
    cudaEvent_t open_start = nullptr;
    double open_ops = 0, open_bytes = 0;
    // ops: algorithmic 64-bit modular multiply-equivalents (one NTT butterfly =
    // one Shoup modmul); bytes: algorithmic (minimal) global-memory bytes.
    struct Stat {
        double ms = 0, ops = 0, bytes = 0;
        unsigned long long launches = 0;
    };
    std::map<std::string, Stat> stats;
    cudaEvent_t take();
    void begin(const char* name, cudaStream_t s, double ops, double bytes);
    void end(cudaStream_t s);
    void collect();  // call after the stream is synchronized
    void reset();
};

struct Launch {
    cudaStream_t stream = nullptr;
    unsigned long long* counter = nullptr;
    Profiler* prof = nullptr;
    // side stream for independent work inside one operation (fork/join with
    // the events below); null: everything runs on `stream`
    cudaStream_t aux = nullptr;
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
    void begin(const char* name, double ops = 0, double bytes = 0) const {
        if (prof && prof->enabled) prof->begin(name, stream, ops, bytes);
    }
    void count(unsigned long long k = 1) const {
        if (counter) *counter += k;
        if (prof && prof->enabled) prof->end(stream);
    }
};

void check_launch(const char* what);
void cuda_check(cudaError_t e, const char* what);  // throws std::runtime_error on failure
// Dynamic shared memory above 48 KB for `kernel` on the current device. The
// attribute lives in each device's context, so it is set once per (kernel,
// device, size), not once per process: a process driving two GPUs sets both.
void smem_opt_in(const void* kernel, int bytes);
template <class K>
void smem_opt_in(K* kernel, int bytes) {
    smem_opt_in(reinterpret_cast<const void*>(kernel), bytes);
}

// ---- NTT (ntt.cu). polys: [count][level+1][n], limb index = poly % (level+1)
void ntt_forward(const DevRing& R, u64* polys, int level, std::size_t count, const Launch& L);
// out of place (src may equal dst)
void ntt_forward_to(const DevRing& R, const u64* src, u64* dst, int level, std::size_t count, const Launch& L);
void ntt_inverse(const DevRing& R, u64* polys, int level, std::size_t count, const Launch& L);
// out = rescale(INTT(d)) for `groups` polys of level+1 limbs (d is overwritten); false (nothing
// launched) when the ring needs a column pass (N > 2^14): call ntt_inverse + rescale instead.
// add0 (optional, [groups][n] coefficients mod q0) is added to limb 0 after its INTT
bool ntt_inverse_rescale(const DevRing& R, u64* d, u64* out, int level, std::size_t groups, const Launch& L,
                         const u64* add0 = nullptr);
// in-place inverse NTT (with n^-1, canonical) of limbs [limb0, limb0 + nsel) of
// `groups` groups of `limbs` polys [groups][limbs][n] (N <= 2^14)
void ntt_inverse_limbs(const DevRing& R, u64* data, int limbs, int limb0, int nsel, std::size_t groups, const Launch& L,
                       const char* name = nullptr);
// d2 = INTT(x1 * y1): x, y forward-transformed ciphertexts [count][2][level+1][n] (y may equal
// x), the product formed in the first butterfly round; d2 [count][level+1][n] coefficients
void ntt_inverse_product(const DevRing& R, const u64* x, const u64* y, u64* d2, int level, std::size_t count,
                         const Launch& L);

// ---- elementwise ring ops (ring_ops.cu), [count][level+1][n]
enum class EwOp { Add, Sub, Neg, Mul, Mac };
void poly_elementwise(const DevRing& R, EwOp op, const u64* a, const u64* b, u64* out, int level,
                      std::size_t count, const Launch& L);
// rescale_poly on [count][level+1][n] -> [count][level][n] (ring.hpp:419-442)
// Terms added by rescale's fused epilogue: ciphertext tensors read at their first
// `level` limbs (+ c0 on coefficient 0 of component 0)
constexpr int kMaxTerms = 8;
struct SumTerms {
    const u64* ptr[kMaxTerms];
    int limbs[kMaxTerms];
    int count;
    const u64* c0;  // [level+1] residues or null
    // optional: + rescale(rs_c * rs) for a ciphertext tensor rs at rs_level > level
    // (mul_plain + rescale, then mod-switched: ckks.hpp:395-398, 474-493)
    const u64* rs;
    int rs_level;
    const ulonglong2* rs_c;  // [rs_level+1] (c, shoup)
};
// scale_by: optional per-limb (c, shoup) multiplied into the input first (mul_plain + rescale);
// add: optional terms (ciphertext tensors of >= level limbs, read as their first `level` limbs,
// i.e. mod-switched) and constant added to the result (count = polys = 2 x ciphertexts)
void rescale(const DevRing& R, const u64* in, u64* out, int level, std::size_t count, const Launch& L,
             const ulonglong2* scale_by = nullptr, const SumTerms* add = nullptr);
// copy limbs 0..to_level of [count][level+1][n] into [count][to_level+1][n]
void drop_limbs(const DevRing& R, const u64* in, u64* out, int level, int to_level, std::size_t count,
                const Launch& L);
// NTT-domain tensor products, F* = [count][2][level+1][n]:
//   d01 = [count][2][level+1][n] (d0, d1), d2 = [count][level+1][n]
void tensor_mul(const DevRing& R, const u64* fx, const u64* fy, u64* d01, u64* d2, int level, std::size_t count,
                const Launch& L);
void tensor_square(const DevRing& R, const u64* fx, u64* d01, u64* d2, int level, std::size_t count,
                   const Launch& L);
// out = in * c_i (Shoup) per limb; consts = [level+1] (value, shoup) pairs (ckks.hpp:588-597)
void scalar_mul(const DevRing& R, const u64* in, const ulonglong2* consts, u64* out, int level, std::size_t count,
                const Launch& L);
// c0[ct][i][0] += consts[i] for every ciphertext of a [count][2][level+1][n] batch
// (add_scalar_inplace / add_plain of a constant, ckks.hpp:305-311, 468-472)
void add_coeff0(const DevRing& R, u64* cts, const u64* consts, int level, std::size_t count, const Launch& L);
// ciphertexts [cells][2][level+1][n] against one plaintext [level+1][n]: op 0 c0 += p
// (coefficient domain), op 1 c0, c1 *= p (NTT domain); out may equal x
void plain_bcast(const DevRing& R, const u64* x, const u64* p, u64* out, int level, std::size_t cells, int op,
                 const Launch& L);
// acc [cells][2][level+1][n] += x * c_i; consts [ncs][level+1] (c, shoup), cell k uses row k % ncs
void scalar_mac(const DevRing& R, const u64* x, const ulonglong2* consts, std::size_t ncs, u64* acc, int level,
                std::size_t cells, const Launch& L);

// Shoup companions floor(w * 2^64 / q_i) of a [count][limbs][n] table (evk)
void shoup_table(const DevRing& R, const u64* in, u64* out, int limbs, std::size_t count, const Launch& L);
// FP64-path copy (exact doubles) of a [count][limbs][n] residue table (evk)
void fp_table(const DevRing& R, const u64* in, double* out, int limbs, std::size_t count, const Launch& L);

// ---- key switching (keyswitch.cu)
// CRT reconstruction + base-2^20 digits of d2 (coefficient domain): digits [count][D][n] u32
void crt_digits(const DevRing& R, const u64* d2, u32* digits, int level, int D, std::size_t count,
                const Launch& L);
// acc01[ct] (NTT domain, [count][2][level+1][n]) += sum_t NTT(digit_t) * evk_t
//   evk: [Dtop][2][limbs][n] values, evk_sh: Shoup companions
//   evk_f: FP64-path copy (used for limbs with q < 2^42)
//   mode 0: acc01 holds (d0, d1); mode 1: acc01 holds NTT(x) and d0 = x0^2, d1 = 2 x0 x1 are
//   formed in the epilogue; mode 2: likewise d0 = x0 y0, d1 = x0 y1 + x1 y0 with fy = NTT(y)
// aux_scratch: optional [count][(2 x 4 + 2) n] words; when given and the
// chain allows it, limb 0's key switch runs through limbs 1..3 (exact CRT)
// instead of on the integer pipes
// defer_limb0: the caller inverse-transforms acc01 next, so limb 0's E is not
// forward-transformed: the return value (non-null when deferred) holds E mod q0
// as coefficients [count][2][n], to be added to limb 0 after that INTT
// (ntt_inverse_rescale's add0, or add_limb0)
const u64* keyswitch_mac(const DevRing& R, const u32* digits, const u64* evk, const u64* evk_sh, const double* evk_f,
                         u64* acc01, int level, int D, std::size_t count, const Launch& L, int mode = 0,
                         const u64* fy = nullptr, u64* aux_scratch = nullptr, bool defer_limb0 = false);
// d [groups][limbs][n] (coefficients): limb 0 += add0 [groups][n] mod q0
void add_limb0(const DevRing& R, u64* d, const u64* add0, int limbs, std::size_t groups, const Launch& L);
// the limb-0-through-limbs-1..3 key switch is usable at this level / digit count
bool keyswitch_aux_ok(const DevRing& R, int level, int D);
// aux_tab of DevRing from the evaluation key (one-time, at keygen / key import):
// out [Dtop][2][4][n] doubles; tmp scratch [2 Dtop][5 n] words
void keyswitch_aux_tables(const DevRing& R, const u64* evk, std::size_t evk_limbs, int Dtop, double* out, u64* tmp,
                          const Launch& L);

// Integer-pipe peak probe: chained Shoup modmuls (the NTT butterfly's
// multiply), `iters` per thread over the whole GPU; returns modmuls issued.
double modmul_probe(const DevRing& R, int iters, u64* sink, const Launch& L);
// FP64-pipe peak probe: chained exact FP64 modmuls (ntt_core.cuh fmodmul).
double fp64_modmul_probe(const DevRing& R, int iters, u64* sink, const Launch& L);

// ---- linear layers (linear.cu)
// Gather-MAC for conv/dense: see linear.cu for the table formats.
struct GatherMac {
    const int* src;            // [pixels][K] input cell index per tap (-1: invalid tap); tap k uses weight row k
    const ulonglong2* weights; // [limbs][K][oc_pad] (residue, shoup) at level, oc_pad % 16 == 0
    const u64* bias;           // [oc][level+1] residues (added to c0 coeff 0), or null
    const uint2* wsplit;       // [limbs][K][oc_pad] residue split (w mod 2^21, w >> 21) for q < 2^42
    const ulonglong2* recomb;  // [limbs][2]: (2^21 mod q, shoup), (2^42 mod q, shoup)
    int pixels, K, oc, oc_pad, out_stride_pixel;  // output cell = pixel * out_stride_pixel + oc
};
// limbs [limb0, limb1) only (both components)
void gather_mac(const DevRing& R, const GatherMac& g, const u64* x, u64* y, int level, int limb0, int limb1,
                const Launch& L);
// The same layer on the integer tensor cores for limbs with q < 2^40 (conv_imma.cu).
struct ImmaMac {
    const int* src;          // [pixels][kpad] input cell per tap, -1 for invalid / padding taps
    const uint4* wfrag;      // [limbs][oc_tiles][ksteps][5 byte planes][32 lanes] m16n8k32 A fragments
    const u64* bias;         // [oc][level+1] residues (added to c0 coeff 0), or null
    const double* shift;     // [limbs][9]: 2^(8s) mod q as exact doubles
    int pixels, K, kpad, ksteps, oc, oc_tiles, out_stride_pixel;  // kpad = 32 * ksteps; oc_tiles even if >= 2
    // limbs with q >= 2^40: signed base-256 digits of the weight integers (one
    // copy for all limbs) [oc_tiles][ksteps][6][32 lanes], and (2^8s mod q, shoup)
    const uint4* wfrag_wide;
    const ulonglong2* shift_wide;  // [limbs][16]
    // tcgen05 path (conv_tc.cu): [limbs][ceil(oc/48)][ksteps] weight tiles of
    // 240 (byte plane, oc) rows x 32 taps in the UMMA K-major core-matrix layout
    const uint4* wtc = nullptr;
    // the 60-bit limb on tcgen05: [ceil(oc/32)][ksteps] tiles of 192 (signed digit b, oc) rows x 32 taps
    const uint4* wtc_wide = nullptr;
};
bool imma_mac_supported(const DevRing& R, std::size_t K);
// 5th-gen tensor-core conv (tcgen05.mma kind::i8, TMEM accumulators), limbs q < 2^40
// (wide: the limbs with q >= 2^40, signed weight digits)
int tc_oc_tile(bool wide);
bool tc_mac_supported(const DevRing& R, const ImmaMac& g, bool wide);
void tc_mac(const DevRing& R, const ImmaMac& g, const u64* x, u64* y, int level, int limb0, int limb1, bool wide,
            const Launch& L);
void imma_mac(const DevRing& R, const ImmaMac& g, const u64* x, u64* y, int level, int limb0, int limb1, bool wide,
              const Launch& L);
// 2x2-style average pool: out cell p sums srcs[p][0..taps) (plus y[p] when accumulate)
// then multiplies by w (shoup; w == null: no multiply), level kept
void pool_sum_scale(const DevRing& R, const u64* x, const int* srcs, int taps, const ulonglong2* w, u64* y,
                    int level, std::size_t out_cells, const Launch& L, bool accumulate = false);
// gather whole cells: y[i] = x[idx[i]] for idx >= 0 (ciphertext-sized copies)
void gather_cells(const u64* x, const int* idx, u64* y, std::size_t cell_words, std::size_t cells, const Launch& L);

// ---- encryption pieces (ring_ops.cu)
// signed small coefficients [count][n] (int8) -> residues [count][level+1][n]
void small_to_rns(const DevRing& R, const signed char* s, u64* out, int level, std::size_t count, const Launch& L);
// i64 coefficients [count][n] -> residues [count][level+1][n]
void i64_to_rns(const DevRing& R, const long long* s, u64* out, int level, std::size_t count, const Launch& L);
// out[ct][comp][i][j] = rt[ct][i][j] * pk[comp][i][j]   (NTT domain, pk at its own limb stride)
void mul_by_key(const DevRing& R, const u64* rt, const u64* pk, std::size_t pk_limbs, u64* out, int level,
                std::size_t count, const Launch& L);
// out[ct][0] += e0 + m, out[ct][1] += e1 (coefficient domain); m may be null
void add_noise_msg(const DevRing& R, u64* ct, const signed char* e0, const signed char* e1, const u64* m,
                   int level, std::size_t count, const Launch& L);
// decrypt pieces: t[ct] (NTT domain, [count][level+1][n]) *= s_ntt (limb stride n), then
// t[ct] += c0 of ct batch [count][2][level+1][n]
void mul_secret(const DevRing& R, u64* t, const u64* s_ntt, int level, std::size_t count, const Launch& L);
void add_c0(const DevRing& R, const u64* ct, u64* t, int level, std::size_t count, const Launch& L);

}  // namespace hecnn_b200
