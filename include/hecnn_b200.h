/*
 * hecnn_b200.h -- C-ABI of the B200-native CKKS evaluation engine.
 *
 * This is the drop-in boundary for the encrypted-CNN hot path of the
 * reference library `hecnn` (/root/reference/proj/include/hecnn, header-only
 * C++20). The reference has no FFI of its own: its public surface is the C++
 * API (`CkksEngine`, ring free functions, `forward_encrypted`). Every entry
 * point below names the reference interface it replaces (file:line relative
 * to proj/include/hecnn/). The C++ mirror in include/hecnn_b200/hecnn.hpp
 * re-exposes these entry points under the reference's own class names.
 *
 * Conventions
 *   - Plain pointers and sizes only; no C++ or torch types cross the ABI.
 *   - Every function returns an int status. On failure the thread-local
 *     message is available from hecnn_last_error(); HECNN_EINVAL maps to the
 *     reference's std::invalid_argument and HECNN_ERUNTIME to
 *     std::runtime_error, with the reference's message text.
 *   - Polynomials are limb-major: [limb 0..level][coefficient 0..n-1] u64,
 *     residues canonical in [0, q_i) (ring.hpp:239-253, RingPoly::rns).
 *   - A ciphertext is [c0 | c1] = [2][level+1][n]; a batch of `count`
 *     ciphertexts is [count][2][level+1][n]. Ciphertexts are always in the
 *     coefficient domain between operations (ckks.hpp:68-72).
 *   - One context per GPU. Work is issued on the context's stream (default:
 *     a stream created by the context; replace with hecnn_context_set_stream).
 *   - Ownership never crosses the ABI except via explicit create/destroy.
 */
#ifndef HECNN_B200_H
#define HECNN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HECNN_OK 0
#define HECNN_EINVAL 1   /* std::invalid_argument in the reference */
#define HECNN_ERUNTIME 2 /* std::runtime_error in the reference */
#define HECNN_ECUDA 3    /* CUDA failure (no reference analogue) */

typedef struct hecnn_context hecnn_context;
typedef struct hecnn_tensor hecnn_tensor;
typedef struct hecnn_model hecnn_model;

/* ---- errors / version ------------------------------------------------- */
const char* hecnn_last_error(void);
int hecnn_abi_version(void);

/* ---- parameters (host) -------------------------------------------------
 * RingParams::create (ring.hpp:20-30) + find_ntt_primes (common.hpp:146-162):
 * for each entry of prime_bits, the largest prime p < 2^bits with
 * p == 1 (mod 2n) not already taken. */
int hecnn_find_chain(size_t n, const int* prime_bits, size_t count, uint64_t* primes_out);

/* ---- host-only numerics (no device needed) -----------------------------
 * encode_real (ckks.hpp:105-129): residues [(level+1)][n] of the encoding. */
int hecnn_host_encode_real(size_t n, const uint64_t* primes, size_t nprimes, const double* values, size_t len,
                           double scale, size_t level, uint64_t* out);
/* decode (ckks.hpp:142-154): real parts of the first `count` slots. */
int hecnn_host_decode_real(size_t n, const uint64_t* primes, size_t nprimes, const uint64_t* poly, size_t level,
                           double scale, double* out, size_t count);
/* make_encryption_randomness (ckks.hpp:238-244): signed coefficients [n]. */
int hecnn_host_encryption_randomness(size_t n, double sigma, int degenerate_noise, uint64_t seed, int64_t* r,
                                     int64_t* e0, int64_t* e1);

/* ---- context: RingContext (ring.hpp:171-237) + CkksEngine ctor
 * (ckks.hpp:79-93). Builds NTT/CRT/rescale tables on the host and uploads
 * them to `device`. */
int hecnn_context_create(size_t n, const uint64_t* primes, size_t nprimes, double scale, double sigma,
                         int degenerate_noise, int device, hecnn_context** out);
int hecnn_context_destroy(hecnn_context* ctx);
int hecnn_context_set_stream(hecnn_context* ctx, void* cuda_stream);
int hecnn_context_synchronize(hecnn_context* ctx);
/* Return the device arena's wholly free segments to the driver. */
int hecnn_context_trim(hecnn_context* ctx, size_t* freed_bytes);
int hecnn_context_info(const hecnn_context* ctx, size_t* n, size_t* top_level, double* scale);
/* CkksEngine::relin_digits (ckks.hpp:509-512) */
int hecnn_relin_digits(const hecnn_context* ctx, size_t level, size_t* digits);
/* Number of kernel launches issued by this context since creation. */
int hecnn_launch_count(const hecnn_context* ctx, uint64_t* launches);

/* ---- measurement (no reference analogue) ------------------------------
 * Per-kernel timing with CUDA events on the context stream (enabled region
 * only); read returns JSON {"kernel": {"ms": total, "launches": k}, ...}. */
int hecnn_profile_enable(hecnn_context* ctx, int on);
int hecnn_profile_reset(hecnn_context* ctx);
int hecnn_profile_read(hecnn_context* ctx, char* buf, size_t len);
/* Integer-pipe roofline probe: chained 64-bit Shoup modular multiplies/s. */
int hecnn_modmul_peak(hecnn_context* ctx, double* modmul_per_s);
/* FP64-pipe roofline probe: chained exact FP64 modular multiplies/s (the
 * arithmetic the NTT/key-switch kernels use for primes below 2^42). */
int hecnn_fp64_modmul_peak(hecnn_context* ctx, double* modmul_per_s);

/* ---- keys: CkksEngine::keygen (ckks.hpp:200-236). Randomness is sampled on
 * the host (mt19937_64 + libm, bit-identical to the reference); NTTs and
 * pointwise work run on the device. Keys stay resident on the device. */
int hecnn_keygen(hecnn_context* ctx, uint64_t seed);
/* Import keys produced elsewhere (e.g. by the reference): secret key in
 * coefficient domain [(L+1)][n]; pk (b,a) NTT domain [(L+1)][n] each;
 * evk [digits][2 (b,a)][(L+1)][n] NTT domain. */
int hecnn_import_keys(hecnn_context* ctx, const uint64_t* secret, const uint64_t* pk_b, const uint64_t* pk_a,
                      const uint64_t* evk, size_t evk_digits);
int hecnn_export_secret_key(const hecnn_context* ctx, uint64_t* secret);
int hecnn_export_public_key(const hecnn_context* ctx, uint64_t* pk_b, uint64_t* pk_a);
int hecnn_eval_key_digits(const hecnn_context* ctx, size_t* digits);
int hecnn_export_eval_key(const hecnn_context* ctx, uint64_t* evk);

/* ---- raw device memory ------------------------------------------------- */
int hecnn_device_alloc(hecnn_context* ctx, size_t bytes, void** dptr);
int hecnn_device_free(hecnn_context* ctx, void* dptr);
int hecnn_memcpy_h2d(hecnn_context* ctx, void* dst, const void* src, size_t bytes);
int hecnn_memcpy_d2h(hecnn_context* ctx, void* dst, const void* src, size_t bytes);

/* ---- ring tier on raw device pointers ([count][level+1][n] u64) -------- */
/* NttTables::forward / ntt_transform (ring.hpp:83-108, :326-342) */
int hecnn_ntt_forward(hecnn_context* ctx, uint64_t* polys, size_t level, size_t count);
/* NttTables::inverse (ring.hpp:110-137) */
int hecnn_ntt_inverse(hecnn_context* ctx, uint64_t* polys, size_t level, size_t count);
/* poly_add / poly_sub / poly_neg (ring.hpp:291-322) */
int hecnn_poly_add(hecnn_context* ctx, const uint64_t* a, const uint64_t* b, uint64_t* out, size_t level,
                   size_t count);
int hecnn_poly_sub(hecnn_context* ctx, const uint64_t* a, const uint64_t* b, uint64_t* out, size_t level,
                   size_t count);
int hecnn_poly_neg(hecnn_context* ctx, const uint64_t* a, uint64_t* out, size_t level, size_t count);
/* poly_pointwise_mul / poly_pointwise_mac (ring.hpp:345-370) */
int hecnn_poly_pointwise_mul(hecnn_context* ctx, const uint64_t* a, const uint64_t* b, uint64_t* out,
                             size_t level, size_t count);
int hecnn_poly_pointwise_mac(hecnn_context* ctx, uint64_t* acc, const uint64_t* a, const uint64_t* b,
                             size_t level, size_t count);
/* rescale_poly (ring.hpp:419-442): in [count][level+1][n] -> out [count][level][n] */
int hecnn_rescale_poly(hecnn_context* ctx, const uint64_t* in, uint64_t* out, size_t level, size_t count);
/* key_switch (ckks.hpp:601-630) on a batch of d2 polys (coefficient domain,
 * [count][level+1][n]); writes (acc0, acc1) NTT domain as [count][2][level+1][n]. */
int hecnn_key_switch(hecnn_context* ctx, const uint64_t* d2, uint64_t* out, size_t level, size_t count);

/* ---- encrypted tensors: a device batch of ciphertexts with one shared
 * (scale, level), i.e. TensorEncrypted (tensor.hpp:61-75) / a single
 * Ciphertext when cells == 1. ------------------------------------------- */
int hecnn_tensor_create(hecnn_context* ctx, size_t cells, uint32_t level, double scale, hecnn_tensor** out);
int hecnn_tensor_destroy(hecnn_tensor* t);
int hecnn_tensor_info(const hecnn_tensor* t, size_t* cells, uint32_t* level, double* scale);
int hecnn_tensor_set_shape(hecnn_tensor* t, int flat, size_t h, size_t w, size_t c, size_t batch);
int hecnn_tensor_shape(const hecnn_tensor* t, int* flat, size_t* h, size_t* w, size_t* c, size_t* batch);
/* device pointer of the [cells][2][level+1][n] buffer */
int hecnn_tensor_data(const hecnn_tensor* t, uint64_t** dptr);
int hecnn_tensor_upload(hecnn_context* ctx, hecnn_tensor* t, const uint64_t* host);
int hecnn_tensor_download(hecnn_context* ctx, const hecnn_tensor* t, uint64_t* host);
/* Asynchronous variants for pipelined serving: the copy is enqueued on `stream`
 * (a cudaStream_t; NULL = the context's stream) and the call returns at once.
 * `host` must be pinned and stay valid until the stream reaches the copy; the
 * caller orders the copy against the context's work with CUDA events. */
int hecnn_tensor_upload_async(hecnn_context* ctx, hecnn_tensor* t, const uint64_t* host, void* stream);
int hecnn_tensor_download_async(hecnn_context* ctx, const hecnn_tensor* t, uint64_t* host, void* stream);
/* device-to-device copy of the words (e.g. into an NCCL buffer) */
int hecnn_tensor_copy_to_device(hecnn_context* ctx, const hecnn_tensor* t, void* dst);

/* encrypt_tensor (tensor.hpp:77-94): data is [batch][positions] (TensorPlain
 * layout). Encode on the host (ckks.hpp:105-123), randomness on the host
 * (derive_seed(seed, 0xce11 + pos)), public-key encryption on the device. */
int hecnn_encrypt_tensor(hecnn_context* ctx, const double* data, size_t batch, size_t positions, uint64_t seed,
                         hecnn_tensor** out);
/* CkksEngine::encrypt with explicit randomness (ckks.hpp:249-266): plaintext
 * polys [count][(L+1)][n] coefficient domain at the top level; r, e0, e1
 * small signed coefficients [count][n]. */
int hecnn_encrypt_raw(hecnn_context* ctx, const uint64_t* m, const int64_t* r, const int64_t* e0,
                      const int64_t* e1, size_t count, double scale, hecnn_tensor** out);
/* decrypt (ckks.hpp:273-279) on the device: out [cells][level+1][n] */
int hecnn_decrypt_raw(hecnn_context* ctx, const hecnn_tensor* t, uint64_t* out_host);
/* decrypt_tensor (tensor.hpp:96-106): out [batch][positions] real parts */
int hecnn_decrypt_tensor(hecnn_context* ctx, const hecnn_tensor* t, size_t batch, double* out);

/* ---- scheme tier on tensors (cellwise) ---------------------------------- */
int hecnn_ct_add(hecnn_context* ctx, const hecnn_tensor* x, const hecnn_tensor* y, hecnn_tensor** out);
int hecnn_ct_sub(hecnn_context* ctx, const hecnn_tensor* x, const hecnn_tensor* y, hecnn_tensor** out);
/* CkksEngine::mul (ckks.hpp:315-342): tensor, relinearize, rescale */
int hecnn_ct_mul(hecnn_context* ctx, const hecnn_tensor* x, const hecnn_tensor* y, hecnn_tensor** out);
/* CkksEngine::square (ckks.hpp:345-369) */
int hecnn_ct_square(hecnn_context* ctx, const hecnn_tensor* x, hecnn_tensor** out);
/* CkksEngine::rescale / mod_switch (ckks.hpp:474-493) */
int hecnn_ct_rescale(hecnn_context* ctx, const hecnn_tensor* x, hecnn_tensor** out);
int hecnn_ct_mod_switch(hecnn_context* ctx, const hecnn_tensor* x, uint32_t to_level, hecnn_tensor** out);
/* mul_plain(x, encode_const(c, scale, x.level)) (ckks.hpp:372-398, :132-140) */
int hecnn_ct_mul_const(hecnn_context* ctx, const hecnn_tensor* x, double c, double scale, hecnn_tensor** out);
/* add_plain(x, encode_const(c, x.scale, x.level)) (ckks.hpp:305-311) */
int hecnn_ct_add_const(hecnn_context* ctx, const hecnn_tensor* x, double c, hecnn_tensor** out);
/* ---- scalar fast path and plaintext operands (ckks.hpp:283-311, 372-472) --
 * CkksEngine's per-ciphertext helpers, applied to every cell of a tensor.
 * In-place functions modify `acc` / `ct`. Errors carry the reference's texts
 * ("mul_scalar_mac: level mismatch", "add_plain: level mismatch", ...). */
/* make_scalar_plain (:407-423): residues_out[level+1] = round(c * scale) mod q_i */
int hecnn_make_scalar_plain(hecnn_context* ctx, double c, double scale, size_t level, uint64_t* residues_out);
/* make_zero_ciphertext (:431-438): `cells` zero ciphertexts at (level, scale) */
int hecnn_ct_zero(hecnn_context* ctx, size_t cells, uint32_t level, double scale, hecnn_tensor** out);
/* add_inplace (:440-445): acc += x */
int hecnn_ct_add_inplace(hecnn_context* ctx, hecnn_tensor* acc, const hecnn_tensor* x);
/* mul_scalar_mac (:448-465): acc += x * sp, residues [ncs][sp_level+1] from
 * hecnn_make_scalar_plain; ncs = 1 (one scalar for every cell) or the cell count */
int hecnn_ct_scalar_mac(hecnn_context* ctx, hecnn_tensor* acc, const hecnn_tensor* x, const uint64_t* residues,
                        size_t ncs, double sp_scale, uint32_t sp_level);
/* add_scalar_inplace (:468-472): ct += c, encoded at ct's own scale */
int hecnn_ct_add_scalar(hecnn_context* ctx, hecnn_tensor* ct, double c);
/* add_plain (:305-311), mul_plain_raw / mul_plain (:372-398) with one plaintext
 * polynomial pt (host, [pt_level+1][n], coefficient domain) for every cell;
 * is_constant: pt is a constant polynomial (encode_const), multiplied as a
 * scalar; rescale != 0: mul_plain, else mul_plain_raw */
int hecnn_ct_add_plain(hecnn_context* ctx, const hecnn_tensor* x, const uint64_t* pt, uint32_t pt_level,
                       double pt_scale, hecnn_tensor** out);
int hecnn_ct_mul_plain(hecnn_context* ctx, const hecnn_tensor* x, const uint64_t* pt, uint32_t pt_level,
                       double pt_scale, int is_constant, int rescale, hecnn_tensor** out);

/* eval_encrypted (activation.hpp:228-265) on every cell */
int hecnn_eval_activation(hecnn_context* ctx, const double* coefficients, size_t n_coefficients,
                          double interval_bound, const hecnn_tensor* x, hecnn_tensor** out);

/* ---- wire format: CKKS blob v1 (ckks_serialize.hpp:3-152) ----------------
 * Blobs are byte-identical to the reference's save_* output, so keys and
 * ciphertexts move between the CPU reference and this engine as files.
 * Save functions write into `buf` (`cap` bytes) and set *len to the blob
 * size; buf == NULL only queries the size. Load functions require the blob's
 * parameters to equal the context's (same_params, :145-148). Errors carry the
 * reference's texts ("ckks blob: bad magic", "ckks blob: wrong object kind",
 * "io: unexpected end of file", ... -> HECNN_ERUNTIME). */
enum { HECNN_BLOB_SECRET_KEY = 1, HECNN_BLOB_PUBLIC_KEY = 2, HECNN_BLOB_EVAL_KEY = 3, HECNN_BLOB_CIPHERTEXT = 4 };
/* read_header (:41-58) without a context: the kind is read from the blob;
 * primes (capacity *nprimes, may be NULL) and *nprimes = chain length */
int hecnn_blob_params(const uint8_t* blob, size_t len, int* kind, size_t* n, uint64_t* primes, size_t* nprimes,
                      double* scale, double* sigma, int* degenerate);
/* save_secret_key / save_public_key / save_evaluation_key (:79-114) of the
 * context's keys, kind = HECNN_BLOB_*_KEY */
int hecnn_blob_save_key(const hecnn_context* ctx, int kind, uint8_t* buf, size_t cap, size_t* len);
/* load_*_key (:84-122) into the context (any of the three kinds, by `kind`) */
int hecnn_blob_load_key(hecnn_context* ctx, int kind, const uint8_t* blob, size_t len);
/* save_ciphertext (:124-130) of cell `cell` of a tensor */
int hecnn_blob_save_ciphertext(hecnn_context* ctx, const hecnn_tensor* t, size_t cell, uint8_t* buf, size_t cap,
                               size_t* len);
/* load_ciphertext (:133-141) of `count` blobs into one tensor of `count`
 * cells (TensorEncrypted's uniform level and scale, tensor.hpp:52-62) */
int hecnn_blob_load_ciphertexts(hecnn_context* ctx, const uint8_t* const* blobs, const size_t* lens, size_t count,
                                hecnn_tensor** out);

/* ---- network tier ------------------------------------------------------- */
enum {
    HECNN_LAYER_CONV2D = 0,
    HECNN_LAYER_AVG_POOL2D = 1,
    HECNN_LAYER_ZERO_PAD2D = 2,
    HECNN_LAYER_DENSE = 3,
    HECNN_LAYER_ACTIVATION = 4,
    HECNN_LAYER_SIGMOID = 5
};

/* LayerSpec (model.hpp:12-76) */
typedef struct hecnn_layer_desc {
    int32_t kind;
    int32_t filters, kernel_h, kernel_w, stride;
    int32_t padding_valid; /* 0 = Same, 1 = Valid */
    int32_t pool, pad, units;
    int32_t activation; /* index into hecnn_model_desc.activations */
    const double* weights;
    size_t n_weights;
    const double* biases;
    size_t n_biases;
} hecnn_layer_desc;

/* PolyActivation (activation.hpp:24-45) */
typedef struct hecnn_activation_desc {
    const double* coefficients; /* ascending degree */
    size_t n_coefficients;
    double interval_bound;
} hecnn_activation_desc;

/* ModelSpec (model.hpp:78-97) */
typedef struct hecnn_model_desc {
    int32_t input_flat;
    size_t input_h, input_w, input_c, input_features;
    const hecnn_layer_desc* layers;
    size_t n_layers;
    const hecnn_activation_desc* activations;
    size_t n_activations;
} hecnn_model_desc;

/* Validates the model (shape_infer, model.hpp:145-157) and keeps a copy. */
int hecnn_model_create(hecnn_context* ctx, const hecnn_model_desc* desc, hecnn_model** out);
int hecnn_model_destroy(hecnn_model* m);
/* depth_cost (model.hpp:169-182) */
int hecnn_model_depth_cost(const hecnn_model* m, size_t* cost);
/* Execution of the spatial layers when their tensors exceed device memory
 * (no reference counterpart: the reference materialises every layer tensor,
 * layers.hpp:299-368). mode 0: row-stream only the layers whose whole
 * tensors do not fit (default); 1: row-stream every spatial stage; 2: never.
 * tile: stage-output columns per tile (0: sized to the memory budget);
 * mem_budget: device bytes a forward pass may plan with (0: free memory).
 * Results are identical word for word in every mode. */
int hecnn_model_set_streaming(hecnn_model* m, int mode, size_t tile, size_t mem_budget);
/* forward_encrypted (layers.hpp:299-368). x must carry the model's input
 * shape (hecnn_tensor_set_shape). layer_seconds (optional) receives one
 * device-timed entry per layer. */
int hecnn_forward_encrypted(hecnn_context* ctx, const hecnn_model* m, const hecnn_tensor* x, uint64_t seed,
                            hecnn_tensor** out, double* layer_seconds);

#ifdef __cplusplus
}
#endif
#endif /* HECNN_B200_H */
