// Device-resident CKKS engine: context (tables, keys, stream, memory),
// ciphertext tensors and the scheme / network operations built from the
// kernels in kernels.hpp. Host code here only orders kernels, keeps the
// scale/level ledger with the reference's exact double arithmetic and turns
// model weights into integer residues; no ciphertext word is computed on the
// CPU.
#pragma once
#include <cstddef>
#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "host_ckks.hpp"
#include "kernels.hpp"
#include "ring_host.hpp"

namespace hecnn_b200 {

struct Context;

// Caching device arena: segments from cudaMalloc (>= 1 GiB, kept until the
// context dies), sub-allocated best-fit with coalescing. All work of a context
// runs on its one stream, so a block freed on the host can be handed out again
// immediately: later kernels on that stream are ordered after earlier users.
// (cudaMallocAsync's pool re-mapped 17 GB tensors on some steps, costing
// 0.4-1.6 s per allocation.)
class Arena {
public:
    ~Arena();
    void* alloc(std::size_t bytes);
    void release(void* p);
    // Return segments that are entirely free to the driver; returns bytes freed.
    std::size_t trim();
    // Keep the first `bytes` of the used block at p, free the rest.
    void shrink(void* p, std::size_t bytes);
    std::size_t reserved() const { return reserved_; }
    std::size_t free_bytes() const {
        std::size_t b = 0;
        for (const auto& f : free_) b += f.second.size;
        return b;
    }

private:
    struct Block {
        std::size_t size;
        int seg;
    };
    std::vector<std::pair<char*, std::size_t>> segs_;
    std::map<char*, Block> free_, used_;
    std::size_t reserved_ = 0;
};

// Device allocation from the context's arena.
class DevBuf {
public:
    DevBuf() = default;
    DevBuf(Context* ctx, std::size_t bytes);
    ~DevBuf() { reset(); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept { *this = std::move(o); }
    DevBuf& operator=(DevBuf&& o) noexcept;
    void reset();
    // Non-owning view of memory owned elsewhere (e.g. a slice of a tensor).
    static DevBuf alias(void* ptr, std::size_t bytes);
    // Take ownership of an arena block allocated by the caller (released on reset).
    static DevBuf adopt(Context* ctx, void* ptr, std::size_t bytes);
    // Give up ownership without releasing (the caller keeps the block).
    void* release_ownership() {
        void* p = ptr_;
        ptr_ = nullptr;
        bytes_ = 0;
        ctx_ = nullptr;
        return p;
    }
    template <class T>
    T* as() const { return static_cast<T*>(ptr_); }
    void* get() const { return ptr_; }
    std::size_t bytes() const { return bytes_; }

private:
    Context* ctx_ = nullptr;
    void* ptr_ = nullptr;
    std::size_t bytes_ = 0;
};

struct Context {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    RingTables ring;
    std::unique_ptr<Encoder> enc;
    double scale = 0.0, sigma = 3.2;
    bool degenerate = false;
    DevRing dev;
    std::vector<DevBuf> tables;
    // keys (device resident; the secret also kept on the host for export)
    std::vector<u64> secret_host;  // [(L+1)][n] coefficient domain
    DevBuf s_ntt, pk, evk, evk_sh, evk_f;
    DevBuf aux_tab;  // limb 0's key switch through limbs 1..3 (keyswitch.cu), when the chain allows it
    void build_aux_tables();
    std::size_t evk_digits = 0;
    bool has_secret = false, has_pk = false;
    unsigned long long launches = 0;
    Profiler prof;
    Arena arena;

    cudaStream_t aux = nullptr;  // side stream (key switch: integer-limb kernel beside the FP64 one)
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;

    Context(std::size_t n, const std::vector<u64>& primes, double scale, double sigma, bool degenerate, int device);
    ~Context();
    Launch L() { return Launch{stream, &launches, &prof, aux, fork_ev, join_ev}; }
    std::size_t n() const { return ring.n; }
    std::size_t top() const { return ring.limbs - 1; }
    void upload(void* dst, const void* src, std::size_t bytes);
    void download(void* dst, const void* src, std::size_t bytes);
    void sync();
    template <class T>
    DevBuf upload_vec(const std::vector<T>& v) {
        DevBuf b(this, v.size() * sizeof(T));
        if (!v.empty()) upload(b.get(), v.data(), v.size() * sizeof(T));
        return b;
    }
};

struct Shape {
    bool flat = true;
    std::size_t h = 0, w = 0, c = 0, feat = 0;
    static Shape spatial(std::size_t h, std::size_t w, std::size_t c) { return {false, h, w, c, 0}; }
    static Shape flattened(std::size_t f) { return {true, 0, 0, 0, f}; }
    std::size_t positions() const { return flat ? feat : h * w * c; }
    Shape as_flat() const { return flattened(positions()); }
    bool operator==(const Shape& o) const {
        return flat == o.flat && (flat ? feat == o.feat : (h == o.h && w == o.w && c == o.c));
    }
    std::string str() const;
};

// A device batch of ciphertexts with one shared (scale, level):
// [cells][2][level+1][n] u64.
struct Tensor {
    Context* ctx = nullptr;
    DevBuf buf;
    std::size_t cells = 0;
    std::uint32_t level = 0;
    double scale = 0.0;
    Shape shape;
    std::size_t batch = 0;
    std::size_t cell_words() const { return 2 * (level + 1) * ctx->n(); }
    u64* data() const { return buf.as<u64>(); }
    u64* cell(std::size_t i) const { return data() + i * cell_words(); }
};
using TensorPtr = std::unique_ptr<Tensor>;

TensorPtr make_tensor(Context& C, std::size_t cells, std::uint32_t level, double scale);
// Integer-pipe peak: Shoup modmuls per second measured with CUDA events.
double measure_modmul_peak(Context& C, bool fp64 = false);

// ---- keys
void keygen(Context& C, u64 seed);
void import_keys(Context& C, const u64* secret, const u64* pk_b, const u64* pk_a, const u64* evk, std::size_t digits);

// ---- scheme ops (ckks.hpp)
TensorPtr ct_add(Context& C, const Tensor& x, const Tensor& y, bool subtract);
TensorPtr ct_mul(Context& C, const Tensor& x, const Tensor& y);
TensorPtr ct_square(Context& C, const Tensor& x);
TensorPtr ct_rescale(Context& C, const Tensor& x);
TensorPtr ct_mod_switch(Context& C, const Tensor& x, std::uint32_t to_level);
TensorPtr ct_mul_const(Context& C, const Tensor& x, double c, double scale);
TensorPtr ct_add_const(Context& C, const Tensor& x, double c);
// ---- the reference's scalar fast path and plaintext ops (ckks.hpp:283-311, 372-472),
// each applied to every cell of a tensor
struct ScalarPlain {  // CkksEngine::ScalarPlain (residues per active prime)
    std::vector<u64> residues;
    double scale = 0.0;
    std::uint32_t level = 0;
};
ScalarPlain make_scalar_plain(const Context& C, double c, double scale, std::size_t level);
TensorPtr ct_zero(Context& C, std::size_t cells, std::uint32_t level, double scale);
void ct_add_inplace(Context& C, Tensor& acc, const Tensor& x);
// acc += x * sp; residues [ncs][level+1] with ncs = 1 (every cell) or acc.cells (one scalar per cell)
void ct_scalar_mac(Context& C, Tensor& acc, const Tensor& x, const u64* residues, std::size_t ncs, double sp_scale,
                   std::uint32_t sp_level);
void ct_add_scalar(Context& C, Tensor& ct, double c);
// plaintext operand: a host polynomial [pt_level+1][n] in the coefficient domain
TensorPtr ct_add_plain(Context& C, const Tensor& x, const u64* pt, std::uint32_t pt_level, double pt_scale);
TensorPtr ct_mul_plain(Context& C, const Tensor& x, const u64* pt, std::uint32_t pt_level, double pt_scale,
                       bool is_constant, bool rescale);
// key_switch on raw d2 polys: out [count][2][level+1][n] NTT domain
void key_switch_raw(Context& C, const u64* d2, u64* out, std::size_t level, std::size_t count);

struct Activation {
    std::vector<double> coefficients;
    double interval_bound = 0.0;
    std::size_t degree() const { return coefficients.empty() ? 0 : coefficients.size() - 1; }
    std::size_t encrypted_depth() const;
    void validate() const;
};
// dst: optional device storage for the result cells (the returned tensor is then a view of it)
TensorPtr eval_activation(Context& C, const Activation& act, const Tensor& x, u64* dst = nullptr);

// ---- client side
TensorPtr encrypt_tensor(Context& C, const double* data, std::size_t batch, std::size_t positions, u64 seed);
TensorPtr encrypt_raw(Context& C, const u64* m, const long long* r, const long long* e0, const long long* e1,
                      std::size_t count, double scale);
void decrypt_raw(Context& C, const Tensor& t, u64* out_host);
void decrypt_tensor(Context& C, const Tensor& t, std::size_t batch, double* out);

// ---- network
struct Layer {
    int kind = 0;
    std::size_t filters = 0, kh = 0, kw = 0, stride = 1, pool = 0, pad = 0, units = 0;
    bool valid = false;
    int act = -1;
    std::vector<double> w, b;
    const char* kind_name() const;
};

struct StreamPlan;  // stream.cpp

struct Model {
    Shape input;
    std::vector<Layer> layers;
    std::vector<Activation> acts;
    std::vector<Shape> shapes;  // per-layer output shapes (shape_infer)
    // tap table of a conv / dense layer: the input cell each (pixel, tap) reads,
    // -1 for a clipped tap; src_pad is the same padded to whole 32-tap steps
    // (tensor-core paths). Pixels may be listed in any order.
    struct Taps {
        DevBuf src, src_pad;
        std::size_t pixels = 0;
    };
    // integer-weight caches, keyed by (layer, level) and (layer, level, scale)
    struct LinearCache {
        DevBuf weights, wsplit, recomb;
        int K = 0, oc = 0, oc_pad = 0;
        bool conv = false;
        // integer tensor-core path (limbs with q < 2^40): fragment-ordered weight
        // byte planes, 2^8s mod q table
        DevBuf wfrag, shift, wfrag_wide, shift_wide;
        DevBuf wtc, wtc_wide;  // tcgen05 weight tiles (conv_tc.cu), when the shape qualifies
        int kpad = 0, ksteps = 0, oc_tiles = 0;
        bool wide_ok = false;  // limbs with q >= 2^40 also on the tensor cores (signed weight digits)
        Taps taps;             // whole-tensor layout (built on first non-streamed use)
    };
    std::map<std::pair<std::size_t, std::uint32_t>, LinearCache> linear;
    std::map<std::tuple<std::size_t, std::uint32_t, double>, DevBuf> bias;
    std::map<std::pair<std::size_t, std::uint32_t>, DevBuf> pool_srcs;

    // Row-streamed execution of the spatial layers (stream.cpp) for tensors
    // that do not fit in device memory: 0 = only when the whole-tensor pass
    // does not fit, 1 = always (tests), 2 = never.
    int stream_mode = 0;
    std::size_t stream_tile = 0;  // stage-output columns per tile (0: sized to the budget)
    std::size_t mem_budget = 0;   // device bytes a forward pass may use (0: what is free)
    std::map<std::string, std::shared_ptr<StreamPlan>> plans;  // by segment, input level / scale, options

    void infer_shapes();
    std::size_t depth_cost() const;
};

TensorPtr forward_encrypted(Context& C, Model& M, const Tensor& x, u64 seed, double* layer_seconds);

}  // namespace hecnn_b200
