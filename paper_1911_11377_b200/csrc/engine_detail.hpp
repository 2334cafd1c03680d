// Engine internals shared by engine.cpp and stream.cpp (not part of the C-ABI).
#pragma once
#include <cstddef>
#include <cstdint>
#include <future>
#include <map>
#include <memory>
#include <vector>

#include "engine.hpp"

namespace hecnn_b200::detail {

// Scratch budget per batched scheme op; chunks of ciphertexts are sized to it.
constexpr std::size_t kScratchBytes = std::size_t(3) << 30;

// Public-key encryptions of `count` messages (or zeros, msgs == nullptr) at
// limbs 0..level with the randomness of make_encryption_randomness(seeds[i])
// (ckks.hpp:238-266); out: [count][2][level+1][n] device words.
void encrypt_into(Context& C, std::size_t count, const u64* seeds, const std::vector<EncodedCoeffs>* msgs,
                  std::uint32_t level, u64* out);

// Device part of encrypt_into with host-sampled randomness: r, e0, e1 are
// [count][n] int8 (ternary / clamped gaussian), messages zero.
void encrypt_sampled(Context& C, std::size_t count, const signed char* r, const signed char* e0, const signed char* e1,
                     std::uint32_t level, u64* out);

// zero_pad2d border randomness (layers.hpp:255-262), sampled on host threads
// while the device runs the layers before the pad: make_encryption_randomness
// (derive_seed(layer_seed, 0xbad0 + p)) for every border position p.
struct PadNoise {
    std::vector<int> border;             // position -> border index (-1: inside)
    std::vector<signed char> r, e0, e1;  // [borders][n]
};
using PadNoiseFuture = std::shared_future<std::shared_ptr<const PadNoise>>;
using PadNoiseMap = std::map<std::size_t, PadNoiseFuture>;  // by pad layer
PadNoiseMap start_pad_noise(Context& C, const Model& M, u64 seed);

// Conv / dense weight caches of layer li at `level` (rows = taps x in_c, or in_f).
Model::LinearCache& linear_weights(Context& C, Model& M, std::size_t li, std::uint32_t level, std::size_t rows);
// Device tap table from src [pixels][K] (input cell per tap, -1 clipped).
Model::Taps make_taps(Context& C, const Model::LinearCache& lc, const std::vector<int>& src);
// Same-padding offsets of a conv (ConvGeom, layers.hpp:24-50).
void conv_offsets(const Layer& l, std::size_t in_h, std::size_t in_w, std::size_t out_h, std::size_t out_w,
                  long long& pad_top, long long& pad_left);
// Bias residues [oc][level+1] at the accumulator scale x.scale * Delta.
const u64* linear_bias(Context& C, Model& M, std::size_t li, std::uint32_t level, double acc_scale);
// MAC + bias + rescale of pixels [p0, p0 + m) of `taps` over input cells at x
// (all at `level`); writes [m][oc] cells at level - 1 to out.
void linear_apply(Context& C, Model::LinearCache& lc, const Model::Taps& taps, const u64* bias, const u64* x,
                  std::uint32_t level, std::size_t p0, std::size_t m, u64* out);

// Row-streamed forward over layers [first, end) (stream.cpp): returns the
// output tensor of layer end - 1, or null when the plan decides the
// whole-tensor pass fits (the caller then runs layers one by one).
// `end` is filled with the first layer not covered.
// layer_ms (optional, one entry per layer): device milliseconds are added per layer.
TensorPtr forward_streamed(Context& C, Model& M, const Tensor& x, std::size_t first, std::size_t& end, u64 seed,
                           std::vector<double>* layer_ms, const PadNoiseMap& pads);

}  // namespace hecnn_b200::detail
