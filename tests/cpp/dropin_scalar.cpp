// A hand-written layer kernel against the drop-in header, the way the
// reference's conv/dense kernels (layers.hpp:174-293) use CkksEngine's scalar
// fast path: zero accumulator -> mul_scalar_mac per input -> bias ->
// rescale, then mul_plain / add_plain with encoded plaintexts. Writes the
// result words for tests/test_gpu_dropin.py to compare with the reference.
#include <cstdio>
#include <fstream>

#include "hecnn_b200/hecnn.hpp"

using namespace hecnn;

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    CkksParams params = preset_params("nn-n4096-d8");
    CkksEngine eng(params);
    KeySet keys = eng.keygen(1);
    const std::size_t top = eng.top_level();
    std::vector<double> v = {0.5, -0.25, 0.125, 1.0}, u = {-0.75, 0.5, 0.25, -0.125};
    Ciphertext x = eng.encrypt(keys.public_key, eng.encode_real(v, params.scale, top), 21);
    Ciphertext y = eng.encrypt(keys.public_key, eng.encode_real(u, params.scale, top), 22);

    Ciphertext acc = eng.make_zero_ciphertext(top, x.scale * params.scale);
    eng.mul_scalar_mac(acc, x, eng.make_scalar_plain(0.3, params.scale, top));
    eng.mul_scalar_mac(acc, y, eng.make_scalar_plain(-1.25, params.scale, top));
    eng.add_scalar_inplace(acc, 0.0625);
    Ciphertext z = eng.rescale(acc);  // 0.3 v - 1.25 u + 0.0625
    Ciphertext w = eng.mul_plain(z, eng.encode_const(0.5, params.scale, z.level));
    Ciphertext s = eng.add_plain(w, eng.encode_real(v, w.scale, w.level));
    eng.add_inplace(s, s);

    PlaintextVector dec = eng.decode(eng.decrypt(keys.secret, s));
    for (std::size_t i = 0; i < v.size(); ++i) {
        const double want = 2.0 * (0.5 * (0.3 * v[i] - 1.25 * u[i] + 0.0625) + v[i]);
        std::printf("slot %zu: %.8f (want %.8f)\n", i, dec[i].real(), want);
    }
    std::ofstream of(argv[1], std::ios::binary);
    std::uint32_t lvl = s.level;
    of.write(reinterpret_cast<const char*>(&lvl), 4);
    of.write(reinterpret_cast<const char*>(&s.scale), 8);
    for (const auto* poly : {&s.c0, &s.c1})
        for (const auto& row : poly->rns) of.write(reinterpret_cast<const char*>(row.data()), row.size() * 8);
    return 0;
}
