// The reference's sample flow (proj/samples/encrypted_inference.cpp and
// roundtrip.cpp) compiled against the drop-in header instead of the
// reference: same names, same call sites. Writes the encrypted logits'
// ciphertext words and the decrypted logits for tests/test_gpu_dropin.py.
#include <cstdio>
#include <fstream>

#include "hecnn_b200/hecnn.hpp"

using namespace hecnn;

int main(int argc, char** argv) {
    if (argc < 3) return 2;
    CkksParams params = preset_params("nn-n4096-d8");
    CkksEngine engine(params);
    KeySet keys = engine.keygen(7);
    EvalKeys eval_keys{keys.public_key, keys.eval};

    // roundtrip.cpp: encode -> encrypt -> square -> decrypt
    std::vector<double> v = {0.5, -0.25, 0.125, 1.0};
    Ciphertext ct = engine.encrypt(keys.public_key, engine.encode_real(v, params.scale, engine.top_level()), 3);
    Ciphertext sq = engine.square(ct, keys.eval);
    PlaintextVector dec = engine.decode(engine.decrypt(keys.secret, sq));
    for (std::size_t i = 0; i < v.size(); ++i) std::printf("square %zu: %.8f (want %.8f)\n", i, dec[i].real(), v[i] * v[i]);

    // encrypted_inference.cpp: tiny_preset over an encrypted batch
    ModelSpec model = tiny_preset();
    std::ifstream wf(argv[1], std::ios::binary);  // weights/biases/inputs from the test (reference-generated)
    auto read_vec = [&](std::vector<double>& out) {
        std::uint64_t count = 0;
        wf.read(reinterpret_cast<char*>(&count), 8);
        out.resize(count);
        wf.read(reinterpret_cast<char*>(out.data()), static_cast<std::streamsize>(count * 8));
    };
    read_vec(model.weights[0]);
    read_vec(model.biases[0]);
    read_vec(model.weights[3]);
    read_vec(model.biases[3]);
    TensorPlain batch{model.input, 4, {}};
    read_vec(batch.data);

    TensorEncrypted enc = encrypt_tensor(engine, keys.public_key, batch, 11);
    std::vector<double> secs;
    TensorEncrypted out = forward_encrypted(model, enc, engine, eval_keys, 13, 1, &secs);
    TensorPlain logits = decrypt_tensor(engine, keys.secret, out);
    std::ofstream of(argv[2], std::ios::binary);
    const Ciphertext& o = out.cells[0];
    std::uint32_t lvl = o.level;
    of.write(reinterpret_cast<const char*>(&lvl), 4);
    of.write(reinterpret_cast<const char*>(&o.scale), 8);
    for (const auto* poly : {&o.c0, &o.c1})
        for (const auto& row : poly->rns) of.write(reinterpret_cast<const char*>(row.data()), row.size() * 8);
    of.write(reinterpret_cast<const char*>(logits.data.data()), logits.data.size() * 8);
    // ckks_serialize.hpp: the logits ciphertext and the evaluation key as blobs
    if (argc >= 4) {
        std::ofstream bf(argv[3], std::ios::binary);
        save_ciphertext(bf, params, o);
        save_evaluation_key(bf, params, keys.eval);
    }
    for (std::size_t i = 0; i < logits.batch; ++i) std::printf("image %zu logit %.8f\n", i, logits.at(i, 0));
    std::printf("layers: %zu timed\n", secs.size());
    return 0;
}
