"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck, one tool per run): the smoke C1 forward + HE square, the N = 2^13
and N = 2^14 key switch (limb 0 through limbs 1..3, column stage), the raw key
switch, a fused degree-2 activation, the scalar / plaintext ops, an 11x11
tcgen05 conv, and a row-streamed forward whose rings wrap. Exits 0 when every
result still matches (sanitizer output is checked by the caller)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import __graft_entry__ as g
import paper_1911_11377_b200 as hb
from tools.kbench import uniform_words

g.smoke()
for preset, lv, cells in (("net-n8192-d8", 7, 3), ("large-n16384-d24", 4, 2)):
    p = hb.preset_params(preset)
    e = hb.CkksEngine(p).keygen(1)
    x = e.tensor_from_words(uniform_words(p, cells, lv), lv, p.scale)
    a = e.square(x).words()
    b = e.mul(x, x).words()
    assert np.array_equal(a, b), "square != mul(x, x)"
    print(preset, "square == mul(x, x)", flush=True)

# raw key switch (NTT-domain output: the aux route's CRT + forward NTT mod q0 and combine),
# a degree-2 activation (its linear term fused into the last rescale), the scalar fast path
p = hb.preset_params("net-n8192-d8")
e = hb.CkksEngine(p).keygen(1)
d2 = uniform_words(p, 2, 5)[:, 0]
ks = e.key_switch(d2, 5)
act = e.eval_activation(hb.relu_default_surrogate(), e.tensor_from_words(uniform_words(p, 3, 6), 6, p.scale))
x = e.tensor_from_words(uniform_words(p, 3, 6), 6, p.scale)
acc = e.make_zero_ciphertext(6, p.scale * p.scale, 3)
e.mul_scalar_mac(acc, x, [e.make_scalar_plain(w, p.scale, 6) for w in (0.5, -0.25, 1.0)])
e.add_scalar_inplace(acc, 0.125)
m = e.mul_plain(x, e.encode_real(np.linspace(-1, 1, 16), 2.0 ** 30, 6))
a2 = e.add_plain(x, e.encode_const(0.5, p.scale, 6))
print("key switch / activation / scalar ops ok", ks.shape, act.level, m.level, flush=True)

p = hb.preset_params("net-n8192-d8")
e = hb.CkksEngine(p).keygen(2)
spec = hb.ModelSpec(hb.Shape.spatial(4, 4, 3))
spec.layers = [hb.LayerSpec.conv2d(8, 11, 11)]
spec = hb.glorot_weights(spec, 3)
data = np.random.default_rng(1).uniform(0, 1, size=(16, spec.input.positions()))
x = e.encrypt_tensor(data, seed=5, shape=spec.input)
e.profile_reset()
e.profile(True)
y1 = hb.forward_encrypted(spec, x, e, seed=7)
e.synchronize()
e.profile(False)
assert "k_conv_tc" in e.profile_read(), "tcgen05 conv did not run"
print("tcgen05 conv ok", flush=True)

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_stream import tall_params, tall_spec  # noqa: E402
p = tall_params()
spec = tall_spec()
e = hb.CkksEngine(p).keygen(2)
data = np.random.default_rng(17).uniform(0, 1, size=(64, spec.input.positions()))
x = e.encrypt_tensor(data, seed=31, shape=spec.input)
w = hb.forward_encrypted(e.model(spec).set_streaming(hb.Model.STREAM_NEVER), x, e, seed=41)
s = hb.forward_encrypted(e.model(spec).set_streaming(hb.Model.STREAM_ALWAYS, tile=1), x, e, seed=41)
assert np.array_equal(w.words(), s.words()), "streamed != whole"
print("streamed forward ok", flush=True)
print("SANITIZE_RUN_OK")
