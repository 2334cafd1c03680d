"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck, one tool per run): the smoke C1 forward + HE square, the N = 2^13
and N = 2^14 key switch (both CTA groups, column stage), an 11x11 tcgen05
conv, and a row-streamed forward whose rings wrap. Exits 0 when every
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
