"""One HE square at C4's activation shape (net-n8192-d8, level 7, 512
ciphertexts of uniform residues) for ncu captures of k_keyswitch and the NTT
kernels. Not part of the bench contract."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1911_11377_b200 as hb
from tools.kbench import uniform_words

p = hb.preset_params(os.environ.get("KS_PRESET", "net-n8192-d8"))
lv = int(os.environ.get("KS_LEVEL", "7"))
cells = int(os.environ.get("KS_CELLS", "512"))
eng = hb.CkksEngine(p).keygen(1)
x = eng.tensor_from_words(uniform_words(p, cells, lv), lv, p.scale)
for _ in range(int(os.environ.get("KS_REPS", "2"))):
    y = eng.square(x)
eng.synchronize()
print("ok", y.level)
