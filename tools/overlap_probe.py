"""Upper bound on cross-kernel overlap: two engines square independent
ciphertext batches (net-n8192-d8, level 7, 1024 each) on two streams from two
host threads, against one engine doing both batches back to back. Measured
0.972 (2.8%): the persistent key switch holds every SM, and the kernels around
it are not complementary enough to gain from sharing SMs. Not part of the bench."""
import sys, os, time, threading
sys.path.insert(0, os.getcwd())
import torch
import paper_1911_11377_b200 as hb
from tools.kbench import uniform_words
p = hb.preset_params("net-n8192-d8")
engs, xs, streams = [], [], []
for k in range(2):
    e = hb.CkksEngine(p).keygen(1)
    s = torch.cuda.Stream()
    e.set_stream(s.cuda_stream)
    engs.append(e); streams.append(s)
    xs.append(e.tensor_from_words(uniform_words(p, 1024, 7, seed=5 + k), 7, p.scale))
REPS = 4
def run(k, reps):
    for _ in range(reps):
        y = engs[k].square(xs[k])
    engs[k].synchronize()
for k in range(2): run(k, 1)
torch.cuda.synchronize()
t0 = time.perf_counter(); run(0, 2 * REPS); torch.cuda.synchronize(); seq = time.perf_counter() - t0
t0 = time.perf_counter()
th = [threading.Thread(target=run, args=(k, REPS)) for k in range(2)]
[t.start() for t in th]; [t.join() for t in th]
torch.cuda.synchronize(); par = time.perf_counter() - t0
print(f"sequential {seq*1e3:.1f} ms, two streams {par*1e3:.1f} ms, ratio {par/seq:.3f}")
