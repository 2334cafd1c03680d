#!/usr/bin/env python
"""SURVEY §8(d) C2 sweep (one GPU): NTT/INTT and ciphertext mul + relinearize
+ rescale throughput for N = 2^12 .. 2^16, chain [60, 40 x 8] (level 8), on the
device (1024 ciphertexts of uniform residues per N, bench.microbench) and on
the reference CPU path beside it (oracle/_ref, all host threads through its
parallel_for, a bounded sample of the same ops). Prints one JSON object."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1911_11377_b200 as hb  # noqa: E402
from oracle import ref  # noqa: E402


def main():
    import torch
    torch.cuda.set_device(0)
    threads = os.cpu_count() or 1
    out = {"chain": "[60,40x8]", "level": 8, "threads": threads, "rows": []}
    for logn in range(12, 17):
        n = 1 << logn
        dev = bench.microbench(hb, 0, n=n, count=1024)
        p = hb.CkksParams(n, hb.find_chain(n, [60] + [40] * 8), 2.0 ** 40)
        r = ref.RefEngine.from_params(p).keygen(1)
        k_ntt = max(threads, (1 << 20) // n * threads // 16)
        k_mul = max(threads, 2 * threads * 4096 // n)
        t_ntt = r.time_ntt(8, k_ntt, threads)
        t_mul = r.time_mul(8, k_mul, threads)
        row = {"n": n, "gpu_ntt_ops_per_s": dev["ntt_ops_per_s"], "gpu_he_mul_ops_per_s": dev["he_mul_ops_per_s"],
               "cpu_ntt_ops_per_s": k_ntt * 2 * 9 / t_ntt, "cpu_he_mul_ops_per_s": k_mul / t_mul,
               "cpu_sample": f"{k_ntt} polys x 9 limbs fwd+inv, {k_mul} muls"}
        out["rows"].append(row)
        print(json.dumps(row), file=sys.stderr, flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
