"""Host-side checks of the measurement method in bench.py (no GPU): the
per-layer work counts used to extrapolate crop timings to the full input
(the C5 method, validated on C4 by bench.py's method_check_on_c4) follow the
reference's loops -- conv: output pixels x valid taps x filters
(layers.hpp:174-211 skips clipped taps), activation / pool: output cells,
zero-pad: new border cells, dense: inputs x units."""
import bench
import paper_1911_11377_b200 as hb


def _valid_taps(n, k):
    # same padding, stride 1: taps of a k-wide window inside [0, n)
    pad = (n - 1 + k - n) // 2
    return sum(sum(1 for kk in range(k) if 0 <= o + kk - pad < n) for o in range(n))


def test_layer_work_c4():
    spec = bench.c4_spec(hb, 32)
    w = bench.layer_work(hb, spec)
    assert w[0] == _valid_taps(32, 3) ** 2 * 3 * 16          # conv1 3x3, 3 -> 16
    assert w[1] == 32 * 32 * 16                               # activation cells
    assert w[2] == 16 * 16 * 16                               # pool output cells
    assert w[3] == _valid_taps(16, 3) ** 2 * 16 * 32          # conv2 3x3, 16 -> 32
    assert w[4] == 16 * 16 * 32
    assert w[5] == 16 * 16 * 32 * 10                          # dense inputs x units


def test_layer_work_alexnet_crop_ratios():
    """conv1 (11x11) on an 8x8 crop vs the 64x64 COWC input: the ratio is the
    exact valid-tap ratio, not the pixel ratio (borders clip most taps)."""
    small = bench.layer_work(hb, hb.alexnet32_preset(image=8))
    full = bench.layer_work(hb, hb.alexnet32_preset(image=64))
    assert small[0] == _valid_taps(8, 11) ** 2 * 3 * 96
    assert full[0] == _valid_taps(64, 11) ** 2 * 3 * 96
    assert full[0] / small[0] > 64  # more than the 8^2 pixel ratio: the crop clips taps
    assert full[1] / small[1] == 64  # activations scale with cells
    kinds = [l.kind for l in hb.alexnet32_preset(image=64).layers]
    for i, k in enumerate(kinds):
        if k == hb.ZERO_PAD2D:
            assert full[i] > 0 and small[i] > 0
