"""Pins for the fp64 conv2d oracle (SURVEY.md 8(c) checks O1-O10).

Each check ties the oracle to something other than itself: a closed form, a
library routine (numpy matmul), an identity of convolution, brute force on
tiny inputs, or a cited golden value.  A dropped term, a flipped filter, a
wrong pad placement, a transposed operand or a wrong group offset fails at
least one of them.
"""
import itertools
import os

import numpy as np
import pytest

from oracle import conv as oc
from paper_2008_03602_b200 import datagen

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def shp(n, c, h, w, k, r, s, stride=1, pad=0, dil=1, groups=1, **kw):
    d = dict(n=n, c=c, h=h, w=w, k=k, r=r, s=s, stride_h=stride, stride_w=stride,
             pad_h=pad, pad_w=pad, dil_h=dil, dil_w=dil, groups=groups)
    d.update(kw)
    return d


def rand_int(rng, shape, lo=-3, hi=3):
    return rng.integers(lo, hi + 1, size=shape).astype(np.float64)


# ---- O1: output-size closed form vs a brute-force count of window origins ----
def test_o1_output_size_closed_form():
    for h, r, st, p, d in itertools.product(range(1, 17), range(1, 8), range(1, 4), range(0, 4), (1, 2)):
        origins = [o for o in range(-p, h + p) if (o + p) % st == 0 and o + d * (r - 1) <= h - 1 + p]
        assert oc.out_dim(h, r, st, p, d) == len(origins), (h, r, st, p, d)


def test_o1_golden_resnet50_sizes():
    with open(os.path.join(GOLDEN, "resnet50_feature_sizes.txt")) as f:
        rows = [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]
    assert len(rows) == 10
    for name, h, r, st, pad, want in rows:
        assert oc.out_dim(int(h), int(r), int(st), int(pad), 1) == int(want), name


def test_golden_box_filter():
    with open(os.path.join(GOLDEN, "conv_box_4x4.txt")) as f:
        vals = [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]
    P, Q = map(int, vals[0])
    want = np.array([[float(v) for v in row] for row in vals[1:]])
    x = np.arange(1, 17, dtype=np.float64).reshape(1, 1, 4, 4)
    w = np.ones((1, 1, 3, 3))
    y = oc.conv2d_c(shp(1, 1, 4, 4, 1, 3, 3), x, w)
    assert y.shape == (1, 1, P, Q)
    np.testing.assert_array_equal(y[0, 0], want)


# ---- O2: 1x1, s=1, p=0, g=1 conv is the GEMM Y = W X ----
@pytest.mark.parametrize("integer", [True, False])
def test_o2_1x1_equals_gemm(integer):
    rng = np.random.default_rng(2)
    n, c, h, w, k = 2, 5, 4, 3, 7
    x = rand_int(rng, (n, c, h, w)) if integer else rng.standard_normal((n, c, h, w))
    wt = rand_int(rng, (k, c, 1, 1)) if integer else rng.standard_normal((k, c, 1, 1))
    y = oc.conv2d_c(shp(n, c, h, w, k, 1, 1), x, wt)
    ref = np.matmul(wt[:, :, 0, 0], x.reshape(n, c, h * w)).reshape(n, k, h, w)
    if integer:
        np.testing.assert_array_equal(y, ref)
    else:
        assert np.max(np.abs(y - ref)) <= 1e-12 * np.max(np.abs(ref))


# ---- O3: identity filters reproduce the input ----
def test_o3_identity_filters():
    rng = np.random.default_rng(3)
    x = rng.standard_normal((2, 4, 6, 5))
    eye1 = np.eye(4).reshape(4, 4, 1, 1)
    np.testing.assert_array_equal(oc.conv2d_c(shp(2, 4, 6, 5, 4, 1, 1), x, eye1), x)
    eye3 = np.zeros((4, 4, 3, 3))
    for c in range(4):
        eye3[c, c, 1, 1] = 1.0
    np.testing.assert_array_equal(oc.conv2d_c(shp(2, 4, 6, 5, 4, 3, 3, pad=1), x, eye3), x)


# ---- O4: shifted delta pins filter orientation (no flip) and pad placement ----
@pytest.mark.parametrize("r0,s0", [(0, 0), (0, 2), (2, 1), (1, 0)])
def test_o4_shifted_delta(r0, s0):
    rng = np.random.default_rng(4)
    x = rng.standard_normal((1, 1, 5, 6))
    w = np.zeros((1, 1, 3, 3))
    w[0, 0, r0, s0] = 1.0
    y = oc.conv2d_c(shp(1, 1, 5, 6, 1, 3, 3, pad=1), x, w)[0, 0]
    want = np.zeros((5, 6))
    for p in range(5):
        for q in range(6):
            hi, wi = p - 1 + r0, q - 1 + s0
            if 0 <= hi < 5 and 0 <= wi < 6:
                want[p, q] = x[0, 0, hi, wi]
    np.testing.assert_array_equal(y, want)
    # cross-correlation: y[p,q] = x[p + r0 - pad, q + s0 - pad]; a flipped filter would read x[p - r0 + pad]
    if (r0, s0) != (1, 1):
        flipped = np.zeros((5, 6))
        for p in range(5):
            for q in range(6):
                hi, wi = p + 1 - r0, q + 1 - s0
                if 0 <= hi < 5 and 0 <= wi < 6:
                    flipped[p, q] = x[0, 0, hi, wi]
        assert not np.array_equal(y, flipped)


# ---- O5: tiny shapes, C oracle vs numpy formulation vs brute force ----
TINY = [(n, c, hw, k, rs, st, p, g)
        for n in (1, 2) for c in (1, 2, 4) for hw in (5, 7) for k in (1, 3, 4)
        for rs in (1, 2, 3) for st in (1, 2, 3) for p in (0, 1, 2) for g in (1, c)
        if (g == 1 or k == c) and k % g == 0]


@pytest.mark.parametrize("case", TINY[::7])
def test_o5_tiny_shapes_three_ways(case):
    n, c, hw, k, rs, st, p, g = case
    rng = np.random.default_rng(hash(case) & 0xFFFF)
    d = shp(n, c, hw, hw - 1, k, rs, rs, stride=st, pad=p, groups=g)
    x = rand_int(rng, (n, c, hw, hw - 1))
    w = rand_int(rng, (k, c // g, rs, rs))
    b = rand_int(rng, (k,))
    yc = oc.conv2d_c(d, x, w, b, relu=True)
    yn = oc.conv2d_numpy(d, x, w, b, relu=True)
    yb = oc.conv2d_brute(d, x, w, b, relu=True)
    np.testing.assert_array_equal(yc, yn)
    np.testing.assert_array_equal(yc, yb)
    xr, wr = rng.standard_normal(x.shape), rng.standard_normal(w.shape)
    yc, yn = oc.conv2d_c(d, xr, wr), oc.conv2d_numpy(d, xr, wr)
    assert np.max(np.abs(yc - yn)) <= 1e-12 * max(1.0, np.max(np.abs(yn)))


def test_o5_dilation_and_rect():
    rng = np.random.default_rng(55)
    d = shp(1, 3, 9, 8, 2, 3, 2, dil=2, pad=1, stride_h=2, stride_w=1)
    x, w = rand_int(rng, (1, 3, 9, 8)), rand_int(rng, (2, 3, 3, 2))
    np.testing.assert_array_equal(oc.conv2d_c(d, x, w), oc.conv2d_brute(d, x, w))
    np.testing.assert_array_equal(oc.conv2d_numpy(d, x, w), oc.conv2d_brute(d, x, w))


# ---- O6: linearity in x and in w ----
def test_o6_linearity():
    rng = np.random.default_rng(6)
    d = shp(2, 3, 8, 8, 4, 3, 3, stride=2, pad=1)
    x1, x2 = rng.standard_normal((2, 2, 3, 8, 8))
    w1, w2 = rng.standard_normal((2, 4, 3, 3, 3))
    a, b = 0.75, -1.25
    lhs = oc.conv2d_c(d, a * x1 + b * x2, w1)
    rhs = a * oc.conv2d_c(d, x1, w1) + b * oc.conv2d_c(d, x2, w1)
    assert np.max(np.abs(lhs - rhs)) <= 1e-12 * np.max(np.abs(rhs))
    lhs = oc.conv2d_c(d, x1, a * w1 + b * w2)
    rhs = a * oc.conv2d_c(d, x1, w1) + b * oc.conv2d_c(d, x1, w2)
    assert np.max(np.abs(lhs - rhs)) <= 1e-12 * np.max(np.abs(rhs))


# ---- O7/O8: depthwise = per-channel conv = dense conv with block-diagonal weight ----
def test_o7_o8_depthwise():
    rng = np.random.default_rng(7)
    c = 5
    d = shp(2, c, 7, 6, c, 3, 3, stride=2, pad=1, groups=c)
    x, w = rand_int(rng, (2, c, 7, 6)), rand_int(rng, (c, 1, 3, 3))
    y = oc.conv2d_c(d, x, w)
    for ch in range(c):
        y1 = oc.conv2d_c(shp(2, 1, 7, 6, 1, 3, 3, stride=2, pad=1), x[:, ch:ch + 1], w[ch:ch + 1])
        np.testing.assert_array_equal(y[:, ch:ch + 1], y1)
    wd = np.zeros((c, c, 3, 3))
    for ch in range(c):
        wd[ch, ch] = w[ch, 0]
    np.testing.assert_array_equal(y, oc.conv2d_c(shp(2, c, 7, 6, c, 3, 3, stride=2, pad=1), x, wd))


def test_groups_offset():
    """Group g reads channels [g*Cg, (g+1)*Cg): a group offset bug fails this."""
    rng = np.random.default_rng(77)
    d = shp(1, 4, 5, 5, 6, 3, 3, pad=1, groups=2)
    x, w = rand_int(rng, (1, 4, 5, 5)), rand_int(rng, (6, 2, 3, 3))
    y = oc.conv2d_c(d, x, w)
    lo = oc.conv2d_c(shp(1, 2, 5, 5, 3, 3, 3, pad=1), x[:, :2], w[:3])
    hi = oc.conv2d_c(shp(1, 2, 5, 5, 3, 3, 3, pad=1), x[:, 2:], w[3:])
    np.testing.assert_array_equal(y, np.concatenate([lo, hi], axis=1))


# ---- O9: full padding sum identity ----
def test_o9_full_padding_sum():
    rng = np.random.default_rng(9)
    n, c, h, w, k, r = 2, 3, 6, 5, 4, 3
    x, wt = rand_int(rng, (n, c, h, w)), rand_int(rng, (k, c, r, r))
    y = oc.conv2d_c(shp(n, c, h, w, k, r, r, pad=r - 1), x, wt)
    lhs = y.sum(axis=(2, 3))
    rhs = np.einsum("nc,kc->nk", x.sum(axis=(2, 3)), wt.sum(axis=(2, 3)))
    np.testing.assert_array_equal(lhs, rhs)


# ---- O10: stride-s conv = stride-1 conv (same pad) sampled every s ----
@pytest.mark.parametrize("st", [2, 3])
def test_o10_stride_subsample(st):
    rng = np.random.default_rng(10 + st)
    x, w = rand_int(rng, (1, 3, 11, 10)), rand_int(rng, (2, 3, 3, 3))
    y1 = oc.conv2d_c(shp(1, 3, 11, 10, 2, 3, 3, pad=1), x, w)
    ys = oc.conv2d_c(shp(1, 3, 11, 10, 2, 3, 3, pad=1, stride=st), x, w)
    np.testing.assert_array_equal(ys, y1[:, :, ::st, ::st])


# ---- epilogue (bias then ReLU, reading C9) and the sampled-points entry ----
def test_bias_relu_epilogue():
    rng = np.random.default_rng(11)
    d = shp(1, 3, 6, 6, 4, 3, 3, pad=1)
    x, w, b = rng.standard_normal((1, 3, 6, 6)), rng.standard_normal((4, 3, 3, 3)), rng.standard_normal(4)
    y0 = oc.conv2d_c(d, x, w)
    np.testing.assert_array_equal(oc.conv2d_c(d, x, w, b), y0 + b[None, :, None, None])
    np.testing.assert_array_equal(oc.conv2d_c(d, x, w, b, relu=True),
                                  np.maximum(y0 + b[None, :, None, None], 0.0))


def test_points_match_full():
    d = shp(2, 8, 9, 9, 6, 3, 3, stride=2, pad=1)
    x, w, b = datagen.make_inputs(d, 123)
    y = oc.conv2d_c(d, x, w, b, relu=True)
    idx = datagen.sample_points(y.size, 50, 5)
    pts = oc.conv2d_points_c(d, x, w, b, True, idx)
    np.testing.assert_array_equal(pts, y.reshape(-1)[idx])


def test_invalid_shape_rejected():
    with pytest.raises(ValueError):
        oc.conv2d_c(shp(1, 1, 2, 2, 1, 5, 5), np.zeros((1, 1, 2, 2)), np.zeros((1, 1, 5, 5)))
