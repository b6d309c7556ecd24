"""Pins for the CPU schedule-space enumeration (oracle/space.py), and
bit-exact agreement of libtp's host-only space functions with it (P-S)."""
import itertools

import numpy as np
import pytest

from oracle import space as sp
from paper_2008_03602_b200 import workloads as wl


def test_splitmix64_reference_vector():
    # Published SplitMix64 outputs for seed 0 (Vigna's reference implementation).
    g = sp.splitmix64(0)
    assert next(g) == 0xE220A8397B1DCDAF
    assert next(g) == 0x6E789E6AA1B965F4
    assert next(g) == 0x06C45D188009454F


def test_sample_properties():
    for n, t, seed in [(100, 10, 1), (920, 1000, 7), (5, 5, 3), (384, 383, 42), (1, 1, 0)]:
        s = sp.sample(n, t, seed)
        assert len(s) == min(n, t)
        assert len(set(s)) == len(s)
        assert all(0 <= i < n for i in s)
        assert s == sp.sample(n, t, seed)
    assert sp.sample(10, 20, 0) == list(range(10))
    assert sp.sample(1000, 10, 1) != sp.sample(1000, 10, 2)


def test_sample_hand_vector():
    # Reading C17 worked by hand from the published SplitMix64(0) outputs above:
    # o0 = 0xE220A8397B1DCDAF, o1 = 0x6E789E6AA1B965F4, o2 = 0x06C45D188009454F.
    # n = 10, t = 3: o0 mod 10 = 5 -> swap a[0], a[5]; o1 mod 9 = 0 -> j = 1 (no swap);
    # o2 mod 8 = 7 -> j = 9, swap a[2], a[9]  =>  [5, 1, 9].
    # n = 6, t = 3: o0 mod 6 = 1 -> swap a[0], a[1]; o1 mod 5 = 0 -> j = 1; o2 mod 4 = 3 -> j = 5 => [1, 0, 5].
    # (A swap index drawn as next() mod n would give [1, 5, 9] and [0, 2, 1].)
    assert (0xE220A8397B1DCDAF % 10, 0x6E789E6AA1B965F4 % 9, 0x06C45D188009454F % 8) == (5, 0, 7)
    assert sp.sample(10, 3, 0) == [5, 1, 9]
    assert sp.sample(6, 3, 0) == [1, 0, 5]


def test_direct_smem_depthwise_hand():
    # Depthwise smem (reading C25): halo rows x halo cols x (lanes_k vec_k) channels +
    # R S (lanes_k vec_k) weights, fp32 -- the CTA's channel tile, which the kernel allocates even
    # where lanes_k vec_k exceeds C.  MobileNetV2 dw.960.7.s1 (C = K = 960, 7x7, 3x3 s1 p1):
    # threads 64, tile_q 1, vec_k 8, tile_p 1: ceil(960/8) = 120 -> np2 128, lanes_k = min(128, 64) = 64,
    #   lanes_q = 1; channel tile 512, halo 3 x 3: 4 (9 x 512 + 9 x 512) = 36864 B.
    # threads 512, tile_q 4, vec_k 8, tile_p 1: lanes_k = 128, lanes_q = 4, 16 output columns -> 18 input
    #   columns; channel tile 1024 (> C = 960): 4 (3 x 18 x 1024 + 9 x 1024) = 258048 B > 232448 -> invalid.
    d = [x for x in wl.catalog("mobilenetv2") if x["name"] == "mb2.dw.960.7.s1"][0]
    assert sp.direct_smem_bytes(d, 64, 1, 8, 1) == 36864
    assert sp.direct_smem_bytes(d, 512, 4, 8, 1) == 258048
    assert not sp._valid_direct(d, 512, 4, 8, 1, 1) and sp._valid_direct(d, 512, 4, 8, 1, 0)
    # dense (g = 1) branch: at most 16 input channels staged.  cfg1 (C = 64, 56x56, K = 64, 3x3 s1):
    # threads 256, tile_q 2, vec_k 4, tile_p 2: lanes_k = min(np2(16), 128) = 16, lanes_q = 256 / 32 = 8;
    # 16 output columns -> 18 input columns, 2 output rows -> 4 input rows, channel tile 64:
    # 4 (4 x 18 x 16 + 9 x 16 x 64) = 4 (1152 + 9216) = 41472 B.
    assert sp.direct_smem_bytes(wl.catalog("cfg1")[0], 256, 2, 4, 2) == 41472


def test_mobilenetv2_space_totals():
    # Mirror totals with reading C25: direct 3628 + IGEMM_TC 6148 + gathered 48 + stem 8 (+ 15 strip) = 9832
    # base + appended kinds;
    # the SURVEY 8(a) a2 count (10,180, stem on the direct kind) clamps the depthwise channel tile at C
    # and so admits 20 more direct schedules: 9776 + 384 (stem's direct space) = 10,160 here.
    cat = wl.catalog("mobilenetv2")
    kinds = {}
    for d in cat:
        for x in sp.enumerate_space(d):
            kinds[x["kind"]] = kinds.get(x["kind"], 0) + 1
    assert kinds == {sp.KIND_DIRECT: 3628, sp.KIND_IGEMM_TC: 6148, sp.KIND_IGEMM_TC_GATHER: 48,
                     sp.KIND_IGEMM_TC_STEM: 8, sp.KIND_IGEMM_TC_STRIP: 15}
    stem = [d for d in cat if sp.layer_kind(d) == sp.KIND_IGEMM_TC_GATHER]
    assert len(stem) == 1 and kinds[sp.KIND_DIRECT] + kinds[sp.KIND_IGEMM_TC] + _direct_count(stem[0]) == 10160


def test_argmin_tie_break():
    recs = [dict(status=0, median_us=5.0, space_index=9), dict(status=4, median_us=1.0, space_index=1),
            dict(status=0, median_us=5.0, space_index=3), dict(status=0, median_us=6.0, space_index=0)]
    assert sp.argmin(recs) == 2
    assert sp.argmin([dict(status=5, median_us=1.0, space_index=0)]) == -1


def _direct_count(d):
    return sum(1 for th, tq, vk, tpp, sm in itertools.product(*[v for _, v in sp.DIRECT_KNOBS])
               if sp._valid_direct(d, th, tq, vk, tpp, sm))


def test_space_counts_and_order():
    # Totals cross-checked against SURVEY.md 8(a) a2's independent count of the same
    # predicate (R50 14,432; VGG-19 6,672), which put the C = 3 stems on the direct
    # kind; they now take the gathered tensor-core kind, so the SURVEY totals hold
    # for the other layers plus the stems' direct-space counts.
    for name, total in (("resnet50", 14432), ("vgg19_b16", 6672)):
        cat = wl.catalog(name)
        stems = [d for d in cat if sp.layer_kind(d) == sp.KIND_IGEMM_TC_GATHER]
        rest = [d for d in cat if sp.layer_kind(d) != sp.KIND_IGEMM_TC_GATHER]
        assert len(stems) == 1 and stems[0]["c"] == 3
        n_rest = sum(1 for d in rest for x in sp.enumerate_space(d)
                     if x["kind"] not in (sp.KIND_IGEMM_TC_ROW, sp.KIND_IGEMM_TC_ROWW, sp.KIND_IGEMM_TC_MT))
        assert n_rest + _direct_count(stems[0]) == total
    d = wl.catalog("resnet50")[2]
    s = sp.enumerate_space(d)
    keys = [(x["kind"], x["bm"], x["bn"], x["bk"], x["stages"], x["threads"], x["split_k"]) for x in s]
    assert keys == sorted(keys)      # kind is the outermost key (appended kinds follow the TMA ones)
    assert [x["space_index"] for x in s] == list(range(len(s)))


def test_gather_space_hand_count():
    # R50 conv1 (C=3, 7x7 s2, K=64, M=12544): reduction R*S*C = 147 (np2 256).
    # BN in {32, 64}; BM in {64, 128}; every BK; split_k <= ceil(147/BK);
    # smem = stages (BM+BN) BK 2 + 1024 + 16 BM + 8 ceil(147/BK) BK <= 232448.
    n = 0
    for bm in (64, 128):
        for bn in (32, 64):
            for bk in (16, 32, 64, 128):
                nkb = -(-147 // bk)
                for st in (2, 3, 4, 6):
                    if st * (bm + bn) * bk * 2 + 1024 + 16 * bm + 8 * nkb * bk > 232448:
                        continue
                    n += 2 * sum(1 for sk in (1, 2, 4, 8) if sk <= nkb)
    d = wl.catalog("resnet50")[0]
    g = [s for s in sp.enumerate_space(d) if s["kind"] == sp.KIND_IGEMM_TC_GATHER]
    assert len(g) == n and sp.enumerate_space(d)[:n] == g


def test_stem_kind_hand_count():
    # R50 conv1 (C=3, 7x7 s2 p3, Q=112): KP = 64 ceil(147/64) = 192; BM {64, 128} (<= np2(112));
    # BN <= max(32, np2(64)) -> {32, 64}; tiles_per_cta {2, 4, 8, 16}; the largest smem
    # (BM=128, BN=64) = 64*192*2 + 2*128*192*2 + 2 ceil(7*786*2/1024) KiB + 1 KiB (k table) + 128*64*4
    # (output staging) + 1024 = 24576 + 98304 + 22528 + 1024 + 32768 + 1024 = 180224 fits: 2 x 2 x 4 = 16,
    # appended right after the gathered tuples (the strip kind follows).
    d = wl.catalog("resnet50")[0]
    sps = sp.enumerate_space(d)
    st = [s for s in sps if s["kind"] == sp.KIND_IGEMM_TC_STEM]
    g = [s for s in sps if s["kind"] == sp.KIND_IGEMM_TC_GATHER]
    assert len(st) == 16 and sps[len(g):len(g) + 16] == st and all(s["bk"] == 192 for s in st)
    x = [s for s in st if s["bm"] == 64 and s["bn"] == 32 and s["tiles_per_cta"] == 8][0]
    assert (x["grid_x"], x["grid_y"], x["grid_z"]) == (-(-(112 * 2) // 8), 2, 1)
    # VGG conv1_1 (C=3, 3x3 s1, Q=224, b16): KP = 64; eligible; MobileNetV2 conv0 (3x3 s2, Q=112): eligible
    v = wl.catalog("vgg19_b16")[0]
    assert sp.stem_eligible(v) and sp.stem_kp(v) == 64
    assert sp.stem_eligible(wl.catalog("mobilenetv2")[0])
    # not eligible: C % 8 == 0 layers, narrow outputs, R S C > 256
    assert not sp.stem_eligible(wl.catalog("resnet50")[1])
    assert not sp.stem_eligible(dict(v, h=32, w=32))
    assert not sp.stem_eligible(dict(v, c=6, r=7, s=7))


def test_roww_kind_hand_count():
    # Row-halo kind with resident weights (C = 64 row-halo layers), appended right after the row-halo
    # tuples.  VGG conv1_2 (Q = 224, K = 64): BM {64, 128}, BN {32, 64}, stages {2, 4, 6, 8},
    # tiles_per_cta {2, 4, 8, 16}; the largest (BM 128, BN 64, 8 strips): 8 x 17 KiB + 9 x 64 x 128 + 1 KiB
    # = 139264 + 73728 + 1024 = 214016 fits -> 2 x 2 x 4 x 4 = 64.  conv2_1 (K = 128): BN = 128 weights are
    # 147456 B, so with BM = 128 (17 KiB strips) only 2 or 4 stages fit (6 x 17408 + 147456 + 1024 > 232448):
    # BN 32/64 -> 2 x 2 x 4 x 4 = 64, BN 128 -> (BM 64: 9 KiB strips, all 4 stages; BM 128: 2) x 4 = 24 -> 88.
    v = wl.catalog("vgg19_b16")
    for d, n in ((v[1], 64), (v[2], 88)):
        space = sp.enumerate_space(d)
        rw = [x for x in space if x["kind"] == sp.KIND_IGEMM_TC_ROWW]
        row = [i for i, x in enumerate(space) if x["kind"] == sp.KIND_IGEMM_TC_ROW]
        assert len(rw) == n and space[row[-1] + 1:row[-1] + 1 + n] == rw
        assert all(x["bk"] == 64 and x["threads"] == 256 and x["split_k"] == 1 for x in rw)
    assert not sp.roww_eligible(v[3])             # conv2_2: C = 128
    assert [d["name"] for d in wl.catalog("resnet50") if sp.roww_eligible(d)] == ["r50.l1.b0.c2"]   # Q = 56, C = 64


def test_strip_kind_hand_count():
    # Strip kind, appended after the stem tuples.  Phase-box pixels:
    # BM + 2 ceil(ceil(S / s_w) / 2) - 1; s_w x that <= 256 (TMA box extent).
    # R50 conv1 (7x7 s2, K = 64, Q = 112): 4 taps in phase 0 -> BM + 3 px; BM = 128 -> 2 x 131 = 262 > 256,
    #   so BM = 64 only (2 x 67 = 134); BN {32, 64}; stages {2, 4, 6}; tiles_per_cta {1, 2, 4, 8, 16}:
    #   smem <= 6 x 2 x 1152 + 7 x 9 x 64 x 16 (64512 -> 63 KiB) + 1 KiB fits -> 1 x 2 x 3 x 5 = 30.
    # VGG conv1_1 (3x3 s1, K = 64): BM + 3 px <= 256 for both BM -> 2 x 2 x 3 x 5 = 60.
    # MobileNetV2 conv0 (3x3 s2, K = 32): phase 0 has 2 taps -> BM + 1 px; BM = 128 -> 258 > 256 -> 15.
    for cat, n, bms in (("resnet50", 30, {64}), ("vgg19_b16", 60, {64, 128}), ("mobilenetv2", 15, {64})):
        d = wl.catalog(cat)[0]
        space = sp.enumerate_space(d)
        st = [x for x in space if x["kind"] == sp.KIND_IGEMM_TC_STRIP]
        assert len(st) == n and {x["bm"] for x in st} == bms and all(x["bk"] == 16 for x in st)
        last_stem = max(i for i, x in enumerate(space) if x["kind"] == sp.KIND_IGEMM_TC_STEM)
        assert space[last_stem + 1:last_stem + 1 + n] == st
    x = [s for s in sp.enumerate_space(wl.catalog("resnet50")[0]) if s["kind"] == sp.KIND_IGEMM_TC_STRIP
         and s["bn"] == 64 and s["tiles_per_cta"] == 4][0]
    assert (x["grid_x"], x["grid_y"], x["grid_z"]) == (-(-(112 * 2) // 4), 1, 1)
    # not eligible: C % 8 == 0 layers, stride 3 columns, filters wider than 8
    v = wl.catalog("vgg19_b16")[0]
    assert not sp.strip_eligible(wl.catalog("resnet50")[1])
    assert not sp.strip_eligible(dict(v, stride_w=3)) and not sp.strip_eligible(dict(v, s=9, pad_w=4))


def test_row_kind_hand_count_and_order():
    # VGG conv1_2 (C=64, 224x224, K=64, 3x3 s1 p1): eligible.  BM in {64, 128}
    # (np2(Q) = 256), BN in {32, 64} (np2(K) = 64), stages {1, 2, 3}, threads x tiles-per-CTA
    # in {(128, 1), (256, 1), (256, 2), (256, 4), (256, 8), (256, 16)}; largest stage = 17408
    # (strip 130 x 128 B -> 1 KiB multiple) + 3 x 64 x 128 = 41984 B, x 3 stages + 1024 fits:
    # 2 x 2 x 3 x 6 = 72.
    d = wl.catalog("vgg19_b16")[1]
    space = sp.enumerate_space(d)
    row = [x for x in space if x["kind"] == sp.KIND_IGEMM_TC_ROW]
    assert len(row) == 72
    first = space.index(row[0])
    assert all(x["kind"] == sp.KIND_IGEMM_TC for x in space[:first]) and space[first:first + len(row)] == row
    assert all(x["bk"] == 64 and x["split_k"] == 1 for x in row)
    assert row[0]["grid_x"] == 16 * 224 * 4 and row[0]["grid_y"] == 2          # BM=64, BN=32, 1 tile/CTA
    r4 = [x for x in row if x["tiles_per_cta"] == 4 and x["bm"] == 128][0]
    assert r4["grid_x"] == 16 * 224 * 2 // 4 and r4["threads"] == 256
    # not eligible: stride 2, pad 0, C % 64 != 0, Q < 56
    r50 = wl.catalog("resnet50")
    assert [sp.row_eligible(x) for x in r50].count(True) == 1 and sp.row_eligible(r50[2])   # l1.b0.c2 only


def test_mt_kind_hand_count():
    # VGG conv3_1 (b16, C=128, 56x56, K=256): 784 x 8 >= 1024 64x32 tiles -> eligible.  BM {64, 128},
    # BN {32..256}, stages {2, 3, 4}, tiles_per_cta {2, 4, 8}; smem = stages (BM+BN) 128 + 1024 fits
    # for every combination (max 4 x 384 x 128 + 1024 = 197632): 2 x 4 x 3 x 3 = 72, appended last.
    d = wl.catalog("vgg19_b16")[4]
    space = sp.enumerate_space(d)
    mt = [x for x in space if x["kind"] == sp.KIND_IGEMM_TC_MT]
    assert len(mt) == 72 and space[-72:] == mt and all(x["threads"] == 256 for x in mt)
    x = [m for m in mt if m["bm"] == 128 and m["bn"] == 128 and m["tiles_per_cta"] == 4][0]
    assert (x["grid_x"], x["grid_y"], x["grid_z"]) == (-(-(16 * 56 * 56 // 128) // 4), 2, 1)
    assert not any(sp.mt_eligible(r) for r in wl.catalog("resnet50"))


def test_tf32_kind_hand_count():
    # cfg1 (fp32, C = K = 64, 56x56, 3x3): eligible (C % 4 == 0, K % 8 == 0, g = 1).  BM {64, 128}
    # (M = 3136), BN <= max(32, np2(64)) -> {32, 64}, stages {2, 3, 4}, split_k {1, 2, 4, 8} (<= 9 taps x
    # 2 channel blocks); smem = stages (BM+BN) 256 + [split > 1] BM (BN+4) 4 + 1024 fits for all (max
    # 4 x 192 x 256 + 128 x 68 x 4 + 1024 = 232448 = the limit): 2 x 2 x 3 x 4 = 48, after the direct tuples.
    d = wl.catalog("cfg1")[0]
    space = sp.enumerate_space(d)
    tf = [x for x in space if x["kind"] == sp.KIND_IGEMM_TF32X3]
    assert len(tf) == 48 and space[-48:] == tf
    assert all(x["bk"] == 32 and x["threads"] == 256 for x in tf)
    x = [t for t in tf if t["bm"] == 128 and t["bn"] == 64 and t["stages"] == 3 and t["split_k"] == 4][0]
    assert (x["grid_x"], x["grid_y"], x["grid_z"]) == (-(-3136 // 128), 1, 4)
    # not eligible: bf16 layers, C % 4 != 0, K % 8 != 0, depthwise
    e = dict(d)
    assert not sp.tf32_eligible(dict(e, c=3)) and not sp.tf32_eligible(dict(e, k=60))
    assert not sp.tf32_eligible(dict(e, groups=64)) and not sp.tf32_eligible(dict(e, dtype=sp.DTYPE_BF16))
    # BN = 256 at BM = 128 fits only with 2 stages (3 x 384 x 256 + 1024 = 295936 > 232448), and then
    # only without the split-K receive buffer (197632 + 128 x 260 x 4 = 330752 > 232448)
    big = dict(e, k=256, h=16, w=16)
    tf2 = [x for x in sp.enumerate_space(big) if x["kind"] == sp.KIND_IGEMM_TF32X3]
    assert [(x["stages"], x["split_k"]) for x in tf2 if x["bn"] == 256 and x["bm"] == 128] == [(2, 1)]
    # split_k <= k-blocks: a 1x1 layer with C = 36 has 2 k-blocks
    one = dict(e, c=36, r=1, s=1, pad_h=0, pad_w=0)
    assert {x["split_k"] for x in sp.enumerate_space(one) if x["kind"] == sp.KIND_IGEMM_TF32X3} == {1, 2}


def test_kind_selection():
    r50 = wl.catalog("resnet50")
    assert sp.layer_kind(r50[0]) == sp.KIND_IGEMM_TC_GATHER  # C = 3 stem
    assert all(sp.layer_kind(d) == sp.KIND_IGEMM_TC for d in r50[1:])
    assert sp.layer_kind(wl.catalog("cfg1")[0]) == sp.KIND_DIRECT   # fp32
    mb = wl.catalog("mobilenetv2")
    assert all(sp.layer_kind(d) == sp.KIND_DIRECT for d in mb if d["groups"] > 1)


def test_waves_example():
    # R50 l1.b0.c2 with 128x64 tiles -> 25 CTAs.
    d = wl.catalog("resnet50")[2]
    g = sp.geometry(d, dict(kind=0, bm=128, bn=64, split_k=1, threads=128))
    assert g["ctas"] == 25
    assert [sp.waves(25, m, 1) for m in (16, 32, 72, 148)] == [2, 1, 1, 1]
    assert [sp.waves(100, m, 1) for m in (16, 32, 72, 148)] == [7, 4, 2, 1]


# ---------------- libtp host-only functions vs the mirror (bit-exact) ----------------
def _lib_or_skip():
    try:
        from paper_2008_03602_b200 import tp
        return tp
    except Exception as e:  # pragma: no cover
        pytest.fail(f"libtp.so failed to load: {e}")


SHAPES = wl.catalog("cfg1") + wl.catalog("resnet50") + wl.catalog("vgg19_b16") + wl.catalog("mobilenetv2")


@pytest.mark.parametrize("d", SHAPES, ids=[d["name"] for d in SHAPES])
def test_libtp_space_matches_mirror(d):
    tp = _lib_or_skip()
    mirror = sp.enumerate_space(d)
    assert tp.space_size(d) == len(mirror)
    fields_tc = ("bm", "bn", "bk", "stages", "threads", "split_k")
    fields_dir = ("threads", "tile_q", "vec_k", "tile_p", "smem_stage")
    for m in mirror:
        s = tp.space_get(d, m["space_index"])
        assert s["kind"] == m["kind"]
        for f in (fields_dir if m["kind"] == sp.KIND_DIRECT else fields_tc + ("kind",)):
            assert s[f] == m[f], (f, m)
        if m["kind"] in (sp.KIND_IGEMM_TC_ROW, sp.KIND_IGEMM_TC_MT, sp.KIND_IGEMM_TC_STEM, sp.KIND_IGEMM_TC_STRIP):
            f = "tiles_per_cta"
            assert s[f] == m[f], (f, m)
        assert (s["grid_x"], s["grid_y"], s["grid_z"]) == (m["grid_x"], m["grid_y"], m["grid_z"])
        assert s["space_index"] == m["space_index"]


@pytest.mark.parametrize("trials,seed", [(10, 42), (100, 43), (1000, 44), (5000, 45), (1, 0)])
def test_libtp_sampler_matches_mirror(trials, seed):
    tp = _lib_or_skip()
    for d in wl.catalog("resnet50")[:6]:
        n = tp.space_size(d)
        assert tp.space_sample(d, trials, seed) == sp.sample(n, trials, seed)


def test_libtp_argmin_matches_mirror():
    tp = _lib_or_skip()
    rng = np.random.default_rng(0)
    for _ in range(20):
        n = int(rng.integers(1, 50))
        recs = [dict(status=int(rng.choice([0, 0, 0, 5])), median_us=float(rng.choice([1.5, 2.0, 2.5, 3.0])),
                     space_index=int(i)) for i in rng.permutation(n)]
        assert tp.select_best(recs) == sp.argmin(recs)


@pytest.mark.parametrize("d", SHAPES, ids=[d["name"] for d in SHAPES])
def test_gate_points_cover_the_output(d):
    # Consensus-gate fallback points (a10): distinct, sorted, in range, and spread over
    # pixels AND channels (a fixed stride i*total/4096 put every VGG-19 b16 point in column q = 0).
    tp = _lib_or_skip()
    P, Q = sp.out_pq(d)
    total = d["n"] * d["k"] * P * Q
    idx = tp.gate_points(d, 4096)
    assert len(idx) == min(4096, total) and np.all(np.diff(idx) > 0) and idx[0] >= 0 and idx[-1] < total
    assert np.array_equal(idx, tp.gate_points(d, 4096))   # deterministic
    q = idx % Q
    p = (idx // Q) % P
    k = (idx // (P * Q)) % d["k"]
    n = idx // (P * Q * d["k"])
    pix = len(set(zip(n.tolist(), p.tolist(), q.tolist())))
    assert len(set(q.tolist())) >= min(Q, len(idx) // 8)
    assert len(set(p.tolist())) >= min(P, len(idx) // 8)
    assert len(set(k.tolist())) >= min(d["k"], len(idx) // 8) * 0.9
    assert pix >= min(d["n"] * P * Q, len(idx)) * 0.5


def test_libtp_output_shape():
    tp = _lib_or_skip()
    for d in SHAPES:
        assert tp.output_shape(d) == sp.out_pq(d)
    bad = dict(SHAPES[1], h=0)
    with pytest.raises(tp.TPError):
        tp.output_shape(bad)
