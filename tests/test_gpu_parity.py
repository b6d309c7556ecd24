"""GPU parity: libtp's CUDA path (through the C-ABI) vs the fp64 oracle.

Bars (north_star): bf16 inputs with fp32 accumulation within 2e-2 max relative
error (reading C10: max|y - ref| / max|ref|), fp32 path within 1e-5; integer
data (x, w in {-3..3}) bit-exact for every schedule with fp32 output (O11,
"the output of the inference remains the same").
"""
import numpy as np
import pytest
import torch

from oracle import conv as oc
from oracle import space as sp
from paper_2008_03602_b200 import datagen, tp, workloads as wl

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _init():
    if not torch.cuda.is_available():
        pytest.fail("gpu test without a GPU")
    tp.init(0)
    yield


def bf16_round(a):
    return torch.tensor(np.asarray(a, dtype=np.float32)).bfloat16().double().numpy()


def oracle_ref(d, x, w, b):
    if d["dtype"] == tp.BF16:
        x, w = bf16_round(x), bf16_round(w)
    return oc.conv2d_c(d, x, w, b if d["epilogue"] & 1 else None, relu=bool(d["epilogue"] & 2))


def rel_err(y, ref):
    return float(np.max(np.abs(y - ref)) / max(np.max(np.abs(ref)), 1e-30))


def mk(n, c, h, w, k, r, s, st=1, pad=0, g=1, dtype=tp.BF16, out=None, epi=3, layout=tp.NHWC):
    return dict(n=n, c=c, h=h, w=w, k=k, r=r, s=s, stride_h=st, stride_w=st, pad_h=pad, pad_w=pad, dil_h=1, dil_w=1,
                groups=g, in_layout=layout, dtype=dtype, out_dtype=dtype if out is None else out, epilogue=epi)


# ------------------------------------------------------------------ exhaustive integer sweeps (O11)
TC_TINY = [mk(1, 64, 10, 9, 64, 3, 3, 1, 1, out=tp.FP32, epi=1),
           mk(2, 32, 7, 7, 48, 1, 1, 1, 0, out=tp.FP32, epi=1),
           mk(1, 136, 9, 11, 40, 3, 3, 2, 1, out=tp.FP32, epi=1),
           # row-halo kind appended (3x3 s1 p1, C % 64 == 0, Q >= 56): ragged rows, 2 channel blocks, N = 2
           mk(1, 64, 6, 60, 40, 3, 3, 1, 1, out=tp.FP32, epi=1),
           mk(2, 128, 4, 57, 24, 3, 3, 1, 1, out=tp.FP32, epi=1),
           # gathered kind (C % 8 != 0): the ResNet/VGG/MobileNet stems, ragged M tails
           mk(1, 3, 23, 21, 64, 7, 7, 2, 3, out=tp.FP32, epi=1),
           mk(2, 3, 9, 10, 24, 3, 3, 1, 1, out=tp.FP32, epi=1),
           mk(1, 5, 12, 12, 32, 3, 3, 2, 1, out=tp.FP32, epi=1)]


@pytest.mark.parametrize("d", TC_TINY, ids=lambda d: f"tc_{d['c']}x{d['h']}x{d['w']}_k{d['k']}_r{d['r']}s{d['stride_h']}")
def test_tc_every_schedule_bit_exact_integer(d):
    x, w, b = datagen.make_inputs(d, 11, integer=True)
    ref = oracle_ref(d, x, w, b)
    buf = tp.LayerBuffers(d, x, w, b)
    n = tp.space_size(d)
    assert sp.layer_kind(d) == (tp.KIND_IGEMM_TC if d["c"] % 8 == 0 else tp.KIND_IGEMM_TC_GATHER)
    bad = []
    for i in range(n):
        s = tp.space_get(d, i)
        buf.poison()
        tp.conv2d_run(buf, s)
        torch.cuda.synchronize()
        y = buf.output()
        if not np.array_equal(y, ref):
            bad.append((i, {k: s[k] for k in ("bm", "bn", "bk", "stages", "threads", "split_k")},
                        float(np.nanmax(np.abs(y - ref)))))
    assert not bad, f"{len(bad)}/{n} schedules differ, first: {bad[:5]}"


DIRECT_TINY = [mk(1, 8, 9, 10, 12, 3, 3, 1, 1, dtype=tp.FP32, epi=1),
               mk(2, 3, 11, 11, 16, 7, 7, 2, 3, dtype=tp.FP32, epi=1),
               mk(1, 16, 9, 9, 16, 3, 3, 2, 1, g=16, dtype=tp.FP32, epi=1),
               mk(1, 24, 7, 7, 24, 3, 3, 1, 1, g=24, dtype=tp.BF16, out=tp.FP32, epi=1)]


@pytest.mark.parametrize("d", DIRECT_TINY, ids=lambda d: f"direct_{d['c']}_g{d['groups']}_s{d['stride_h']}_{d['dtype']}")
def test_direct_every_schedule_bit_exact_integer(d):
    x, w, b = datagen.make_inputs(d, 12, integer=True)
    ref = oracle_ref(d, x, w, b)
    buf = tp.LayerBuffers(d, x, w, b)
    n = tp.space_size(d)
    bad = []
    for i in range(n):
        s = tp.space_get(d, i)
        buf.poison()
        tp.conv2d_run(buf, s)
        torch.cuda.synchronize()
        y = buf.output()
        if not np.array_equal(y, ref):
            bad.append((i, s["threads"], s["tile_q"], s["vec_k"], s["tile_p"], s["smem_stage"]))
    assert not bad, f"{len(bad)}/{n} schedules differ, first: {bad[:5]}"


# ------------------------------------------------------------------ random data, tolerance bars
def _sampled_scheds(d, k=12, seed=0):
    n = tp.space_size(d)
    return [tp.space_get(d, i) for i in sp.sample(n, k, seed)]


CFG_SHAPES = (wl.catalog("cfg1") + wl.catalog("resnet50") + wl.catalog("mobilenetv2")[:12])


@pytest.mark.parametrize("d", CFG_SHAPES, ids=[d["name"] for d in CFG_SHAPES])
def test_layer_random_parity(d):
    x, w, b = datagen.make_inputs(d, datagen.data_seed(9, 0))
    ref = oracle_ref(d, x, w, b)
    buf = tp.LayerBuffers(d, x, w, b)
    tol = 2e-2 if d["dtype"] == tp.BF16 else 1e-5
    for s in _sampled_scheds(d, 6, 1):
        buf.poison()
        tp.conv2d_run(buf, s)
        torch.cuda.synchronize()
        err = rel_err(buf.output(), ref)
        assert err <= tol, (s, err)


@pytest.mark.parametrize("d", wl.catalog("vgg19_b16")[0:3], ids=lambda d: d["name"])
def test_vgg_full_size_sampled_points(d):
    """Full BASELINE size (batch 16): oracle evaluated at 4096 sampled outputs."""
    x, w, b = datagen.make_inputs(d, datagen.data_seed(4, 1))
    buf = tp.LayerBuffers(d, x, w, b)
    P, Q = tp.output_shape(d)
    idx = datagen.sample_points(d["n"] * d["k"] * P * Q, 4096, 3)
    ref = oc.conv2d_points_c(d, bf16_round(x), bf16_round(w), b, True, idx)
    for s in _sampled_scheds(d, 4, 2):
        tp.conv2d_run(buf, s)
        torch.cuda.synchronize()
        got = buf.gather(idx)
        assert rel_err(got, ref) <= 2e-2, s


def test_nchw_layout_matches_nhwc():
    d = mk(1, 64, 12, 12, 32, 3, 3, 1, 1, out=tp.FP32, epi=3)
    dn = dict(d, in_layout=tp.NCHW)
    x, w, b = datagen.make_inputs(d, 5)
    ref = oracle_ref(d, x, w, b)
    for dd in (d, dn):
        buf = tp.LayerBuffers(dd, x, w, b)
        for s in _sampled_scheds(dd, 4, 3):
            tp.conv2d_run(buf, s)
            torch.cuda.synchronize()
            assert rel_err(buf.output(), ref) <= 2e-2


def test_split_k_deterministic():
    d = wl.catalog("resnet50")[18]
    x, w, b = datagen.make_inputs(d, 8)
    buf = tp.LayerBuffers(d, x, w, b)
    s = next(tp.space_get(d, i) for i in range(tp.space_size(d)) if tp.space_get(d, i)["split_k"] == 8)
    outs = []
    for _ in range(3):
        tp.conv2d_run(buf, s)
        torch.cuda.synchronize()
        outs.append(buf.y.clone())
    assert all(torch.equal(outs[0], o) for o in outs[1:])
    # the workspace counters are left zeroed
    assert int(buf.ws[:4 * 64].view(torch.int32).abs().sum()) == 0


def test_pack_kernels_bit_exact():
    d = mk(2, 24, 5, 7, 8, 3, 3, 1, 1)
    x, w, b = datagen.make_inputs(d, 4)
    buf = tp.LayerBuffers(d, x, w, b)
    xb = buf.x.view(torch.bfloat16).cpu()
    want = torch.tensor(x).permute(0, 2, 3, 1).contiguous().bfloat16().reshape(-1)
    assert torch.equal(xb.view(torch.int16), want.view(torch.int16))
    wb = buf.w.view(torch.bfloat16).cpu()
    wwant = torch.tensor(w).permute(0, 2, 3, 1).contiguous().bfloat16().reshape(-1)
    assert torch.equal(wb.view(torch.int16), wwant.view(torch.int16))


@pytest.mark.parametrize("d", [TC_TINY[0], TC_TINY[4], TC_TINY[6]], ids=["tc", "row", "gather"])
def test_every_schedule_bit_exact_global_splitk(d, monkeypatch):
    """Split-K through the global workspace (the fallback when a context cannot
    co-schedule the (1,1,split_k) cluster), interleaved with split-1 schedules
    of every kind in the space, twice: the arrival counters must survive them."""
    monkeypatch.setenv("TP_NO_CLUSTER", "1")
    x, w, b = datagen.make_inputs(d, 13, integer=True)
    ref = oracle_ref(d, x, w, b)
    buf = tp.LayerBuffers(d, x, w, b)
    bad = []
    for rep in range(2):
        for i in range(tp.space_size(d)):
            s = tp.space_get(d, i)
            buf.poison()
            tp.conv2d_run(buf, s)
            torch.cuda.synchronize()
            if not np.array_equal(buf.output(), ref):
                bad.append((rep, i, s["kind"], s["split_k"]))
    assert not bad, f"{len(bad)} schedule runs differ, first: {bad[:5]}"


def test_multitile_kind_every_schedule_bit_exact_integer():
    """IGEMM_TC_MT (>= 1024 tiles of 64 x 32): every multi-tile schedule, ragged
    tile counts per CTA (tiles_per_cta 8 over 128 or 256 tiles of 128/64)."""
    d = mk(1, 64, 128, 128, 128, 3, 3, 1, 1, out=tp.FP32, epi=1)
    assert sp.mt_eligible(d)
    x, w, b = datagen.make_inputs(d, 17, integer=True)
    ref = oracle_ref(d, x, w, b)
    buf = tp.LayerBuffers(d, x, w, b)
    bad, n = [], 0
    for i in range(tp.space_size(d)):
        s = tp.space_get(d, i)
        if s["kind"] != tp.KIND_IGEMM_TC_MT:
            continue
        n += 1
        buf.poison()
        tp.conv2d_run(buf, s)
        torch.cuda.synchronize()
        if not np.array_equal(buf.output(), ref):
            bad.append((i, {k: s[k] for k in ("bm", "bn", "stages", "tiles_per_cta")}))
    # BM {64, 128} x BN {32, 64, 128} (K = 128) x stages {2, 3, 4} x tiles_per_cta {2, 4, 8}
    assert n == 54 and not bad, f"{len(bad)}/{n} differ, first: {bad[:5]}"


@pytest.mark.parametrize("d", TC_TINY + [mk(1, 64, 128, 128, 128, 3, 3, 1, 1, out=tp.FP32, epi=1)],
                         ids=lambda d: f"early_{d['c']}x{d['h']}x{d['w']}_k{d['k']}_r{d['r']}s{d['stride_h']}")
def test_timed_launches_weight_prefetch_bit_exact_integer(d):
    """Timed runs (time_plan): the first launch waits on the PDL dependency
    before any load; every later launch issues its first ring pass of weight
    boxes before griddepcontrol.wait (TcArgs::w_early).  The last launch of a
    timed run is such a launch, so y after timing must still equal the oracle
    bit-exactly (O11) for every tensor-core schedule."""
    x, w, b = datagen.make_inputs(d, 13, integer=True)
    ref = oracle_ref(d, x, w, b)
    buf = tp.LayerBuffers(d, x, w, b)
    tm = tp.timing(warmup=1, groups=1, n_min=2, target_group_us=1.0)
    bad, n = [], tp.space_size(d)
    for i in range(n):
        s = tp.space_get(d, i)
        buf.poison()
        m = tp.conv2d_run(buf, s, timing_cfg=tm)
        torch.cuda.synchronize()
        if m["status"] != 0 or not np.array_equal(buf.output(), ref):
            bad.append((i, s["kind"], s["bm"], s["bn"], s["bk"], s["stages"], s["split_k"]))
    assert not bad, f"{len(bad)}/{n} timed schedules differ, first: {bad[:5]}"


# ------------------------------------------------------------------ 3xTF32 tensor-core kind
TF32_TINY = [mk(1, 64, 10, 9, 64, 3, 3, 1, 1, dtype=tp.FP32, epi=1),    # ragged M tail
             mk(2, 36, 7, 7, 48, 1, 1, 1, 0, dtype=tp.FP32, epi=1),     # 1x1/s1/p0: tiled A; C = 32 + 4
             mk(1, 4, 9, 11, 40, 3, 3, 2, 1, dtype=tp.FP32, epi=1),     # one partial channel block, stride 2
             mk(1, 96, 6, 7, 256, 3, 3, 1, 1, dtype=tp.FP32, epi=1)]    # BN up to 256, 3 channel blocks


def _tf32_scheds(d):
    out = [tp.space_get(d, i) for i in range(tp.space_size(d))]
    out = [s for s in out if s["kind"] == tp.KIND_IGEMM_TF32X3]
    assert out, "layer has no 3xTF32 schedules"
    return out


@pytest.mark.parametrize("d", TF32_TINY, ids=lambda d: f"tf32_{d['c']}x{d['h']}x{d['w']}_k{d['k']}_r{d['r']}s{d['stride_h']}")
def test_tf32x3_every_schedule_bit_exact_integer(d):
    """Integers in {-3..3} are exact tf32 values (lo parts are 0) and every
    partial sum is an fp32 integer, so every 3xTF32 schedule equals the oracle
    bit-exactly (O11)."""
    x, w, b = datagen.make_inputs(d, 21, integer=True)
    ref = oracle_ref(d, x, w, b)
    buf = tp.LayerBuffers(d, x, w, b)
    bad = []
    for s in _tf32_scheds(d):
        buf.poison()
        tp.conv2d_run(buf, s)
        torch.cuda.synchronize()
        if not np.array_equal(buf.output(), ref):
            bad.append((s["space_index"], s["bm"], s["bn"], s["stages"]))
    assert not bad, f"{len(bad)} tf32 schedules differ, first: {bad[:5]}"


@pytest.mark.parametrize("d", TF32_TINY + [dict(wl.catalog("cfg1")[0], epilogue=3)],
                         ids=lambda d: f"tf32r_{d['c']}x{d['h']}x{d['w']}_k{d['k']}_e{d['epilogue']}")
def test_tf32x3_random_parity_fp32_bar(d):
    """Random fp32 data: the hi/lo split keeps every schedule within the fp32
    bar of north_star (1e-5, reading C10/C11), which a single tf32 product
    (~1e-3) would miss."""
    x, w, b = datagen.make_inputs(d, datagen.data_seed(1, 5))
    ref = oracle_ref(d, x, w, b)
    buf = tp.LayerBuffers(d, x, w, b)
    worst = 0.0
    for s in _tf32_scheds(d):
        buf.poison()
        tp.conv2d_run(buf, s)
        torch.cuda.synchronize()
        err = rel_err(buf.output(), ref)
        worst = max(worst, err)
        assert err <= 1e-5, (s, err)
    assert worst > 0.0 or d["c"] <= 4   # random data does round somewhere


# ------------------------------------------------------------------ stem kind (C < 8: staged patch)
STEM_TINY = [mk(2, 3, 10, 70, 64, 3, 3, 1, 1, out=tp.FP32, epi=1),     # VGG conv1_1-like, 2 images, Q = 70
             mk(1, 3, 23, 140, 64, 7, 7, 2, 3, out=tp.FP32, epi=1),    # R50 conv1-like (7x7 s2 p3), Q = 70
             mk(1, 3, 9, 132, 32, 3, 3, 2, 1, out=tp.FP32, epi=1),     # MobileNetV2 conv0-like (3x3 s2)
             mk(1, 5, 6, 80, 40, 3, 3, 1, 1, out=tp.FP32, epi=1),      # C = 5, K = 40 (ragged N tile)
             # W C % 8 = 0: the 16-byte patch staging mode (rows shifted to 16-byte boundaries)
             mk(2, 3, 10, 72, 64, 3, 3, 1, 1, out=tp.FP32, epi=1),     # VGG conv1_1-like, Q = 72
             mk(1, 3, 23, 136, 64, 7, 7, 2, 3, out=tp.FP32, epi=1),    # R50 conv1-like, Q = 68
             mk(1, 3, 9, 128, 32, 3, 3, 2, 1, out=tp.FP32, epi=1)]     # MobileNetV2 conv0-like, Q = 64


def _stem_scheds(d):
    out = [tp.space_get(d, i) for i in range(tp.space_size(d))]
    out = [s for s in out if s["kind"] == tp.KIND_IGEMM_TC_STEM]
    assert out, "layer has no stem schedules"
    return out


@pytest.mark.parametrize("d", STEM_TINY, ids=lambda d: f"stem_{d['c']}x{d['h']}x{d['w']}_k{d['k']}_r{d['r']}s{d['stride_h']}")
def test_stem_every_schedule_bit_exact_integer(d):
    """O11 for the stem kind: ragged last tile of every output row, zero-padded
    patch borders, several images, every tiles_per_cta (partial last CTA)."""
    x, w, b = datagen.make_inputs(d, 23, integer=True)
    ref = oracle_ref(d, x, w, b)
    buf = tp.LayerBuffers(d, x, w, b)
    bad = []
    for s in _stem_scheds(d):
        buf.poison()
        tp.conv2d_run(buf, s)
        torch.cuda.synchronize()
        if not np.array_equal(buf.output(), ref):
            bad.append((s["space_index"], s["bm"], s["bn"], s["tiles_per_cta"]))
    assert not bad, f"{len(bad)} stem schedules differ, first: {bad[:5]}"


STEM_FULL = [wl.catalog("resnet50")[0], wl.catalog("mobilenetv2")[0]]


@pytest.mark.parametrize("d", STEM_FULL, ids=lambda d: d["name"])
def test_stem_full_size_random_parity(d):
    x, w, b = datagen.make_inputs(d, datagen.data_seed(2, 0))
    ref = oracle_ref(d, x, w, b)
    buf = tp.LayerBuffers(d, x, w, b)
    for s in _stem_scheds(d):
        buf.poison()
        tp.conv2d_run(buf, s, timing_cfg=tp.timing(warmup=1, groups=1, n_min=2, target_group_us=1.0))
        torch.cuda.synchronize()
        assert rel_err(buf.output(), ref) <= 2e-2, s


def test_stem_vgg_conv1_1_sampled_points():
    d = wl.catalog("vgg19_b16")[0]
    x, w, b = datagen.make_inputs(d, datagen.data_seed(4, 0))
    buf = tp.LayerBuffers(d, x, w, b)
    P, Q = tp.output_shape(d)
    idx = datagen.sample_points(d["n"] * d["k"] * P * Q, 4096, 5)
    ref = oc.conv2d_points_c(d, bf16_round(x), bf16_round(w), b, True, idx)
    for s in _stem_scheds(d)[::3]:
        tp.conv2d_run(buf, s)
        torch.cuda.synchronize()
        assert rel_err(buf.gather(idx), ref) <= 2e-2, s


@pytest.mark.parametrize("d", TC_TINY[:3] + [mk(1, 64, 128, 128, 128, 3, 3, 1, 1, out=tp.FP32, epi=1),
                                             mk(1, 64, 40, 40, 96, 1, 1, 1, 0, epi=3)],
                         ids=lambda d: f"ytma_{d['c']}x{d['h']}x{d['w']}_k{d['k']}_r{d['r']}_o{d['out_dtype']}")
def test_tma_store_epilogue_bit_exact_small_partition(d):
    """In a 14-SM partition most split-1 grids have more CTAs than SMs, so the
    staged TMA-store epilogue (TcArgs::y_tma) writes y: every tensor-core
    schedule must still match the oracle (bit-exactly on integers; the bf16
    output case within one bf16 rounding)."""
    part = tp.Partition.get(0.1)
    x, w, b = datagen.make_inputs(d, 29, integer=True)
    ref = oracle_ref(d, x, w, b)
    buf = tp.LayerBuffers(d, x, w, b, part=part)
    bad = []
    for i in range(tp.space_size(d)):
        s = tp.space_get(d, i)
        if s["kind"] not in (tp.KIND_IGEMM_TC, tp.KIND_IGEMM_TC_GATHER) or s["split_k"] != 1:
            continue
        buf.poison()
        tp.conv2d_run(buf, s, part)
        part.sync()
        y = buf.output()
        ok = np.array_equal(y, ref) if d["out_dtype"] == tp.FP32 else rel_err(y, ref) <= 2 ** -8
        if not ok:
            bad.append((i, s["bm"], s["bn"], s["bk"], s["stages"]))
    assert not bad, f"{len(bad)} schedules differ, first: {bad[:5]}"


@pytest.mark.parametrize("d", [mk(2, 128, 4, 57, 24, 3, 3, 1, 1, out=tp.FP32, epi=1),
                               mk(1, 64, 6, 60, 40, 3, 3, 1, 1, epi=3),
                               mk(1, 64, 128, 128, 128, 3, 3, 1, 1, out=tp.FP32, epi=1)],
                         ids=lambda d: f"ytma_mt_{d['c']}x{d['h']}x{d['w']}_k{d['k']}_o{d['out_dtype']}")
def test_multitile_tma_store_epilogue_in_partition(d):
    """Row-halo and multi-tile im2col kinds store y through the staged TMA
    epilogue (3-D [N P][Q][K] map for row tiles, q >= Q clipped): every such
    schedule in a 25% partition matches the oracle (bit-exact for integer data
    with fp32 output, within one bf16 rounding otherwise)."""
    part = tp.Partition.get(0.25)
    x, w, b = datagen.make_inputs(d, 31, integer=True)
    ref = oracle_ref(d, x, w, b)
    buf = tp.LayerBuffers(d, x, w, b, part=part)
    bad, n = [], 0
    for i in range(tp.space_size(d)):
        s = tp.space_get(d, i)
        if s["kind"] not in (tp.KIND_IGEMM_TC_ROW, tp.KIND_IGEMM_TC_ROWW, tp.KIND_IGEMM_TC_MT):
            continue
        n += 1
        buf.poison()
        tp.conv2d_run(buf, s, part)
        part.sync()
        y = buf.output()
        ok = np.array_equal(y, ref) if d["out_dtype"] == tp.FP32 else rel_err(y, ref) <= 2 ** -8
        if not ok:
            bad.append((i, s["kind"], s["bm"], s["bn"], s["stages"], s["tiles_per_cta"]))
    assert n > 0 and not bad, f"{len(bad)}/{n} schedules differ, first: {bad[:5]}"


@pytest.mark.parametrize("d", [mk(2, 128, 4, 57, 24, 3, 3, 1, 1, out=tp.FP32, epi=1),
                               mk(1, 64, 6, 60, 40, 3, 3, 1, 1, out=tp.FP32, epi=1),
                               STEM_TINY[0], STEM_TINY[1]],
                         ids=lambda d: f"slots_{d['c']}x{d['h']}x{d['w']}_k{d['k']}_r{d['r']}")
@pytest.mark.parametrize("sm_tuned", [1, 3, 7])
def test_multitile_balanced_spans_bit_exact(d, sm_tuned):
    """Multi-tile kinds (row-halo, multi-tile im2col, stem): when the frozen
    grid has more CTA columns than the tuned partition holds (sm_tuned x
    CTAs/SM / grid.y), the resident CTAs take balanced tile spans of uneven
    length and the rest exit (TcArgs::slots).  Every such schedule, frozen at
    a few SMs so that the spans are ragged, must match the oracle bit-exactly."""
    x, w, b = datagen.make_inputs(d, 37, integer=True)
    ref = oracle_ref(d, x, w, b)
    buf = tp.LayerBuffers(d, x, w, b)
    bad, n = [], 0
    for i in range(tp.space_size(d)):
        s = tp.space_get(d, i)
        if s["kind"] not in (tp.KIND_IGEMM_TC_ROW, tp.KIND_IGEMM_TC_ROWW, tp.KIND_IGEMM_TC_MT, tp.KIND_IGEMM_TC_STEM) or \
                s["tiles_per_cta"] < 2:
            continue
        s = dict(s, sm_tuned=sm_tuned)
        n += 1
        buf.poison()
        tp.conv2d_run(buf, s)
        torch.cuda.synchronize()
        if not np.array_equal(buf.output(), ref):
            bad.append((i, s["kind"], s["bm"], s["bn"], s["tiles_per_cta"]))
    assert n > 0 and not bad, f"{len(bad)}/{n} schedules differ, first: {bad[:5]}"
