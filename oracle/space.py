"""CPU enumeration of the v0 schedule space -- TEST INFRASTRUCTURE ONLY.

Independent Python mirror of the schedule space that ``libtp`` enumerates in
C++ (paper_2008_03602_b200/csrc/space.cpp).  The two share no code; both are
written from the declarative knob table in DESIGN.md section "Schedule space
v0".  ``north_star`` requires "schedule selection and indexing must be
bit-exact against a CPU enumeration of the same search space"; this module is
that CPU enumeration (SURVEY.md 8(c) check P-S).

Paper basis: the knobs a conv2d autotuner searches are "loop tiles and
ordering, caching, and loop unrolling ... CUDA threading";
the first batch is random when no training data exists; selection
keeps the fastest profiled configuration.  Readings C13
(tie -> lowest index), C16 (trials = distinct candidates, >= |space| means
exhaustive) and C17 (SplitMix64 + partial Fisher-Yates) are DESIGN.md's.
"""
from __future__ import annotations

import itertools
import math

KIND_IGEMM_TC = 0
KIND_DIRECT = 1
KIND_IGEMM_TC_GATHER = 2
KIND_IGEMM_TC_ROW = 3
KIND_IGEMM_TC_MT = 4
KIND_IGEMM_TF32X3 = 5
KIND_IGEMM_TC_STEM = 6
KIND_IGEMM_TC_STRIP = 7
KIND_IGEMM_TC_ROWW = 8
DTYPE_BF16 = 0
DTYPE_FP32 = 1
SMEM_LIMIT = 232448          # 227 KiB usable per CTA on sm_100a

TC_KNOBS = (("bm", (64, 128)), ("bn", (32, 64, 128, 256)), ("bk", (16, 32, 64, 128)),
            ("stages", (2, 3, 4, 6)), ("threads", (128, 256)), ("split_k", (1, 2, 4, 8)))
ROW_KNOBS = (("bm", (64, 128)), ("bn", (32, 64, 128, 256)), ("stages", (1, 2, 3)), ("threads", (128, 256)),
             ("tiles_per_cta", (1, 2, 4, 8, 16)))
MT_KNOBS = (("bm", (64, 128)), ("bn", (32, 64, 128, 256)), ("stages", (2, 3, 4)), ("tiles_per_cta", (2, 4, 8)))
STEM_KNOBS = (("bm", (64, 128)), ("bn", (32, 64, 128)), ("tiles_per_cta", (2, 4, 8, 16)))
ROWW_KNOBS = (("bm", (64, 128)), ("bn", (32, 64, 128, 256)), ("stages", (2, 4, 6, 8)), ("tiles_per_cta", (2, 4, 8, 16)))
STRIP_KNOBS = (("bm", (64, 128)), ("bn", (32, 64, 128)), ("stages", (2, 4, 6)), ("tiles_per_cta", (1, 2, 4, 8, 16)))
TF32_KNOBS = (("bm", (64, 128)), ("bn", (32, 64, 128, 256)), ("stages", (2, 3, 4)), ("split_k", (1, 2, 4, 8)))
DIRECT_KNOBS = (("threads", (64, 128, 256, 512)), ("tile_q", (1, 2, 4)), ("vec_k", (1, 2, 4, 8)),
                ("tile_p", (1, 2, 4, 8)), ("smem_stage", (0, 1)))


def _np2(v: int) -> int:
    p = 1
    while p < v:
        p *= 2
    return p


def _cdiv(a: int, b: int) -> int:
    return -(-a // b)


def out_pq(d: dict) -> tuple[int, int]:
    P = (d["h"] + 2 * d["pad_h"] - d.get("dil_h", 1) * (d["r"] - 1) - 1) // d["stride_h"] + 1
    Q = (d["w"] + 2 * d["pad_w"] - d.get("dil_w", 1) * (d["s"] - 1) - 1) // d["stride_w"] + 1
    return P, Q


def layer_kind(d: dict) -> int:
    """One kind per layer: bf16 dense (g = 1, d = 1,
    K % 8 == 0) layers go to the tensor cores -- TMA im2col when C % 8 == 0,
    the gathered variant otherwise; everything else to the CUDA cores."""
    dense_bf16 = (d["dtype"] == DTYPE_BF16 and d.get("groups", 1) == 1 and d["k"] % 8 == 0
                  and d.get("dil_h", 1) == 1 and d.get("dil_w", 1) == 1)
    if not dense_bf16:
        return KIND_DIRECT
    return KIND_IGEMM_TC if d["c"] % 8 == 0 else KIND_IGEMM_TC_GATHER


def direct_lanes(d: dict, threads: int, tile_q: int, vec_k: int, tile_p: int) -> tuple[int, int]:
    """(lanes_k, lanes_q): threads are split into lanes along K (power of two,
    capped so every output row of the CTA gets at least one thread) and Q."""
    kv = _cdiv(d["k"], vec_k)
    lanes_k = min(_np2(kv), threads // tile_p)
    lanes_q = threads // (lanes_k * tile_p)
    return lanes_k, lanes_q


def direct_smem_bytes(d: dict, threads: int, tile_q: int, vec_k: int, tile_p: int) -> int:
    lanes_k, lanes_q = direct_lanes(d, threads, tile_q, vec_k, tile_p)
    qt, kt = lanes_q * tile_q, lanes_k * vec_k
    rows_in = (tile_p - 1) * d["stride_h"] + d["r"]
    cols_in = (qt - 1) * d["stride_w"] + d["s"]
    if d.get("groups", 1) == 1:
        cc = min(d["c"], 16)
        return 4 * (rows_in * cols_in * cc + d["r"] * d["s"] * cc * kt)
    return 4 * (rows_in * cols_in * kt + d["r"] * d["s"] * kt)


def _valid_tc(d: dict, bm, bn, bk, stages, threads, split_k) -> bool:
    P, Q = out_pq(d)
    M = d["n"] * P * Q
    if stages * (bm + bn) * bk * 2 + 1024 > SMEM_LIMIT:
        return False
    if bn > max(32, _np2(d["k"])) or bm > max(64, _np2(M)) or bk > max(16, _np2(d["c"])):
        return False
    return split_k <= d["r"] * d["s"] * _cdiv(d["c"], bk)


def _valid_tc_gather(d: dict, bm, bn, bk, stages, threads, split_k) -> bool:
    """Gathered tensor-core kind: reduction axis = R*S*C flattened; shared
    memory also holds a 16-B-per-row pixel table and an 8-B-per-k table over
    the k-blocks' padded extent."""
    P, Q = out_pq(d)
    M = d["n"] * P * Q
    kg = d["r"] * d["s"] * d["c"]
    nkb = _cdiv(kg, bk)
    if stages * (bm + bn) * bk * 2 + 1024 + 16 * bm + 8 * nkb * bk > SMEM_LIMIT:
        return False
    if bn > max(32, _np2(d["k"])) or bm > max(64, _np2(M)) or bk > max(16, _np2(kg)):
        return False
    return split_k <= nkb


def row_eligible(d: dict) -> bool:
    """Row-halo kind: TMA-kind layers with a 3x3 filter,
    stride 1, pad 1, C a multiple of 64 and output rows at least 56 wide."""
    P, Q = out_pq(d)
    return (layer_kind(d) == KIND_IGEMM_TC and d["r"] == 3 and d["s"] == 3 and d["stride_h"] == 1
            and d["stride_w"] == 1 and d["pad_h"] == 1 and d["pad_w"] == 1 and d["c"] % 64 == 0 and Q >= 56)


def _valid_row(d: dict, bm, bn, stages, threads, tiles_per_cta) -> bool:
    """Stage = input strip of bm+2 pixels x 128 B (rounded up to 1 KiB) + the
    three taps' bn x 64-channel weight tiles; several tiles per CTA need the
    256-thread layout (six draining warps)."""
    P, Q = out_pq(d)
    strip = -(-((bm + 2) * 128) // 1024) * 1024
    if stages * (strip + 3 * bn * 128) + 1024 > SMEM_LIMIT:
        return False
    if tiles_per_cta > 1 and threads != 256:
        return False
    return bm <= _np2(Q) and bn <= max(32, _np2(d["k"]))


def mt_eligible(d: dict) -> bool:
    """Multi-tile im2col kind: TMA-kind layers with at least 1024 tiles of 64 x 32."""
    P, Q = out_pq(d)
    return layer_kind(d) == KIND_IGEMM_TC and _cdiv(d["n"] * P * Q, 64) * _cdiv(d["k"], 32) >= 1024


def _valid_mt(d: dict, bm, bn, stages, tiles_per_cta) -> bool:
    """BK = 64: smem = stages (bm + bn) 64 2 + 1024; tile bounds as the TMA kind."""
    P, Q = out_pq(d)
    if stages * (bm + bn) * 64 * 2 + 1024 > SMEM_LIMIT:
        return False
    return bn <= max(32, _np2(d["k"])) and bm <= max(64, _np2(d["n"] * P * Q)) and 64 <= max(16, _np2(d["c"]))


def _valid_direct(d: dict, threads, tile_q, vec_k, tile_p, smem_stage) -> bool:
    P, Q = out_pq(d)
    if tile_q > Q or tile_p > P or vec_k > d["k"]:
        return False
    if d.get("groups", 1) != 1 and d["c"] % vec_k != 0:
        return False
    if smem_stage and direct_smem_bytes(d, threads, tile_q, vec_k, tile_p) > SMEM_LIMIT:
        return False
    return True


def stem_eligible(d: dict) -> bool:
    """Stem kind: gathered (C % 8 != 0) tensor-core layers with C <= 8, R S C <= 256
    and output rows at least 64 wide."""
    P, Q = out_pq(d)
    return (layer_kind(d) == KIND_IGEMM_TC_GATHER and d["c"] <= 8 and d["r"] * d["s"] * d["c"] <= 256
            and Q >= 64)


def stem_kp(d: dict) -> int:
    return _cdiv(d["r"] * d["s"] * d["c"], 64) * 64


def _valid_stem(d: dict, bm: int, bn: int, tiles_per_cta: int) -> bool:
    # resident weights bn x KP, two im2col tiles bm x KP (bf16), two input patches of
    # R rows x ((bm-1) s_w + S) C + 2 bf16 each rounded up to 1 KiB, the KP-entry k table, barriers
    P, Q = out_pq(d)
    kp = stem_kp(d)
    cols = (bm - 1) * d["stride_w"] + d["s"]
    prow = (cols * d["c"] + 3) // 2 * 2          # even row pitch >= cols C + 1 (a row starts on a word)
    patch = 2 * _cdiv(d["r"] * prow * 2, 1024) * 1024   # two buffers
    stage = bm * bn * 4                          # output staging of the TMA-store epilogue (fp32 size)
    if bn * kp * 2 + 2 * bm * kp * 2 + patch + _cdiv(kp * 4, 1024) * 1024 + stage + 1024 > SMEM_LIMIT:
        return False
    return bm <= _np2(Q) and bn <= max(32, _np2(d["k"]))


def roww_eligible(d: dict) -> bool:
    """Row-halo kind with resident weights: row-halo layers with C = 64."""
    return row_eligible(d) and d["c"] == 64


def _valid_roww(d: dict, bm: int, bn: int, stages: int, tiles_per_cta: int) -> bool:
    # stages input strips of (bm + 2) x 128 B (each rounded up to 1 KiB) + the nine taps' weight
    # tiles bn x 128 B + 1 KiB of barriers
    P, Q = out_pq(d)
    strip = _cdiv((bm + 2) * 128, 1024) * 1024
    if stages * strip + 9 * bn * 128 + 1024 > SMEM_LIMIT:
        return False
    return bm <= _np2(Q) and bn <= max(32, _np2(d["k"]))


def strip_eligible(d: dict) -> bool:
    """Strip kind: gathered layers with C <= 8, column
    stride 1 or 2 and filters of at most 8 x 8."""
    return (layer_kind(d) == KIND_IGEMM_TC_GATHER and d["c"] <= 8 and d["stride_w"] in (1, 2)
            and d["s"] <= 8 and d["r"] <= 8)


def _valid_strip(d: dict, bm: int, bn: int, stages: int, tiles_per_cta: int) -> bool:
    # one ring stage = the strip of (bm + 2 ceil(T0 / 2) - 1) 16-byte pixels (T0 = ceil(S / s_w)
    # taps in phase 0): with s_w = 1 whole 512-byte boxes, with s_w = 2 one box per phase rounded
    # up to 128 B; resident weights: R rows of (S + s_w) taps x bn rows x 16 B, rounded up to
    # 1 KiB; + 1 KiB of barriers
    P, Q = out_pq(d)
    sw = d["stride_w"]
    px = bm + 2 * _cdiv(_cdiv(d["s"], sw), 2) - 1
    if sw * px > 256:                # a TMA box spans at most 256 elements per dimension
        return False
    stage = _cdiv(px * 16, 512) * 512 if sw == 1 else sw * _cdiv(px * 16, 128) * 128
    weights = _cdiv(d["r"] * (d["s"] + sw) * bn * 16, 1024) * 1024
    if stages * stage + weights + 1024 > SMEM_LIMIT:
        return False
    return bm <= max(64, _np2(Q)) and bn <= max(32, _np2(d["k"]))


def tf32_eligible(d: dict) -> bool:
    """3xTF32 tensor-core kind: fp32 dense layers whose NHWC
    pixel rows are 16-byte multiples (C % 4 == 0) and K % 8 == 0."""
    return (layer_kind(d) == KIND_DIRECT and d["dtype"] == DTYPE_FP32 and d.get("groups", 1) == 1
            and d["c"] % 4 == 0 and d["k"] % 8 == 0)


def _valid_tf32(d: dict, bm: int, bn: int, stages: int, split_k: int) -> bool:
    # ring: stages x (A + B) tiles of 32 fp32 channels (128-B rows), hi and lo copies;
    # split-K adds the cluster receive buffer of bm rows x (bn + 4) fp32
    P, Q = out_pq(d)
    recv = bm * (bn + 4) * 4 if split_k > 1 else 0
    if stages * (bm + bn) * 32 * 4 * 2 + recv + 1024 > SMEM_LIMIT:
        return False
    if bn > max(32, _np2(d["k"])):
        return False
    if bm > max(64, _np2(d["n"] * P * Q)):
        return False
    return split_k <= d["r"] * d["s"] * _cdiv(d["c"], 32)


def enumerate_space(d: dict) -> list[dict]:
    """Valid schedules in lexicographic knob order (outermost knob first);
    ``space_index`` is the rank among the valid tuples."""
    kind = layer_kind(d)
    knobs, valid = {KIND_IGEMM_TC: (TC_KNOBS, _valid_tc), KIND_IGEMM_TC_GATHER: (TC_KNOBS, _valid_tc_gather),
                    KIND_DIRECT: (DIRECT_KNOBS, _valid_direct)}[kind]
    names = [k for k, _ in knobs]
    out = []
    for combo in itertools.product(*[v for _, v in knobs]):
        if valid(d, *combo):
            s = dict(zip(names, combo))
            s["kind"] = kind
            s["space_index"] = len(out)
            s.update(geometry(d, s))
            out.append(s)
    if row_eligible(d):          # appended after every TMA-kind tuple; bk = 64, split_k = 1
        for combo in itertools.product(*[v for _, v in ROW_KNOBS]):
            if _valid_row(d, *combo):
                s = dict(zip([k for k, _ in ROW_KNOBS], combo), bk=64, split_k=1, kind=KIND_IGEMM_TC_ROW,
                         space_index=len(out))
                s.update(geometry(d, s))
                out.append(s)
    if roww_eligible(d):         # after the row-halo tuples; bk = 64, threads = 256, split_k = 1
        for combo in itertools.product(*[v for _, v in ROWW_KNOBS]):
            if _valid_roww(d, *combo):
                s = dict(zip([k for k, _ in ROWW_KNOBS], combo), bk=64, threads=256, split_k=1,
                         kind=KIND_IGEMM_TC_ROWW, space_index=len(out))
                s.update(geometry(d, s))
                out.append(s)
    if tf32_eligible(d):         # appended after the direct tuples; bk = 32, threads = 256, split_k = 1
        for combo in itertools.product(*[v for _, v in TF32_KNOBS]):
            if _valid_tf32(d, *combo):
                s = dict(zip([k for k, _ in TF32_KNOBS], combo), bk=32, threads=256,
                         kind=KIND_IGEMM_TF32X3, space_index=len(out))
                s.update(geometry(d, s))
                out.append(s)
    if stem_eligible(d):         # after the gathered tuples; bk = KP, stages = 2, threads = 256, split_k = 1
        for combo in itertools.product(*[v for _, v in STEM_KNOBS]):
            if _valid_stem(d, *combo):
                s = dict(zip([k for k, _ in STEM_KNOBS], combo), bk=stem_kp(d), stages=2, threads=256, split_k=1,
                         kind=KIND_IGEMM_TC_STEM, space_index=len(out))
                s.update(geometry(d, s))
                out.append(s)
    if strip_eligible(d):        # after the stem tuples; bk = 16, threads = 256, split_k = 1
        for combo in itertools.product(*[v for _, v in STRIP_KNOBS]):
            if _valid_strip(d, *combo):
                s = dict(zip([k for k, _ in STRIP_KNOBS], combo), bk=16, threads=256, split_k=1,
                         kind=KIND_IGEMM_TC_STRIP, space_index=len(out))
                s.update(geometry(d, s))
                out.append(s)
    if mt_eligible(d):           # appended last; threads = 256, bk = 64, split_k = 1
        for combo in itertools.product(*[v for _, v in MT_KNOBS]):
            if _valid_mt(d, *combo):
                s = dict(zip([k for k, _ in MT_KNOBS], combo), bk=64, threads=256, split_k=1,
                         kind=KIND_IGEMM_TC_MT, space_index=len(out))
                s.update(geometry(d, s))
                out.append(s)
    return out


def geometry(d: dict, s: dict) -> dict:
    """Frozen launch geometry of a schedule (grid, threads per CTA)."""
    P, Q = out_pq(d)
    if s.get("kind") == KIND_IGEMM_TC_MT:
        g = (_cdiv(_cdiv(d["n"] * P * Q, s["bm"]), s["tiles_per_cta"]), _cdiv(d["k"], s["bn"]), 1)
    elif s.get("kind") in (KIND_IGEMM_TC_STEM, KIND_IGEMM_TC_STRIP):
        g = (_cdiv(d["n"] * P * _cdiv(Q, s["bm"]), s["tiles_per_cta"]), _cdiv(d["k"], s["bn"]), 1)
    elif s.get("kind") in (KIND_IGEMM_TC_ROW, KIND_IGEMM_TC_ROWW):
        g = (_cdiv(d["n"] * P * _cdiv(Q, s["bm"]), s["tiles_per_cta"]), _cdiv(d["k"], s["bn"]), 1)
    elif s.get("kind", layer_kind(d)) in (KIND_IGEMM_TC, KIND_IGEMM_TC_GATHER, KIND_IGEMM_TF32X3):
        M = d["n"] * P * Q
        g = (_cdiv(M, s["bm"]), _cdiv(d["k"], s["bn"]), s["split_k"])
    else:
        lanes_k, lanes_q = direct_lanes(d, s["threads"], s["tile_q"], s["vec_k"], s["tile_p"])
        g = (_cdiv(Q, lanes_q * s["tile_q"]) * _cdiv(P, s["tile_p"]),
             _cdiv(d["k"], lanes_k * s["vec_k"]), d["n"])
    return {"grid_x": g[0], "grid_y": g[1], "grid_z": g[2], "threads_per_cta": s["threads"],
            "ctas": g[0] * g[1] * g[2]}


def waves(ctas: int, sm_granted: int, ctas_per_sm: int) -> int:
    """Waves = ceil(CTAs / (SM_granted * CTAs_per_SM))."""
    return _cdiv(ctas, sm_granted * max(1, ctas_per_sm))


MASK64 = (1 << 64) - 1


def splitmix64(state: int):
    """Generator of SplitMix64 outputs from ``state`` (C17)."""
    while True:
        state = (state + 0x9E3779B97F4A7C15) & MASK64
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        yield z ^ (z >> 31)


def sample(n_space: int, trials: int, seed: int) -> list[int]:
    """trials >= |space| -> all of it in order; else partial Fisher-Yates over
    0..n-1 driven by SplitMix64(seed), j = i + next() mod (n - i)."""
    if trials >= n_space:
        return list(range(n_space))
    a = list(range(n_space))
    rng = splitmix64(seed & MASK64)
    for i in range(trials):
        j = i + next(rng) % (n_space - i)
        a[i], a[j] = a[j], a[i]
    return a[:trials]


def argmin(records: list[dict]) -> int:
    """Index into ``records`` of the best OK record: min median_us, ties to the
    lowest space_index (C13). Returns -1 if none is OK."""
    best = -1
    for i, r in enumerate(records):
        if r["status"] != 0:
            continue
        if best < 0:
            best = i
            continue
        b = records[best]
        if r["median_us"] < b["median_us"] or (r["median_us"] == b["median_us"]
                                               and r["space_index"] < b["space_index"]):
            best = i
    return best


def requested_sms(fraction: float, total_sms: int = 148) -> int:
    """requested = floor(total * p) (C14; SPEC's floor rule); 1.0 -> whole device."""
    return max(1, int(math.floor(total_sms * fraction + 1e-9)))
