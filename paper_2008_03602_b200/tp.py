"""Thin ctypes binding of libtp (include/tp.h).  Argument marshalling only:
every step of the hot path runs in libtp's CUDA kernels.  PyTorch is used for
device memory (tensor allocation) and nothing else.

Raises ImportError at import time if libtp.so has not been built -- there is
no CPU fallback (build with ``python -m paper_2008_03602_b200.build`` or
``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

# Concurrent tuners (one green-context stream each) need more
# hardware work queues than the default 8; read when the CUDA context is
# created, so it only takes effect if libtp is imported before CUDA starts.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtp.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"libtp.so not found at {LIB_PATH}: build it first (__graft_entry__.build()); "
                      "there is no CPU fallback")
_lib = ctypes.CDLL(LIB_PATH)

OK, EINVAL, EINVALID_CONFIG, ECAPACITY, ECUDA, EMISMATCH, EUNSUPPORTED = range(7)
(KIND_IGEMM_TC, KIND_DIRECT, KIND_IGEMM_TC_GATHER, KIND_IGEMM_TC_ROW, KIND_IGEMM_TC_MT, KIND_IGEMM_TF32X3,
 KIND_IGEMM_TC_STEM, KIND_IGEMM_TC_STRIP, KIND_IGEMM_TC_ROWW) = range(9)
NHWC, NCHW = 0, 1
BF16, FP32 = 0, 1
PART_FINE_GRAINED = 1

DESC_FIELDS = ("n", "c", "h", "w", "k", "r", "s", "stride_h", "stride_w", "pad_h", "pad_w", "dil_h", "dil_w",
               "groups", "in_layout", "dtype", "out_dtype", "epilogue")


class ConvDesc(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int32) for f in DESC_FIELDS]


class Schedule(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int32) for f in ("kind", "bm", "bn", "bk", "stages", "threads", "split_k", "tile_q",
                                              "vec_k", "tile_p", "smem_stage", "tiles_per_cta")] + \
               [("space_index", ctypes.c_int64)] + \
               [(f, ctypes.c_int32) for f in ("grid_x", "grid_y", "grid_z", "sm_tuned")]


class Measurement(ctypes.Structure):
    _fields_ = [(f, ctypes.c_double) for f in ("median_us", "min_us", "mean_us", "std_us")] + \
               [(f, ctypes.c_int32) for f in ("n_per_group", "groups", "sm_requested", "sm_granted", "device",
                                              "status")] + \
               [("space_index", ctypes.c_int64), ("ctas", ctypes.c_int64)] + \
               [(f, ctypes.c_int32) for f in ("threads_per_cta", "waves", "ctas_per_sm", "kind")] + \
               [("max_abs_err", ctypes.c_double), ("max_ref", ctypes.c_double)]


class Timing(ctypes.Structure):
    _fields_ = [("warmup", ctypes.c_int32), ("groups", ctypes.c_int32), ("n_min", ctypes.c_int32),
                ("target_group_us", ctypes.c_double), ("use_graph", ctypes.c_int32), ("flush_l2", ctypes.c_int32),
                ("prune_ratio", ctypes.c_double)]


_P = ctypes.POINTER
_vp, _i32, _i64, _u64, _dbl, _sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_size_t


def _sig(name, *args):
    fn = getattr(_lib, name)
    fn.argtypes = list(args)
    fn.restype = ctypes.c_int
    return fn


_sig("tp_init", _i32)
_lib.tp_shutdown.restype = None
_lib.tp_status_str.restype = ctypes.c_char_p
_lib.tp_status_str.argtypes = [ctypes.c_int]
_lib.tp_last_error.restype = ctypes.c_char_p
_lib.tp_launch_count.restype = ctypes.c_int64
_sig("tp_partition_get", _i32, _dbl, _i32, _P(_vp), _P(_i32), _P(_i32))
_sig("tp_partition_split", _i32, _i32, _i32, _i32, _P(_vp), _P(_i32))
_sig("tp_partition_shared", _i32, _i32, _P(_vp))
_sig("tp_partition_info", _vp, _P(_i32), _P(_i32), _P(_i32), _P(_vp))
_sig("tp_partition_sync", _vp)
_sig("tp_partition_close", _vp)
_sig("tp_partition_probe", _vp, _i32, _vp)
_sig("tp_partition_floor", _vp, _i32, _i32, _P(Timing), _P(Measurement))
_sig("tp_partition_copy_bw", _vp, _vp, _vp, _sz, _i32, _P(_dbl))
_sig("tp_output_shape", _P(ConvDesc), _P(_i32), _P(_i32))
_sig("tp_layer_kind", _P(ConvDesc), _P(_i32))
_sig("tp_space_size", _P(ConvDesc), _P(_i64))
_sig("tp_space_get", _P(ConvDesc), _i64, _P(Schedule))
_sig("tp_space_sample", _P(ConvDesc), _i32, _u64, _P(_i64), _i32, _P(_i32))
_sig("tp_select_best", _P(Measurement), _i32, _P(_i32))
_sig("tp_gate_points", _P(ConvDesc), _i32, _P(_i64), _i32, _P(_i32))
_sig("tp_partition_open", _i32, _dbl, _i32, _P(_vp), _P(_i32))
_sig("tp_partition_stream", _vp, _P(_vp))
_sig("tp_conv2d_run_at", _P(ConvDesc), _P(Schedule), _dbl, _vp, _vp, _vp, _vp, _vp, _sz, _P(Timing), _P(Measurement))
_sig("tp_tune_at", _P(ConvDesc), _dbl, _i32, _u64, _vp, _vp, _vp, _vp, _vp, _sz, _P(_i64), _P(_dbl), _i32, _dbl,
     _P(Timing), _P(Schedule), _P(Measurement), _P(Measurement), _i32, _P(_i32))
_sig("tp_cross_eval_at", _P(ConvDesc), _P(Schedule), _dbl, _vp, _vp, _vp, _vp, _vp, _sz, _P(Timing), _P(Measurement))
_sig("tp_workspace_size", _P(ConvDesc), _P(Schedule), _P(_sz))
_sig("tp_workspace_size_max", _P(ConvDesc), _P(_sz))
_sig("tp_conv2d_run", _P(ConvDesc), _P(Schedule), _vp, _vp, _vp, _vp, _vp, _vp, _sz, _P(Timing), _P(Measurement))
_sig("tp_tune", _P(ConvDesc), _vp, _i32, _u64, _vp, _vp, _vp, _vp, _vp, _sz, _P(_i64), _P(_dbl), _i32, _dbl,
     _P(Timing), _P(Schedule), _P(Measurement), _P(Measurement), _i32, _P(_i32))
_sig("tp_tune_subset", _P(ConvDesc), _vp, _P(_i64), _i32, _vp, _vp, _vp, _vp, _vp, _sz, _P(_i64), _P(_dbl), _i32,
     _dbl, _P(Timing), _P(Measurement), _i32, _P(_i32))
_sig("tp_search_next", _P(ConvDesc), _i32, _P(_i64), _P(_dbl), _i32, _i32, _dbl, _u64, _P(_i64), _P(_i32))
_sig("tp_tune_guided", _P(ConvDesc), _vp, _i32, _i32, _dbl, _u64, _vp, _vp, _vp, _vp, _vp, _sz, _P(_i64), _P(_dbl),
     _i32, _dbl, _P(Timing), _P(Schedule), _P(Measurement), _P(Measurement), _i32, _P(_i32))
_sig("tp_tune_guided_es", _P(ConvDesc), _vp, _i32, _i32, _dbl, _u64, _i32, _vp, _vp, _vp, _vp, _vp, _sz, _P(_i64),
     _P(_dbl), _i32, _dbl, _P(Timing), _P(Schedule), _P(Measurement), _P(Measurement), _i32, _P(_i32))
_lib.tp_search_should_stop.argtypes = [_P(_dbl), _i32, _i32]
_lib.tp_search_should_stop.restype = _i32
_sig("tp_cross_eval", _P(ConvDesc), _P(Schedule), _vp, _vp, _vp, _vp, _vp, _vp, _sz, _P(Timing), _P(Measurement))
_sig("tp_conv2d_trace", _P(ConvDesc), _P(Schedule), _vp, _vp, _vp, _vp, _vp, _vp, _sz, _P(_u64), _i32, _P(_i32))
_sig("tp_chain_run", _i32, _P(ConvDesc), _P(Schedule), _vp, _P(_vp), _P(_vp), _P(_vp), _P(_vp), _P(_vp), _P(_sz), _i32,
     _P(Timing), _P(Measurement))
_sig("tp_pack_input", _P(ConvDesc), _vp, _vp, _vp)
_sig("tp_pack_weights", _P(ConvDesc), _vp, _vp, _vp)
_sig("tp_gather_output", _P(ConvDesc), _vp, _vp, _P(_i64), _i32, _P(_dbl))


class TPError(RuntimeError):
    def __init__(self, status: int, fn: str):
        self.status = status
        msg = _lib.tp_last_error().decode(errors="replace")
        super().__init__(f"{fn}: {_lib.tp_status_str(status).decode()} ({status}): {msg}")


def _ck(status: int, fn: str):
    if status != OK:
        raise TPError(status, fn)


# --------------------------------------------------------------------- structs <-> dicts
def desc(d: dict) -> ConvDesc:
    defaults = {"dil_h": 1, "dil_w": 1, "groups": 1, "in_layout": NHWC, "epilogue": 0}
    vals = []
    for f in DESC_FIELDS:
        if f in d:
            vals.append(int(d[f]))
        elif f in ("stride_h", "stride_w") and "stride" in d:
            vals.append(int(d["stride"]))
        elif f in ("pad_h", "pad_w") and "pad" in d:
            vals.append(int(d["pad"]))
        elif f == "out_dtype":
            vals.append(int(d["dtype"]))
        else:
            vals.append(defaults[f])
    return ConvDesc(*vals)


def sched_to_dict(s: Schedule) -> dict:
    return {f: getattr(s, f) for f, _ in Schedule._fields_}


def dict_to_sched(d: dict) -> Schedule:
    s = Schedule()
    for f, _ in Schedule._fields_:
        if f in d:
            setattr(s, f, int(d[f]))
    return s


def meas_to_dict(m: Measurement) -> dict:
    return {f: getattr(m, f) for f, _ in Measurement._fields_}


def dict_to_meas(d: dict) -> Measurement:
    m = Measurement()
    for f, _ in Measurement._fields_:
        if f in d:
            setattr(m, f, d[f])
    return m


# --------------------------------------------------------------------- host-only
def output_shape(d: dict) -> tuple[int, int]:
    p, q = _i32(), _i32()
    _ck(_lib.tp_output_shape(ctypes.byref(desc(d)), ctypes.byref(p), ctypes.byref(q)), "tp_output_shape")
    return p.value, q.value


def layer_kind(d: dict) -> int:
    k = _i32()
    _ck(_lib.tp_layer_kind(ctypes.byref(desc(d)), ctypes.byref(k)), "tp_layer_kind")
    return k.value


def space_size(d: dict) -> int:
    n = _i64()
    _ck(_lib.tp_space_size(ctypes.byref(desc(d)), ctypes.byref(n)), "tp_space_size")
    return n.value


def space_get(d: dict, idx: int) -> dict:
    s = Schedule()
    _ck(_lib.tp_space_get(ctypes.byref(desc(d)), int(idx), ctypes.byref(s)), "tp_space_get")
    return sched_to_dict(s)


def space_sample(d: dict, trials: int, seed: int) -> list[int]:
    cap = max(1, min(trials, space_size(d)))
    out = (_i64 * cap)()
    n = _i32()
    _ck(_lib.tp_space_sample(ctypes.byref(desc(d)), int(trials), int(seed) & (2**64 - 1), out, cap,
                             ctypes.byref(n)), "tp_space_sample")
    return list(out[:n.value])


def select_best(records: list[dict]) -> int:
    arr = (Measurement * max(1, len(records)))()
    for i, r in enumerate(records):
        arr[i] = dict_to_meas(r)
    b = _i32()
    _ck(_lib.tp_select_best(arr, len(records), ctypes.byref(b)), "tp_select_best")
    return b.value


def gate_points(d: dict, n: int = 4096) -> np.ndarray:
    """The consensus gate's fallback check points (flat NKPQ indices, sorted)."""
    out = np.empty(max(1, n), dtype=np.int64)
    m = _i32()
    _ck(_lib.tp_gate_points(ctypes.byref(desc(d)), int(n), out.ctypes.data_as(_P(_i64)), out.shape[0],
                            ctypes.byref(m)), "tp_gate_points")
    return out[:m.value].copy()


def search_next(d: dict, sm_granted: int, measured_idx, measured_us, batch: int, explore: float = 0.25,
                seed: int = 42) -> list[int]:
    """Next batch of space indices from the model-guided search (host-only)."""
    mi = np.ascontiguousarray(measured_idx, dtype=np.int64)
    mu = np.ascontiguousarray(measured_us, dtype=np.float64)
    out = (_i64 * max(1, batch))()
    n = _i32()
    _ck(_lib.tp_search_next(ctypes.byref(desc(d)), int(sm_granted), mi.ctypes.data_as(_P(_i64)),
                            mu.ctypes.data_as(_P(_dbl)), int(mi.shape[0]), int(batch), float(explore),
                            int(seed) & (2**64 - 1), out, ctypes.byref(n)), "tp_search_next")
    return list(out[:n.value])


def workspace_size(d: dict, sched: dict | None = None) -> int:
    n = _sz()
    if sched is None:
        _ck(_lib.tp_workspace_size_max(ctypes.byref(desc(d)), ctypes.byref(n)), "tp_workspace_size_max")
    else:
        _ck(_lib.tp_workspace_size(ctypes.byref(desc(d)), ctypes.byref(dict_to_sched(sched)), ctypes.byref(n)),
            "tp_workspace_size")
    return n.value


def launch_count() -> int:
    return int(_lib.tp_launch_count())


# --------------------------------------------------------------------- GPU
def init(device: int = 0):
    _ck(_lib.tp_init(device), "tp_init")


def shutdown():
    _lib.tp_shutdown()


def timing(warmup=3, groups=5, n_min=10, target_group_us=20.0, use_graph=1, flush_l2=0, prune_ratio=2.0) -> Timing:
    return Timing(warmup, groups, n_min, target_group_us, use_graph, flush_l2, prune_ratio)


def device_sm_count(device: int = 0) -> int:
    """SMs of the device: the granted count of its whole-device partition."""
    rq, gr, h = _i32(), _i32(), _vp()
    _ck(_lib.tp_partition_get(device, 1.0, 0, ctypes.byref(h), ctypes.byref(rq), ctypes.byref(gr)),
        "tp_partition_get")
    return gr.value


@dataclass
class Partition:
    handle: int
    device: int
    sm_requested: int
    sm_granted: int
    fraction: float
    owned: bool = False

    @classmethod
    def get(cls, fraction: float, device: int = 0, flags: int = PART_FINE_GRAINED) -> "Partition":
        h, rq, gr = _vp(), _i32(), _i32()
        _ck(_lib.tp_partition_get(device, float(fraction), flags, ctypes.byref(h), ctypes.byref(rq),
                                  ctypes.byref(gr)), "tp_partition_get")
        return cls(h.value, device, rq.value, gr.value, fraction)

    @classmethod
    def split(cls, k: int, sms_each: int, device: int = 0, flags: int = PART_FINE_GRAINED) -> list["Partition"]:
        hs, gr = (_vp * k)(), (_i32 * k)()
        _ck(_lib.tp_partition_split(device, k, sms_each, flags, hs, gr), "tp_partition_split")
        total = device_sm_count(device)
        return [cls(hs[i], device, sms_each, gr[i], sms_each / total, owned=True) for i in range(k)]

    @classmethod
    def shared(cls, k: int, device: int = 0) -> list["Partition"]:
        """k unpartitioned whole-device handles, one stream each (f3: no SM isolation)."""
        hs = (_vp * k)()
        _ck(_lib.tp_partition_shared(device, k, hs), "tp_partition_shared")
        total = device_sm_count(device)
        return [cls(hs[i], device, total, total, 1.0, owned=True) for i in range(k)]

    def stream(self) -> int:
        s = _vp()
        _ck(_lib.tp_partition_info(self.handle, None, None, None, ctypes.byref(s)), "tp_partition_info")
        return s.value or 0

    def sync(self):
        _ck(_lib.tp_partition_sync(self.handle), "tp_partition_sync")

    def close(self):
        if self.owned and self.handle:
            _ck(_lib.tp_partition_close(self.handle), "tp_partition_close")
            self.handle = 0

    def probe_smids(self, ctas: int) -> np.ndarray:
        import torch
        buf = torch.full((ctas,), -1, dtype=torch.int32, device=f"cuda:{self.device}")
        torch.cuda.synchronize(self.device)   # the fill runs on torch's stream, the probe on the partition's
        _ck(_lib.tp_partition_probe(self.handle, ctas, buf.data_ptr()), "tp_partition_probe")
        return buf.cpu().numpy()

    def floor(self, ctas: int = 1, threads: int = 128, timing_cfg: "Timing | None" = None) -> dict:
        """Per-launch latency of an empty kernel under the timing protocol."""
        m = Measurement()
        _ck(_lib.tp_partition_floor(self.handle, int(ctas), int(threads),
                                    ctypes.byref(timing_cfg) if timing_cfg is not None else None, ctypes.byref(m)),
            "tp_partition_floor")
        return meas_to_dict(m)

    def copy_bw(self, nbytes: int = 1 << 30, reps: int = 5) -> float:
        import torch
        a = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{self.device}")
        b = torch.empty_like(a)
        g = _dbl()
        _ck(_lib.tp_partition_copy_bw(self.handle, a.data_ptr(), b.data_ptr(), nbytes, reps, ctypes.byref(g)),
            "tp_partition_copy_bw")
        return g.value


def _h(part):
    return part.handle if part is not None else None


class LayerBuffers:
    """Device operands of one layer: packed x / w (by libtp's pack kernels),
    bias, output y and a zeroed workspace big enough for every schedule."""

    def __init__(self, d: dict, x_nchw_f32, w_kcrs_f32, bias_f32=None, part: Partition | None = None,
                 device: int = 0, ws_bytes: int | None = None):
        import torch
        self.d = d
        self.cd = desc(d)
        dev = f"cuda:{device}"
        eb = 2 if d["dtype"] == BF16 else 4
        ob = 2 if d.get("out_dtype", d["dtype"]) == BF16 else 4
        P, Q = output_shape(d)
        self.P, self.Q = P, Q
        xf = torch.as_tensor(np.ascontiguousarray(x_nchw_f32, dtype=np.float32)).to(dev)
        wf = torch.as_tensor(np.ascontiguousarray(w_kcrs_f32, dtype=np.float32)).to(dev)
        self.x = torch.empty(xf.numel() * eb, dtype=torch.uint8, device=dev)
        self.w = torch.empty(wf.numel() * eb, dtype=torch.uint8, device=dev)
        bias = bias_f32 if bias_f32 is not None else np.zeros(d["k"], np.float32)
        self.b = torch.as_tensor(np.ascontiguousarray(bias, dtype=np.float32)).to(dev)
        self.y = torch.empty(d["n"] * d["k"] * P * Q * ob, dtype=torch.uint8, device=dev)
        self.ws_bytes = workspace_size(d) if ws_bytes is None else ws_bytes
        self.ws = torch.zeros(max(256, self.ws_bytes), dtype=torch.uint8, device=dev)
        torch.cuda.synchronize(dev)   # torch's stream -> libtp's stream ordering
        _ck(_lib.tp_pack_input(ctypes.byref(self.cd), _h(part), xf.data_ptr(), self.x.data_ptr()), "tp_pack_input")
        _ck(_lib.tp_pack_weights(ctypes.byref(self.cd), _h(part), wf.data_ptr(), self.w.data_ptr()),
            "tp_pack_weights")
        _ck(_lib.tp_partition_sync(_h(part)), "tp_partition_sync")
        del xf, wf

    def poison(self):
        """Fill y with NaN bit patterns (0xFF bytes) and wait, so a schedule
        that writes nothing cannot pass a check."""
        import torch
        self.y.fill_(0xFF)
        torch.cuda.synchronize(self.y.device)

    def ptrs(self):
        return (self.x.data_ptr(), self.w.data_ptr(), self.b.data_ptr(), self.y.data_ptr(), self.ws.data_ptr(),
                self.ws.numel())

    def output(self):
        """y as a float64 numpy array in logical NKPQ order (host copy)."""
        import torch
        d = self.d
        ob = d.get("out_dtype", d["dtype"])
        t = self.y.view(torch.bfloat16 if ob == BF16 else torch.float32).double().cpu().numpy()
        if d.get("in_layout", NHWC) == NHWC:
            return t.reshape(d["n"], self.P, self.Q, d["k"]).transpose(0, 3, 1, 2)
        return t.reshape(d["n"], d["k"], self.P, self.Q)

    def gather(self, idx, part: Partition | None = None) -> np.ndarray:
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        out = np.empty(idx.shape[0], dtype=np.float64)
        _ck(_lib.tp_gather_output(ctypes.byref(self.cd), _h(part), self.y.data_ptr(),
                                  idx.ctypes.data_as(_P(_i64)), idx.shape[0], out.ctypes.data_as(_P(_dbl))),
            "tp_gather_output")
        return out


def conv2d_run(buf: LayerBuffers, sched: dict, part: Partition | None = None, timing_cfg: Timing | None = None,
               measure: bool = False):
    x, w, b, y, ws, wsb = buf.ptrs()
    s = dict_to_sched(sched)
    if not measure and timing_cfg is None:
        _ck(_lib.tp_conv2d_run(ctypes.byref(buf.cd), ctypes.byref(s), _h(part), x, w, b, y, ws, wsb, None, None),
            "tp_conv2d_run")
        return None
    m = Measurement()
    _ck(_lib.tp_conv2d_run(ctypes.byref(buf.cd), ctypes.byref(s), _h(part), x, w, b, y, ws, wsb,
                           ctypes.byref(timing_cfg) if timing_cfg is not None else None, ctypes.byref(m)),
        "tp_conv2d_run")
    return meas_to_dict(m)


def conv2d_trace(buf: "LayerBuffers", sched: dict, part: Partition | None = None, launches: int = 1) -> np.ndarray:
    """In-kernel timeline of 1-4 back-to-back tensor-core launches, captured in
    one CUDA graph: (launches * ctas, 96) uint64 (see tp.h)."""
    x, w, b, y, ws, wsb = buf.ptrs()
    cap = int(sched.get("grid_x", 0) * sched.get("grid_y", 0) * sched.get("grid_z", 0)) or 65536
    cap *= max(1, min(4, launches))
    out = np.zeros((cap, 96), dtype=np.uint64)
    rows = _i32()
    _ck(_lib.tp_conv2d_trace(ctypes.byref(buf.cd), ctypes.byref(dict_to_sched(sched)), _h(part), x, w, b, y, ws,
                             wsb, out.ctypes.data_as(_P(_u64)), cap, ctypes.byref(rows)), "tp_conv2d_trace")
    return out[:rows.value]


def _check_arrays(check_idx, check_ref):
    if check_idx is None:
        return None, None, 0
    ci = np.ascontiguousarray(check_idx, dtype=np.int64)
    cr = np.ascontiguousarray(check_ref, dtype=np.float64)
    return ci, cr, ci.shape[0]


def tune(buf: LayerBuffers, part: Partition | None, trials: int, seed: int, check_idx=None, check_ref=None,
         tol: float = 0.0, timing_cfg: Timing | None = None):
    """Returns (best schedule dict, best measurement dict, list of record dicts)."""
    x, w, b, y, ws, wsb = buf.ptrs()
    n_space = space_size(buf.d)
    cap = max(1, min(trials, n_space))
    recs = (Measurement * cap)()
    nrec = _i32()
    best, best_m = Schedule(), Measurement()
    ci, cr, nc = _check_arrays(check_idx, check_ref)
    st = _lib.tp_tune(ctypes.byref(buf.cd), _h(part), int(trials), int(seed), x, w, b, y, ws, wsb,
                      ci.ctypes.data_as(_P(_i64)) if nc else None, cr.ctypes.data_as(_P(_dbl)) if nc else None, nc,
                      float(tol), ctypes.byref(timing_cfg) if timing_cfg is not None else None,
                      ctypes.byref(best), ctypes.byref(best_m), recs, cap, ctypes.byref(nrec))
    records = [meas_to_dict(recs[i]) for i in range(nrec.value)]
    _ck(st, "tp_tune")
    return sched_to_dict(best), meas_to_dict(best_m), records


def search_should_stop(us, early_stop: int) -> bool:
    """Early-stopping rule (tp_search_should_stop, reading C19): the last
    `early_stop` measured candidates did not lower the best latency (us < 0 =
    failed candidate)."""
    a = np.ascontiguousarray(us, dtype=np.float64)
    return bool(_lib.tp_search_should_stop(a.ctypes.data_as(_P(_dbl)), int(a.shape[0]), int(early_stop)))


def tune_guided(buf: "LayerBuffers", part: Partition | None, trials: int, batch: int = 16, explore: float = 0.25,
                seed: int = 42, tol: float = 0.0, timing_cfg: Timing | None = None, early_stop: int = 0):
    """Model-guided tuning (tp_tune_guided_es; early_stop = 0: tp_tune_guided):
    (best schedule, best measurement, records in measurement order)."""
    x, w, b, y, ws, wsb = buf.ptrs()
    cap = max(1, min(trials, space_size(buf.d)))
    recs = (Measurement * cap)()
    nrec = _i32()
    best, best_m = Schedule(), Measurement()
    st = _lib.tp_tune_guided_es(ctypes.byref(buf.cd), _h(part), int(trials), int(batch), float(explore),
                                int(seed) & (2**64 - 1), int(early_stop), x, w, b, y, ws, wsb, None, None, 0,
                                float(tol), ctypes.byref(timing_cfg) if timing_cfg is not None else None,
                                ctypes.byref(best), ctypes.byref(best_m), recs, cap, ctypes.byref(nrec))
    records = [meas_to_dict(recs[i]) for i in range(nrec.value)]
    _ck(st, "tp_tune_guided_es")
    return sched_to_dict(best), meas_to_dict(best_m), records


def tune_subset(buf: LayerBuffers, part: Partition | None, cand_idx, check_idx=None, check_ref=None,
                tol: float = 0.0, timing_cfg: Timing | None = None) -> list[dict]:
    x, w, b, y, ws, wsb = buf.ptrs()
    cand = np.ascontiguousarray(cand_idx, dtype=np.int64)
    cap = max(1, cand.shape[0])
    recs = (Measurement * cap)()
    nrec = _i32()
    ci, cr, nc = _check_arrays(check_idx, check_ref)
    _ck(_lib.tp_tune_subset(ctypes.byref(buf.cd), _h(part), cand.ctypes.data_as(_P(_i64)), cand.shape[0], x, w, b, y,
                            ws, wsb, ci.ctypes.data_as(_P(_i64)) if nc else None,
                            cr.ctypes.data_as(_P(_dbl)) if nc else None, nc, float(tol),
                            ctypes.byref(timing_cfg) if timing_cfg is not None else None, recs, cap,
                            ctypes.byref(nrec)), "tp_tune_subset")
    return [meas_to_dict(recs[i]) for i in range(nrec.value)]


def conv2d_run_at(buf: LayerBuffers, sched: dict, sm_fraction: float, timing_cfg: Timing | None = None) -> dict:
    """tp_conv2d_run_at: the run call with GPU% as a fraction."""
    x, w, b, y, ws, wsb = buf.ptrs()
    m = Measurement()
    _ck(_lib.tp_conv2d_run_at(ctypes.byref(buf.cd), ctypes.byref(dict_to_sched(sched)), float(sm_fraction), x, w, b,
                              y, ws, wsb, ctypes.byref(timing_cfg or timing()), ctypes.byref(m)), "tp_conv2d_run_at")
    return meas_to_dict(m)


def tune_at(buf: LayerBuffers, sm_fraction: float, trials: int, seed: int, check_idx=None, check_ref=None,
            tol: float = 0.0, timing_cfg: Timing | None = None):
    """tp_tune_at: (best schedule, best measurement, records) at a GPU% fraction."""
    x, w, b, y, ws, wsb = buf.ptrs()
    cap = max(1, min(trials, space_size(buf.d)))
    recs = (Measurement * cap)()
    nrec = _i32()
    best, best_m = Schedule(), Measurement()
    ci, cr, nc = _check_arrays(check_idx, check_ref)
    st = _lib.tp_tune_at(ctypes.byref(buf.cd), float(sm_fraction), int(trials), int(seed), x, w, b, y, ws, wsb,
                         ci.ctypes.data_as(_P(_i64)) if nc else None, cr.ctypes.data_as(_P(_dbl)) if nc else None, nc,
                         float(tol), ctypes.byref(timing_cfg) if timing_cfg is not None else None,
                         ctypes.byref(best), ctypes.byref(best_m), recs, cap, ctypes.byref(nrec))
    records = [meas_to_dict(recs[i]) for i in range(nrec.value)]
    _ck(st, "tp_tune_at")
    return sched_to_dict(best), meas_to_dict(best_m), records


def cross_eval_at(buf: LayerBuffers, tuned_sched: dict, q: float, timing_cfg: Timing | None = None) -> dict:
    """tp_cross_eval_at: schedule tuned at p (frozen geometry) run at fraction q."""
    x, w, b, y, ws, wsb = buf.ptrs()
    m = Measurement()
    _ck(_lib.tp_cross_eval_at(ctypes.byref(buf.cd), ctypes.byref(dict_to_sched(tuned_sched)), float(q), x, w, b, y,
                              ws, wsb, ctypes.byref(timing_cfg) if timing_cfg is not None else None, ctypes.byref(m)),
        "tp_cross_eval_at")
    return meas_to_dict(m)


def cross_eval(buf: LayerBuffers, tuned_sched: dict, part_q: Partition | None,
               timing_cfg: Timing | None = None) -> dict:
    x, w, b, y, ws, wsb = buf.ptrs()
    m = Measurement()
    _ck(_lib.tp_cross_eval(ctypes.byref(buf.cd), ctypes.byref(dict_to_sched(tuned_sched)), _h(part_q), x, w, b, y,
                           ws, wsb, ctypes.byref(timing_cfg) if timing_cfg is not None else None, ctypes.byref(m)),
        "tp_cross_eval")
    return meas_to_dict(m)


def chain_run(bufs: list, scheds: list[dict], part: Partition | None = None, reps: int = 1,
              timing_cfg: Timing | None = None, measure: bool = False):
    """tp_chain_run: the layers of `bufs` in order (layer i+1 may read layer
    i's y as its x), `reps` times, as one graph.  measure=True -> the timing
    protocol over whole sequences; returns the measurement dict (median_us per
    sequence) or None for a single asynchronous replay."""
    n = len(bufs)
    descs = (ConvDesc * n)(*[b.cd for b in bufs])
    ss = (Schedule * n)(*[dict_to_sched(s) for s in scheds])
    ptr = lambda vals: (_vp * n)(*vals)   # noqa: E731
    xs = ptr([b.x.data_ptr() for b in bufs])
    ws_ = ptr([b.w.data_ptr() for b in bufs])
    bs = ptr([b.b.data_ptr() for b in bufs])
    ys = ptr([b.y.data_ptr() for b in bufs])
    wk = ptr([b.ws.data_ptr() for b in bufs])
    wb = (_sz * n)(*[b.ws.numel() for b in bufs])
    if not measure and timing_cfg is None:
        _ck(_lib.tp_chain_run(n, descs, ss, _h(part), xs, ws_, bs, ys, wk, wb, int(reps), None, None), "tp_chain_run")
        return None
    m = Measurement()
    _ck(_lib.tp_chain_run(n, descs, ss, _h(part), xs, ws_, bs, ys, wk, wb, int(reps),
                          ctypes.byref(timing_cfg) if timing_cfg is not None else None, ctypes.byref(m)),
        "tp_chain_run")
    return meas_to_dict(m)


def exported_symbols() -> list[str]:
    """Symbols include/tp.h declares (checked by tests against the .so)."""
    import re
    hdr = open(os.path.join(os.path.dirname(_HERE), "include", "tp.h")).read()
    return sorted(set(re.findall(r"\b(tp_[a-z0-9_]+)\s*\(", hdr)))
