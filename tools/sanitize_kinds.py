"""One tiny launch of every libtp kernel kind, for compute-sanitizer
(tests/test_gpu_r2.py::test_compute_sanitizer_every_kind).  Whole device, no
partition; prints "sanitize_kinds ok" at the end."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2008_03602_b200 import datagen, tp  # noqa: E402


def mk(n, c, h, w, k, r, s, st=1, pad=0, g=1, dtype=tp.BF16, epi=3):
    return dict(n=n, c=c, h=h, w=w, k=k, r=r, s=s, stride_h=st, stride_w=st, pad_h=pad, pad_w=pad, dil_h=1, dil_w=1,
                groups=g, in_layout=tp.NHWC, dtype=dtype, out_dtype=dtype, epilogue=epi)


def pick(d, kind, **want):
    for i in range(tp.space_size(d)):
        s = tp.space_get(d, i)
        if s["kind"] == kind and all(s[k] == v for k, v in want.items()):
            return s
    raise SystemExit(f"no schedule of kind {kind} with {want} for {d}")


CASES = [
    (mk(1, 64, 10, 9, 64, 3, 3, 1, 1), tp.KIND_IGEMM_TC, dict(split_k=1, bm=128, bn=64)),
    (mk(1, 64, 10, 9, 64, 3, 3, 1, 1), tp.KIND_IGEMM_TC, dict(split_k=4, bm=128, bn=64)),
    (mk(1, 64, 8, 8, 64, 1, 1, 1, 0), tp.KIND_IGEMM_TC, dict(split_k=1, bm=64)),
    (mk(1, 3, 23, 21, 64, 7, 7, 2, 3), tp.KIND_IGEMM_TC_GATHER, dict(split_k=1)),
    (mk(1, 3, 23, 21, 64, 7, 7, 2, 3), tp.KIND_IGEMM_TC_GATHER, dict(split_k=2)),
    (mk(1, 64, 6, 60, 40, 3, 3, 1, 1), tp.KIND_IGEMM_TC_ROW, dict(tiles_per_cta=2)),
    (mk(1, 64, 128, 128, 128, 3, 3, 1, 1), tp.KIND_IGEMM_TC_MT, dict(tiles_per_cta=2, bm=128, bn=128)),
    (mk(1, 3, 10, 72, 64, 3, 3, 1, 1), tp.KIND_IGEMM_TC_STEM, dict(tiles_per_cta=2)),
    (mk(1, 36, 9, 9, 40, 3, 3, 1, 1, dtype=tp.FP32), tp.KIND_IGEMM_TF32X3, dict(split_k=1)),
    (mk(1, 36, 9, 9, 40, 3, 3, 1, 1, dtype=tp.FP32), tp.KIND_IGEMM_TF32X3, dict(split_k=2)),
    (mk(1, 8, 9, 10, 12, 3, 3, 1, 1, dtype=tp.FP32), tp.KIND_DIRECT, dict(smem_stage=1)),
    (mk(1, 16, 9, 9, 16, 3, 3, 2, 1, g=16), tp.KIND_DIRECT, dict(smem_stage=0)),
]


def run(cases):
    for d, kind, want in cases:
        x, w, b = datagen.make_inputs(d, 3, integer=True)
        buf = tp.LayerBuffers(d, x, w, b)
        s = pick(d, kind, **want)
        tp.conv2d_run(buf, s)
        torch.cuda.synchronize()
        buf.gather([0, 1, 2])
        print("kind", kind, want, "ok", flush=True)


def main():
    tp.init(0)
    run(CASES)
    # split-K through the global workspace (the fallback when the cluster cannot co-schedule)
    os.environ["TP_NO_CLUSTER"] = "1"
    run([c for c in CASES if c[2].get("split_k", 1) > 1])
    print("sanitize_kinds ok", flush=True)


if __name__ == "__main__":
    main()
