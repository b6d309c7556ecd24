"""Layer catalogs of the synthetic workloads (BASELINE.json configs).

Pure data: each entry is (name, multiplicity, N, C, H, W, K, R, S, stride,
pad, groups).  The paper lists no shapes; these are the standard
architectures it names (ResNet, VGG-19, MobileNet),
with ResNet-50 v1.5 and MobileNetV2 width 1.0 as BASELINE.json's configs ask.
"""
from __future__ import annotations

BF16, FP32 = 0, 1

# config 1: single fp32 conv, 100% SMs.
CFG1 = [("cfg1.conv3x3", 1, 1, 64, 56, 56, 64, 3, 3, 1, 1, 1)]

# config 2/3: ResNet-50 v1.5 batch 1, the 23 unique conv shapes of 53 layers.
RESNET50 = [
    ("r50.conv1", 1, 1, 3, 224, 224, 64, 7, 7, 2, 3, 1),
    ("r50.l1.b0.c1", 1, 1, 64, 56, 56, 64, 1, 1, 1, 0, 1),
    ("r50.l1.b0.c2", 3, 1, 64, 56, 56, 64, 3, 3, 1, 1, 1),
    ("r50.l1.b0.c3", 4, 1, 64, 56, 56, 256, 1, 1, 1, 0, 1),
    ("r50.l1.b1.c1", 2, 1, 256, 56, 56, 64, 1, 1, 1, 0, 1),
    ("r50.l2.b0.c1", 1, 1, 256, 56, 56, 128, 1, 1, 1, 0, 1),
    ("r50.l2.b0.c2", 1, 1, 128, 56, 56, 128, 3, 3, 2, 1, 1),
    ("r50.l2.b0.c3", 4, 1, 128, 28, 28, 512, 1, 1, 1, 0, 1),
    ("r50.l2.b0.ds", 1, 1, 256, 56, 56, 512, 1, 1, 2, 0, 1),
    ("r50.l2.b1.c1", 3, 1, 512, 28, 28, 128, 1, 1, 1, 0, 1),
    ("r50.l2.b1.c2", 3, 1, 128, 28, 28, 128, 3, 3, 1, 1, 1),
    ("r50.l3.b0.c1", 1, 1, 512, 28, 28, 256, 1, 1, 1, 0, 1),
    ("r50.l3.b0.c2", 1, 1, 256, 28, 28, 256, 3, 3, 2, 1, 1),
    ("r50.l3.b0.c3", 6, 1, 256, 14, 14, 1024, 1, 1, 1, 0, 1),
    ("r50.l3.b0.ds", 1, 1, 512, 28, 28, 1024, 1, 1, 2, 0, 1),
    ("r50.l3.b1.c1", 5, 1, 1024, 14, 14, 256, 1, 1, 1, 0, 1),
    ("r50.l3.b1.c2", 5, 1, 256, 14, 14, 256, 3, 3, 1, 1, 1),
    ("r50.l4.b0.c1", 1, 1, 1024, 14, 14, 512, 1, 1, 1, 0, 1),
    ("r50.l4.b0.c2", 1, 1, 512, 14, 14, 512, 3, 3, 2, 1, 1),
    ("r50.l4.b0.c3", 3, 1, 512, 7, 7, 2048, 1, 1, 1, 0, 1),
    ("r50.l4.b0.ds", 1, 1, 1024, 14, 14, 2048, 1, 1, 2, 0, 1),
    ("r50.l4.b1.c1", 2, 1, 2048, 7, 7, 512, 1, 1, 1, 0, 1),
    ("r50.l4.b1.c2", 2, 1, 512, 7, 7, 512, 3, 3, 1, 1, 1),
]

# config 4: VGG-19 batch 16, 9 unique of 16 conv layers.
VGG19_B16 = [
    ("vgg.64.224.0", 1, 16, 3, 224, 224, 64, 3, 3, 1, 1, 1),
    ("vgg.64.224.1", 1, 16, 64, 224, 224, 64, 3, 3, 1, 1, 1),
    ("vgg.128.112.0", 1, 16, 64, 112, 112, 128, 3, 3, 1, 1, 1),
    ("vgg.128.112.1", 1, 16, 128, 112, 112, 128, 3, 3, 1, 1, 1),
    ("vgg.256.56.0", 1, 16, 128, 56, 56, 256, 3, 3, 1, 1, 1),
    ("vgg.256.56.1", 3, 16, 256, 56, 56, 256, 3, 3, 1, 1, 1),
    ("vgg.512.28.0", 1, 16, 256, 28, 28, 512, 3, 3, 1, 1, 1),
    ("vgg.512.28.1", 3, 16, 512, 28, 28, 512, 3, 3, 1, 1, 1),
    ("vgg.512.14.0", 4, 16, 512, 14, 14, 512, 3, 3, 1, 1, 1),
]

# config 5: MobileNetV2 (width 1.0) batch 1, 30 unique of 52 conv layers.
MOBILENETV2 = [
    ("mb2.conv0", 1, 1, 3, 224, 224, 32, 3, 3, 2, 1, 1),
    ("mb2.dw.32.112.s1", 1, 1, 32, 112, 112, 32, 3, 3, 1, 1, 32),
    ("mb2.pw_proj.32->16.112", 1, 1, 32, 112, 112, 16, 1, 1, 1, 0, 1),
    ("mb2.pw_exp.96.112", 1, 1, 16, 112, 112, 96, 1, 1, 1, 0, 1),
    ("mb2.dw.96.112.s2", 1, 1, 96, 112, 112, 96, 3, 3, 2, 1, 96),
    ("mb2.pw_proj.96->24.56", 1, 1, 96, 56, 56, 24, 1, 1, 1, 0, 1),
    ("mb2.pw_exp.144.56", 2, 1, 24, 56, 56, 144, 1, 1, 1, 0, 1),
    ("mb2.dw.144.56.s1", 1, 1, 144, 56, 56, 144, 3, 3, 1, 1, 144),
    ("mb2.pw_proj.144->24.56", 1, 1, 144, 56, 56, 24, 1, 1, 1, 0, 1),
    ("mb2.dw.144.56.s2", 1, 1, 144, 56, 56, 144, 3, 3, 2, 1, 144),
    ("mb2.pw_proj.144->32.28", 1, 1, 144, 28, 28, 32, 1, 1, 1, 0, 1),
    ("mb2.pw_exp.192.28", 3, 1, 32, 28, 28, 192, 1, 1, 1, 0, 1),
    ("mb2.dw.192.28.s1", 2, 1, 192, 28, 28, 192, 3, 3, 1, 1, 192),
    ("mb2.pw_proj.192->32.28", 2, 1, 192, 28, 28, 32, 1, 1, 1, 0, 1),
    ("mb2.dw.192.28.s2", 1, 1, 192, 28, 28, 192, 3, 3, 2, 1, 192),
    ("mb2.pw_proj.192->64.14", 1, 1, 192, 14, 14, 64, 1, 1, 1, 0, 1),
    ("mb2.pw_exp.384.14", 4, 1, 64, 14, 14, 384, 1, 1, 1, 0, 1),
    ("mb2.dw.384.14.s1", 4, 1, 384, 14, 14, 384, 3, 3, 1, 1, 384),
    ("mb2.pw_proj.384->64.14", 3, 1, 384, 14, 14, 64, 1, 1, 1, 0, 1),
    ("mb2.pw_proj.384->96.14", 1, 1, 384, 14, 14, 96, 1, 1, 1, 0, 1),
    ("mb2.pw_exp.576.14", 3, 1, 96, 14, 14, 576, 1, 1, 1, 0, 1),
    ("mb2.dw.576.14.s1", 2, 1, 576, 14, 14, 576, 3, 3, 1, 1, 576),
    ("mb2.pw_proj.576->96.14", 2, 1, 576, 14, 14, 96, 1, 1, 1, 0, 1),
    ("mb2.dw.576.14.s2", 1, 1, 576, 14, 14, 576, 3, 3, 2, 1, 576),
    ("mb2.pw_proj.576->160.7", 1, 1, 576, 7, 7, 160, 1, 1, 1, 0, 1),
    ("mb2.pw_exp.960.7", 3, 1, 160, 7, 7, 960, 1, 1, 1, 0, 1),
    ("mb2.dw.960.7.s1", 3, 1, 960, 7, 7, 960, 3, 3, 1, 1, 960),
    ("mb2.pw_proj.960->160.7", 2, 1, 960, 7, 7, 160, 1, 1, 1, 0, 1),
    ("mb2.pw_proj.960->320.7", 1, 1, 960, 7, 7, 320, 1, 1, 1, 0, 1),
    ("mb2.conv_last", 1, 1, 320, 7, 7, 1280, 1, 1, 1, 0, 1),
]

CATALOGS = {"cfg1": (CFG1, FP32), "resnet50": (RESNET50, BF16), "vgg19_b16": (VGG19_B16, BF16),
            "mobilenetv2": (MOBILENETV2, BF16)}


def layer_dict(entry, dtype: int, relu: bool = True, bias: bool = True, layout: int = 0) -> dict:
    """Descriptor dict (same field names as tp_conv_desc) for one catalog entry."""
    name, mult, n, c, h, w, k, r, s, st, pad, g = entry
    return {"name": name, "mult": mult, "n": n, "c": c, "h": h, "w": w, "k": k, "r": r, "s": s,
            "stride_h": st, "stride_w": st, "pad_h": pad, "pad_w": pad, "dil_h": 1, "dil_w": 1,
            "groups": g, "in_layout": layout, "dtype": dtype, "out_dtype": dtype,
            "epilogue": (1 if bias else 0) | (2 if relu else 0)}


def catalog(name: str, relu: bool = True, bias: bool = True) -> list[dict]:
    entries, dtype = CATALOGS[name]
    return [layer_dict(e, dtype, relu, bias) for e in entries]


def resnet50_sequence() -> list[str]:
    """The 53 conv layers of ResNet-50 v1.5 in execution order, as unique-layer
    names of RESNET50 (each bottleneck block runs c1, c2, c3, then the
    downsample projection of its first block; torchvision's forward order)."""
    seq = ["r50.conv1"]
    for stage, blocks in (("l1", 3), ("l2", 4), ("l3", 6), ("l4", 3)):
        for b in range(blocks):
            if b == 0:
                seq += [f"r50.{stage}.b0.c1", f"r50.{stage}.b0.c2", f"r50.{stage}.b0.c3"]
                seq.append("r50.l1.b0.c3" if stage == "l1" else f"r50.{stage}.b0.ds")
            else:
                c3 = "r50.l1.b0.c3" if stage == "l1" else f"r50.{stage}.b0.c3"
                seq += [f"r50.{stage}.b1.c1", "r50.l1.b0.c2" if stage == "l1" else f"r50.{stage}.b1.c2", c3]
    return seq
