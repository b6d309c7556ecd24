"""Host-side checks of numeric identities the kernels rely on (no GPU).

The stem kind's bias-in-MMA form (TcArgs::bias_mma) splits each fp32
bias b into three bf16 parts b1 = rne(b), b2 = rne(b - b1), b3 = rne(b - b1 - b2)
(residuals formed in fp32) and relies on b1 + b2 + b3 == b exactly, so that the
accumulator holds conv + b up to the MMA's summation order only."""
import numpy as np
import torch


def _bf16(a: np.ndarray) -> np.ndarray:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).bfloat16().float().numpy()


def _split3(b: np.ndarray):
    b = b.astype(np.float32)
    b1 = _bf16(b)
    r1 = (b - b1).astype(np.float32)
    b2 = _bf16(r1)
    b3 = _bf16((r1 - b2).astype(np.float32))
    return b1, b2, b3


def test_three_bf16_parts_sum_exactly_to_the_fp32_bias():
    rng = np.random.default_rng(7)
    vals = np.concatenate([
        rng.standard_normal(200_000).astype(np.float32),
        (rng.standard_normal(50_000) * 1e-3).astype(np.float32),
        (rng.standard_normal(50_000) * 1e3).astype(np.float32),
        rng.integers(-512, 512, 10_000).astype(np.float32),          # the integer-data tests' biases
        np.array([0.0, -0.0, 1.0, -1.0, 3.0e-5, 65504.0, 1.0 + 2.0 ** -23], dtype=np.float32),
    ])
    b1, b2, b3 = _split3(vals)
    total = b1.astype(np.float64) + b2.astype(np.float64) + b3.astype(np.float64)
    assert np.array_equal(total, vals.astype(np.float64))
    # each part really is a bf16 value
    for part in (b1, b2, b3):
        assert np.array_equal(_bf16(part), part)


def test_integer_biases_need_one_part():
    v = np.arange(-256, 257, dtype=np.float32)
    b1, b2, b3 = _split3(v)
    assert np.array_equal(b1, v) and not b2.any() and not b3.any()
