"""Pins of the evaluation metrics (evaluation/quality.py) used for the
paper's quality experiments: closed forms of SSIM and
PSNR on images whose statistics are known exactly."""
import numpy as np

from evaluation import psnr, ssim


def test_ssim_identity_and_symmetry():
    rng = np.random.default_rng(0)
    a = rng.random((40, 50, 3))
    b = np.clip(a + 0.05 * rng.standard_normal(a.shape), 0, 1)
    assert abs(ssim(a, a) - 1.0) < 1e-12
    assert abs(ssim(a, b) - ssim(b, a)) < 1e-12
    assert ssim(a, b) < 1.0


def test_ssim_constant_images_closed_form():
    """Two constant images c1, c2: zero variances, so SSIM = (2 c1 c2 + C1) / (c1^2 + c2^2 + C1)."""
    for c1, c2 in ((0.2, 0.7), (0.5, 0.5), (0.0, 1.0)):
        a = np.full((30, 30, 3), c1)
        b = np.full((30, 30, 3), c2)
        C1 = 0.01 ** 2
        assert abs(ssim(a, b) - (2 * c1 * c2 + C1) / (c1 * c1 + c2 * c2 + C1)) < 1e-12


def test_psnr_closed_form():
    a = np.zeros((10, 10, 3))
    b = np.full((10, 10, 3), 0.1)          # MSE 0.01 -> 20 dB
    assert abs(psnr(a, b) - 20.0) < 1e-9
    assert psnr(a, a) == float("inf")
