"""Evaluation tooling (not the hot path): image-quality metrics of the paper's
quality experiments (SSIM and PSNR against ground-truth
DVR).  Used by tests/ and bench.py; the product library never imports it."""
from .quality import psnr, ssim, to_rgb

__all__ = ["psnr", "ssim", "to_rgb"]
