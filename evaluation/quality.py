"""SSIM (Wang, Bovik, Sheikh, Simoncelli 2004) and PSNR of rendered images,
the two metrics the paper reports against ground-truth DVR (PAPER.md:213,
:278, :304, :330, :356).  Images are premultiplied RGBA composited over a
black background (the RGB channels as they are), values in [0, 1].

SSIM: 11x11 Gaussian window (sigma 1.5), K1 = 0.01, K2 = 0.03, data range 1,
computed per RGB channel and averaged (mean SSIM map); PSNR over all RGB
values with peak 1."""
from __future__ import annotations

import numpy as np
from scipy.ndimage import gaussian_filter


def to_rgb(rgba, w, h):
    """[h*w, 4] premultiplied RGBA (numpy or torch) -> [h, w, 3] float64 over black."""
    a = rgba.detach().cpu().numpy() if hasattr(rgba, "detach") else np.asarray(rgba)
    return np.clip(a.reshape(h, w, 4)[..., :3].astype(np.float64), 0.0, 1.0)


def psnr(a, b, peak=1.0):
    mse = float(np.mean((np.asarray(a, np.float64) - np.asarray(b, np.float64)) ** 2))
    return float("inf") if mse == 0 else 10.0 * np.log10(peak * peak / mse)


def ssim(a, b, data_range=1.0, sigma=1.5):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.ndim == 2:
        a, b = a[..., None], b[..., None]
    c1, c2 = (0.01 * data_range) ** 2, (0.03 * data_range) ** 2
    flt = lambda x: gaussian_filter(x, sigma=sigma, truncate=3.5)  # 11x11 window (radius 5)
    vals = []
    for ch in range(a.shape[-1]):
        x, y = a[..., ch], b[..., ch]
        mx, my = flt(x), flt(y)
        sxx = flt(x * x) - mx * mx
        syy = flt(y * y) - my * my
        sxy = flt(x * y) - mx * my
        m = ((2 * mx * my + c1) * (2 * sxy + c2)) / ((mx * mx + my * my + c1) * (sxx + syy + c2))
        vals.append(m.mean())
    return float(np.mean(vals))
