"""Seeded synthetic inputs standing in for BASELINE.json's five configs.

The reference ships no dataset and BASELINE.json names no public benchmark;
these generators follow SURVEY.md Appendix A exactly (numpy PCG64
`default_rng`, draws in the listed order) so the T/N/M values quoted there
reproduce.
"""

from __future__ import annotations

import numpy as np


def synth(h, w, n_rect, lo, hi, noise_sigma, seed, field_amp=0.0) -> np.ndarray:
    """Rectangles over a linear x-gradient, optional sinusoidal field, noise.

    Returns float64 in [lo, hi].
    """
    rng = np.random.default_rng(seed)
    img = np.tile(np.linspace(lo, hi, w), (h, 1))
    for _ in range(n_rect):
        rh = rng.integers(h // 16, h // 4 + 1)
        rw = rng.integers(w // 16, w // 4 + 1)
        r0 = rng.integers(0, h - rh + 1)
        c0 = rng.integers(0, w - rw + 1)
        img[r0:r0 + rh, c0:c0 + rw] = rng.uniform(lo, hi)
    if field_amp:
        fx = rng.uniform(1, 4)
        fy = rng.uniform(1, 4)
        ph = rng.uniform(0, 2 * np.pi)
        s = max(h, w)
        y = np.arange(h)[:, None] / s
        x = np.arange(w)[None, :] / s
        img += field_amp * np.sin(2 * np.pi * (fx * x + fy * y) + ph)
    img += rng.normal(0, noise_sigma, (h, w))
    return np.clip(img, lo, hi)


# (name, generator call, dtype step, filter parameters)
CONFIGS = {
    1: dict(name="cfg1_512_f64", sigma_s=3.0, sigma_r=30.0, epsilon=0.01),
    2: dict(name="cfg2_1024_f32", sigma_s=5.0, sigma_r=10.0, epsilon=0.01),
    3: dict(name="cfg3_2048_u16_hdr", sigma_s=8.0, sigma_r=800.0, epsilon=0.01),
    4: dict(name="cfg4_64x4096_f32", sigma_s=6.0, sigma_r=20.0, epsilon=0.01),
    5: dict(name="cfg5_3x16384_f32", sigma_s=12.0, sigma_r=15.0, epsilon=0.01),
}


def config_image(cfg: int, index: int = 0, size: int | None = None) -> np.ndarray:
    """The seeded input of config `cfg` (image/channel `index`).

    `size` overrides the square side (parity tests use crops of the same
    distribution); the seed and draw order are unchanged.
    """
    if cfg == 1:
        n = size or 512
        return synth(n, n, 20, 0, 255, 10, seed=1)
    if cfg == 2:
        n = size or 1024
        return synth(n, n, 40, 0, 255, 5, seed=2).astype(np.float32)
    if cfg == 3:
        n = size or 2048
        img = synth(n, n, 60, 0, 65535, 300, seed=3, field_amp=2000)
        return np.round(img).astype(np.uint16).astype(np.float32)
    if cfg == 4:
        n = size or 4096
        return synth(n, n, 20, 0, 255, 10, seed=4000 + index).astype(np.float32)
    if cfg == 5:
        n = size or 16384
        return synth(n, n, 20, 0, 255, 8, seed=5000 + index).astype(np.float32)
    raise ValueError(f"unknown config {cfg}")
