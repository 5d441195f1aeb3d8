"""Synthetic inputs for the bench, the tests and the tools -- not part of the
product package (which only needs the seeded uniform images of the BASELINE
configs, paper_2505_12425_b200/synth.py).

`seeded_smooth_u8_image` restates the reference's codec fixture
(pkg/src/fovea/synth.py:26-45) so the decode -> preprocess row and the JPEG
tests encode the same kind of photographic content; it must match the
reference byte for byte, so it follows its arithmetic exactly.
"""
from __future__ import annotations

import numpy as np


def seeded_smooth_u8_image(width: int, height: int, channels: int, seed: int = 0) -> np.ndarray:
    """Photographic-ish content for codec workloads (the reference's
    synth.py:26-45): per channel 128 + four random 2-D sinusoids (freq
    U(0.5, 4) cycles per frame, amplitude U(20, 60)), plus N(0, 2) noise,
    rounded and clipped."""
    rng = np.random.default_rng(seed)
    y = np.linspace(0, 1, height, endpoint=False)[:, None]
    x = np.linspace(0, 1, width, endpoint=False)[None, :]
    out = np.zeros((height, width, channels), dtype=np.float64)
    for c in range(channels):
        acc = np.zeros((height, width))
        for _ in range(4):
            fy, fx = rng.uniform(0.5, 4.0, size=2)
            phase = rng.uniform(0, 2 * np.pi)
            amp = rng.uniform(20, 60)
            acc += amp * np.sin(2 * np.pi * (fy * y + fx * x) + phase)
        out[:, :, c] = 128.0 + acc
    out += rng.normal(0.0, 2.0, size=out.shape)
    return np.clip(np.round(out), 0, 255).astype(np.uint8)
