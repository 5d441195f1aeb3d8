"""Seeded synthetic workloads for the five BASELINE configs.

Images follow the reference fixtures (synth.py:14-23): i.i.d. uniform u8 in
[0, 255] or f32 in [0, 1), one seed per image so every rank, the oracle and
the CPU baseline can regenerate any image locally. Warp parameters follow the
builder contract: affine theta~U(-30,30) deg, s~U(0.8,1.2),
t~U(-50,50)^2 about the image centre; perspective H = I + N(0, 1e-3) on the
8 free entries.
"""
from __future__ import annotations

import numpy as np
import torch

# per-config image seed bases
SEED_GRAY, SEED_RESIZE, SEED_AFFINE, SEED_PERSP, SEED_FUSED = 11, 20000, 30000, 40000, 50000
SEED_AFFINE_PARAMS, SEED_PERSP_PARAMS = 31000, 41000

MEAN = (0.485, 0.456, 0.406)
STD = (0.229, 0.224, 0.225)


def seeded_u8_image(width: int, height: int, channels: int, seed: int = 0) -> np.ndarray:
    return np.random.default_rng(seed).integers(0, 256, size=(height, width, channels), dtype=np.uint8)


def seeded_f32_image(width: int, height: int, channels: int, seed: int = 0) -> np.ndarray:
    return np.random.default_rng(seed).random(size=(height, width, channels), dtype=np.float32)


def device_u8_batch(n, height, width, channels, seed, device) -> torch.Tensor:
    """Uniform u8 batch generated on the device (bench inputs; same
    distribution as seeded_u8_image, different stream of numbers)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return torch.randint(0, 256, (n, height, width, channels), dtype=torch.uint8, device=device, generator=g)


def device_f32_batch(n, height, width, channels, seed, device) -> torch.Tensor:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return torch.rand((n, height, width, channels), dtype=torch.float32, device=device, generator=g)


def affine_forward(seed: int, width: int, height: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    theta = np.deg2rad(rng.uniform(-30.0, 30.0))
    s = rng.uniform(0.8, 1.2)
    tx, ty = rng.uniform(-50.0, 50.0), rng.uniform(-50.0, 50.0)
    a = s * np.array([[np.cos(theta), -np.sin(theta)], [np.sin(theta), np.cos(theta)]])
    c = np.array([(width - 1) / 2.0, (height - 1) / 2.0])
    b = c + np.array([tx, ty]) - a @ c
    return np.hstack([a, b[:, None]])


def perspective_forward(seed: int) -> np.ndarray:
    eps = np.random.default_rng(seed).normal(0.0, 1e-3, 8)
    hm = np.eye(3).reshape(-1)
    hm[:8] += eps
    hm[8] = 1.0
    return hm.reshape(3, 3)
