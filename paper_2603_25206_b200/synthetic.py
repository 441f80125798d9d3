"""Seeded synthetic stand-ins for the paper's datasets (BASELINE.json configs).

The paper's fields (Ocean, Hurricane, Miranda, NYX, JHTDB)
are not available; these generators reproduce the configs' shapes and value
distributions.  They are input generators, not part of the hot path:
configs 1-4 are generated on the host with numpy/scipy (float64 -> float32,
the same bytes feed the GPU and the CPU oracle); config 5 (2048^3, 32 GiB)
is generated on the GPU slab by slab (``gen_config5_slab``) from a
counter-based RNG so any z-range of any rank is reproducible.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

CONFIGS = {
    1: dict(dims=(1800, 3600), bound=("abs_range", 1e-4), kinds=(0, 1, 2, 3)),
    2: dict(dims=(100, 500, 500), bound=("rel", 1e-3), kinds=(1, 3), region=16),
    3: dict(dims=(256, 384, 384), bound=("rel", 1e-3), kinds=(1, 3), components=3),
    4: dict(dims=(512, 512, 512), bound=("rel", 1e-4), kinds=(0, 1, 2, 3), region=8),
    5: dict(dims=(2048, 2048, 2048), bound=("rel", 1e-3), kinds=(1, 3)),
}


def _modes_2d(rng, nmodes, kmax):
    mag = rng.integers(1, kmax + 1, size=(nmodes, 2))
    sign = rng.choice([-1, 1], size=(nmodes, 2))
    k = mag * sign
    amp = 1.0 / np.sqrt((k.astype(np.float64) ** 2).sum(axis=1))
    phase = rng.uniform(0.0, 2.0 * np.pi, size=nmodes)
    return k, amp, phase


def config1_field(seed: int = 1, dims=(1800, 3600)) -> np.ndarray:
    """32 random 2-D sinusoid modes (|k| in 1..16 cycles/domain, A = 1/|k|, random phase) + N(0, 1e-3^2)."""
    rng = np.random.default_rng(seed)
    n1, n2 = dims
    k, amp, phase = _modes_2d(rng, 32, 16)
    i = np.arange(n1) / n1
    j = np.arange(n2) / n2
    out = np.zeros(dims)
    for (kx, ky), a, ph in zip(k, amp, phase):
        ex = np.exp(2j * np.pi * kx * i)
        ey = np.exp(2j * np.pi * ky * j)
        out += a * np.imag(np.exp(1j * ph) * np.multiply.outer(ex, ey))
    out += rng.normal(0.0, 1e-3, size=dims)
    return out.astype(np.float32)


def config2_field(seed: int = 2, dims=(100, 500, 500)) -> np.ndarray:
    """White noise, isotropic Gaussian filter (sigma 4, reflect, truncate 4), rescaled to [-50, 50]."""
    from scipy.ndimage import gaussian_filter

    rng = np.random.default_rng(seed)
    g = gaussian_filter(rng.standard_normal(dims), sigma=4.0, mode="reflect", truncate=4.0)
    lo, hi = g.min(), g.max()
    return (-50.0 + 100.0 * (g - lo) / (hi - lo)).astype(np.float32)


def _grf(rng, dims, amp_exponent):
    """Gaussian random field: white noise -> rFFT * |k|^amp_exponent (DC = 0) -> irFFT, zero mean, unit std."""
    w = rng.standard_normal(dims)
    f = np.fft.rfftn(w)
    del w
    ks = [np.fft.fftfreq(n) * n for n in dims[:-1]] + [np.fft.rfftfreq(dims[-1]) * dims[-1]]
    k2 = np.zeros(f.shape)
    for ax, kk in enumerate(ks):
        shape = [1] * len(dims)
        shape[ax] = len(kk)
        k2 = k2 + (kk.reshape(shape) ** 2)
    k2.flat[0] = 1.0
    f *= k2 ** (amp_exponent / 2.0)
    f.flat[0] = 0.0
    del k2
    g = np.fft.irfftn(f, s=dims, axes=tuple(range(len(dims))))
    g -= g.mean()
    g /= g.std()
    return g


def config3_fields(seeds=(30, 31, 32), dims=(256, 384, 384)):
    """Three independent GRFs with power spectrum k^-3 (amplitude |k|^-1.5), zero mean, unit std."""
    return [_grf(np.random.default_rng(s), dims, -1.5).astype(np.float32) for s in seeds]


def config4_field(seed: int = 4, dims=(512, 512, 512)) -> np.ndarray:
    """Log-normal: exp of a k^-2 GRF scaled so max - min = ln(1e6) (about six decades)."""
    g = _grf(np.random.default_rng(seed), dims, -1.0)
    g *= math.log(1e6) / (g.max() - g.min())
    g -= 0.5 * (g.max() + g.min())
    return np.exp(g).astype(np.float32)


# ---------------------------------------------------------------------------
# config 5 on the GPU


def config5_modes(seed: int = 5, nmodes: int = 64):
    """64 random 3-D modes: integer k components in +-[1, 16], A = 1/|k|, random phase."""
    rng = np.random.default_rng(seed)
    mag = rng.integers(1, 17, size=(nmodes, 3))
    sign = rng.choice([-1, 1], size=(nmodes, 3))
    k = (mag * sign).astype(np.float64)
    amp = 1.0 / np.sqrt((k ** 2).sum(axis=1))
    phase = rng.uniform(0.0, 2.0 * np.pi, size=nmodes)
    params = np.concatenate([k, amp[:, None], phase[:, None]], axis=1)   # [kz, ky, kx, A, phi]
    return np.ascontiguousarray(params)


def gaussian_weights(sigma: float = 2.0, truncate: float = 4.0):
    """scipy.ndimage's 1-D Gaussian kernel (radius = int(truncate*sigma + 0.5)), normalised."""
    r = int(truncate * sigma + 0.5)
    x = np.arange(-r, r + 1, dtype=np.float64)
    w = np.exp(-0.5 * (x / sigma) ** 2)
    return w / w.sum()


def gen_config5_slab(z0: int, z1: int, dims=(2048, 2048, 2048), seed: int = 5, noise_std: float = 0.01,
                     sigma: float = 2.0):
    """Planes [z0, z1) of the config-5 field as a float32 CUDA tensor (64 modes + smoothed noise)."""
    from . import _lib

    t = _lib.torch()
    N0, N1, N2 = dims
    w = gaussian_weights(sigma)
    r = (len(w) - 1) // 2
    e0, e1 = max(0, z0 - r), min(N0, z1 + r)        # noise halo for the z pass
    nz = e1 - e0
    dev = _lib.device()
    a = t.empty((nz, N1, N2), dtype=t.float32, device=dev)
    b = t.empty((nz, N1, N2), dtype=t.float32, device=dev)
    dims_arr = (ctypes.c_int64 * 3)(N0, N1, N2)
    wt = t.from_numpy(w.astype(np.float32)).to(dev)
    _lib.call("hszg_gen_noise", _lib.ptr(a), e0, nz, ctypes.cast(dims_arr, ctypes.c_void_p), ctypes.c_uint64(seed),
              _lib.stream_handle())
    # separable Gaussian, scipy mode="reflect" at the global boundaries
    _lib.call("hszg_gauss_pass", _lib.ptr(a), _lib.ptr(b), e0, nz, ctypes.cast(dims_arr, ctypes.c_void_p), 2,
              _lib.ptr(wt), r, _lib.stream_handle())
    _lib.call("hszg_gauss_pass", _lib.ptr(b), _lib.ptr(a), e0, nz, ctypes.cast(dims_arr, ctypes.c_void_p), 1,
              _lib.ptr(wt), r, _lib.stream_handle())
    out = b[: z1 - z0]
    _lib.call("hszg_gauss_pass_z", _lib.ptr(a), _lib.ptr(out), e0, nz, z0, z1 - z0,
              ctypes.cast(dims_arr, ctypes.c_void_p), _lib.ptr(wt), r, _lib.stream_handle())
    del a
    # unit-variance white noise through the normalised kernel has variance (sum w^2)^3
    scale = noise_std / math.sqrt(float((w ** 2).sum()) ** 3)
    modes = t.from_numpy(config5_modes(seed)).to(dev)
    _lib.call("hszg_gen_modes", _lib.ptr(out), z0, z1 - z0, ctypes.cast(dims_arr, ctypes.c_void_p), _lib.ptr(modes),
              modes.shape[0], ctypes.c_double(scale), _lib.stream_handle())
    return out
