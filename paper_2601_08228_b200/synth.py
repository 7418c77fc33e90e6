"""Seeded synthetic inputs for BASELINE.json's configs (host-side, numpy).

The paper's datasets (Kaggle / GIC hyperspectral cubes) are not available, so
the benchmark and parity cubes are generated here; parameters that
BASELINE.json leaves open are frozen below and recorded in every report
(SURVEY.md section 8(d)).  This is input generation, not the product path.
"""

from __future__ import annotations

import numpy as np

GENERATOR = {
    "abundance": "Dirichlet(alpha=0.5) over E endmembers per pixel, each map gaussian_filter(sigma=4 px, mode=reflect)",
    "spectra": "sum of 3 Gaussian bumps over band index: amplitude U[0.2,1], centre U[0,p), width U[p/32,p/8]",
    "mix": "X = abundances @ spectra + noise_sigma * N(0,1), clipped to [0, 1]",
    "rng": "numpy.random.default_rng(seed), draw order: abundances, spectra (amp, centre, width), noise",
}


def uniform_pair(seed: int = 0):
    """Config 1: A 64x48x32, B 48x40x32, i.i.d. uniform[-1, 1] from one generator."""
    rng = np.random.default_rng(seed)
    a = rng.uniform(-1, 1, (64, 48, 32))
    b = rng.uniform(-1, 1, (48, 40, 32))
    return a, b


def normal_cube(shape=(512, 512, 256), seed: int = 0):
    """Config 2: i.i.d. standard normal."""
    return np.random.default_rng(seed).standard_normal(shape)


def hyperspectral_cube(n1: int, n2: int, p: int, endmembers: int = 10, seed: int = 0,
                       noise: float = 0.01) -> np.ndarray:
    """Configs 3-5: linear-mixing hyperspectral cube (BASELINE.json configs[2])."""
    from scipy.ndimage import gaussian_filter

    rng = np.random.default_rng(seed)
    ab = rng.dirichlet([0.5] * endmembers, (n1, n2))
    for e in range(endmembers):
        ab[:, :, e] = gaussian_filter(ab[:, :, e], sigma=4, mode="reflect")
    amp = rng.uniform(0.2, 1.0, (endmembers, 3))
    cen = rng.uniform(0.0, p, (endmembers, 3))
    wid = rng.uniform(p / 32, p / 8, (endmembers, 3))
    k = np.arange(p, dtype=np.float64)
    spectra = np.zeros((endmembers, p))
    for e in range(endmembers):
        for j in range(3):
            spectra[e] += amp[e, j] * np.exp(-0.5 * ((k - cen[e, j]) / wid[e, j]) ** 2)
    x = (ab.reshape(-1, endmembers) @ spectra).reshape(n1, n2, p)
    x += noise * rng.standard_normal((n1, n2, p))
    np.clip(x, 0.0, 1.0, out=x)
    return x


def _hsi_draws(rng, n1, n2, p, endmembers):
    """The generator's small host draws, in hyperspectral_cube's order: raw Dirichlet
    abundances, then the spectra parameters."""
    ab = rng.dirichlet([0.5] * endmembers, (n1, n2))
    amp = rng.uniform(0.2, 1.0, (endmembers, 3))
    cen = rng.uniform(0.0, p, (endmembers, 3))
    wid = rng.uniform(p / 32, p / 8, (endmembers, 3))
    k = np.arange(p, dtype=np.float64)
    spectra = np.zeros((endmembers, p))
    for e in range(endmembers):
        for j in range(3):
            spectra[e] += amp[e, j] * np.exp(-0.5 * ((k - cen[e, j]) / wid[e, j]) ** 2)
    return ab, spectra


def gaussian_half_kernel(sigma: float = 4.0, truncate: float = 4.0) -> np.ndarray:
    """Centre-to-edge half of the normalised sampled Gaussian of radius
    int(truncate * sigma + 0.5) (the kernel scipy.ndimage.gaussian_filter applies)."""
    radius = int(truncate * float(sigma) + 0.5)
    x = np.arange(-radius, radius + 1)
    phi = np.exp(-0.5 / (sigma * sigma) * x ** 2)
    phi = phi / phi.sum()
    return np.ascontiguousarray(phi[radius:])


def hyperspectral_cube_device(n1: int, n2: int, p: int, endmembers: int = 10, seed: int = 0,
                              noise: float = 0.01, noise_source: str = "philox", device="cuda"):
    """hyperspectral_cube with its heavy stages on the GPU.

    The host draws only the raw abundances and the spectra parameters from
    ``default_rng(seed)`` (n1 n2 E + 9 E numbers); smoothing (reflect-mode separable
    Gaussian, sigma = 4 px), mixing, noise and clipping run in HBM and the cube is
    returned as a CUDA tensor -- the n1 n2 p cube never crosses PCIe.
    ``noise_source="numpy"`` continues the same numpy stream for the noise and uploads
    it, which reproduces hyperspectral_cube to rounding (parity tests);
    ``"philox"`` (default) draws the noise on the device from the Philox-4x32-10
    stream keyed by ``seed`` -- the same distribution, a different seeded stream."""
    from . import engine as E

    if noise_source not in ("philox", "numpy"):
        raise ValueError(f"unknown noise_source {noise_source!r}")
    rng = np.random.default_rng(seed)
    ab, spectra = _hsi_draws(rng, n1, n2, p, endmembers)
    ab_d = E.gauss_smooth2d(E.as_device(ab, device), E.as_device(gaussian_half_kernel(4.0), device))
    z = None
    if noise_source == "numpy" and noise != 0.0:
        z = E.as_device(rng.standard_normal((n1, n2, p)), device)
    return E.hsi_mix(ab_d, E.as_device(spectra, device), noise, z, seed)


def gaussian_taps(taps: int = 9, sigma: float = 2.0) -> np.ndarray:
    """1-D normalised Gaussian PSF (outer product = taps x taps PSF)."""
    h = taps // 2
    d = np.arange(-h, h + 1, dtype=np.float64)
    c = np.exp(-0.5 * (d / sigma) ** 2)
    return c / c.sum()


def toeplitz_blur(n: int, taps: int = 9, sigma: float = 2.0) -> np.ndarray:
    """Banded symmetric Toeplitz A with A[i, j] = c(|i - j|) (SPEC.md:475-479 form)."""
    c = gaussian_taps(taps, sigma)
    h = taps // 2
    a = np.zeros((n, n))
    for off in range(-h, h + 1):
        idx = np.arange(max(0, -off), min(n, n - off))
        a[idx, idx + off] = c[off + h]
    return a


def slice_constant(m: np.ndarray, p: int) -> np.ndarray:
    """(n, n, p) tensor whose every frontal slice is m."""
    return np.ascontiguousarray(np.broadcast_to(m[:, :, None], m.shape + (p,)))


def deblur_problem(n: int = 512, p: int = 128, endmembers: int = 12, seed: int = 0,
                   noise_seed: int = 1, noise: float = 0.005, taps: int = 9, sigma: float = 2.0):
    """Config 5 inputs: X, A_V (slice-constant Toeplitz), A_H, and the noise draw
    (the blurred B itself is produced by the w-product under test)."""
    x = hyperspectral_cube(n, n, p, endmembers=endmembers, seed=seed)
    av = slice_constant(toeplitz_blur(n, taps, sigma), p)
    ah = av
    eta = noise * np.random.default_rng(noise_seed).standard_normal((n, n, p))
    return x, av, ah, eta
