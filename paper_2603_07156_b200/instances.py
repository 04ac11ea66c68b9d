"""Seeded synthetic instances for the five BASELINE.json configurations.

These are harness inputs (SURVEY.md §8(d) "Synthetic inputs"): numpy PCG64
streams, float64 throughout, built on the host and handed bit-identically to
the CUDA path and to the CPU oracle.  The generators restate the recipes in
BASELINE.json ``configs``; choices the configs leave open are fixed here and
recorded in DESIGN.md ("Config decisions"):

* cost matrices are built from explicit coordinate differences
  ``sum_k (x_ik - y_jk)^2`` (numpy's axis-sum order over coordinates);
* config 2 (grid) and config 4 (colour transfer) costs are *not*
  normalised (the config text does not say "normalised"); configs 1, 3, 5
  are normalised to max 1 like ``normalize_cost`` (core.py:159-175);
* config 2's Gaussian filter uses scipy.ndimage's default boundary mode
  ('reflect', truncate 4.0);
* config 4's GMM components have isotropic std 0.05 (unspecified upstream).

The random positive-uniform marginals redraw exact zeros like
data.py:22-29 of the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Instance:
    name: str
    cost: np.ndarray
    a: np.ndarray
    b: np.ndarray
    eta: float
    kkt_tol: float


CONFIGS = {
    1: dict(name="cfg1-uniform2d-1000", m=1000, n=1000, eta=1e-2, tol=1e-6),
    2: dict(name="cfg2-grid64-4096", m=4096, n=4096, eta=1e-2, tol=1e-6),
    3: dict(name="cfg3-gmm3d-10000", m=10000, n=10000, eta=5e-3, tol=1e-7),
    4: dict(name="cfg4-colour-65536x16384", m=65536, n=16384, eta=1e-2, tol=1e-6),
    5: dict(name="cfg5-uniform2d-50000", m=50000, n=50000, eta=1e-2, tol=1e-6),
}


def positive_uniform(rng: np.random.Generator, size: int) -> np.ndarray:
    """U(0,1) draws with exact zeros redrawn (reference data.py:22-29)."""
    draws = rng.random(size)
    while True:
        zero = draws == 0.0
        if not zero.any():
            return draws
        draws[zero] = rng.random(int(zero.sum()))


def normalise(cost: np.ndarray) -> np.ndarray:
    """cost / max(cost) (reference core.py:159-175), all-zero left unchanged."""
    peak = cost.max()
    return cost.copy() if peak == 0.0 else cost / peak


def sq_dist(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """Squared Euclidean distances, summed over coordinates in order."""
    d = x[:, None, :] - y[None, :, :]
    return (d * d).sum(axis=2)


def _gmm(rng, count, comps, dim, std):
    means = rng.random((comps, dim))
    label = rng.integers(0, comps, size=count)
    return means[label] + std * rng.standard_normal((count, dim))


@dataclass(frozen=True)
class PointInstance:
    """The points and marginals an Instance is built from (cost = squared
    Euclidean distances, normalised to max 1 when `normalised`)."""
    name: str
    x: np.ndarray
    y: np.ndarray
    a: np.ndarray
    b: np.ndarray
    normalised: bool
    eta: float
    kkt_tol: float

    def build(self) -> "Instance":
        cost = sq_dist(self.x, self.y)
        if self.normalised:
            cost = normalise(cost)
        return Instance(self.name, cost, self.a, self.b, self.eta, self.kkt_tol)


def uniform2d_points(m: int, n: int, seed: int, eta: float = 1e-2, tol: float = 1e-6, name=None) -> PointInstance:
    """Configs 1 and 5: points U[0,1]^2, normalised squared distance,
    random positive marginals."""
    rng = np.random.default_rng(seed)
    x = rng.random((m, 2))
    y = rng.random((n, 2))
    a = positive_uniform(rng, m)
    b = positive_uniform(rng, n)
    return PointInstance(name or f"uniform2d-{m}x{n}-s{seed}", x, y, a / a.sum(), b / b.sum(), True, eta, tol)


def uniform2d(m: int, n: int, seed: int, eta: float = 1e-2, tol: float = 1e-6, name=None) -> Instance:
    return uniform2d_points(m, n, seed, eta, tol, name).build()


def grid_points(side: int, seed: int, eta: float = 1e-2, tol: float = 1e-6, sigma: float = 3.0) -> PointInstance:
    """Config 2: side x side pixel grid, unnormalised squared distance,
    marginals exp(gaussian_filter(N(0,1))) + 1e-6 normalised."""
    from scipy.ndimage import gaussian_filter

    rng = np.random.default_rng(seed)
    r, c = np.divmod(np.arange(side * side), side)
    pts = np.stack(((r + 0.5) / side, (c + 0.5) / side), axis=1)
    ha = np.exp(gaussian_filter(rng.standard_normal((side, side)), sigma)) + 1e-6
    hb = np.exp(gaussian_filter(rng.standard_normal((side, side)), sigma)) + 1e-6
    a = ha.ravel()
    b = hb.ravel()
    return PointInstance(f"grid{side}-s{seed}", pts, pts, a / a.sum(), b / b.sum(), False, eta, tol)


def grid_histograms(side: int, seed: int, eta: float = 1e-2, tol: float = 1e-6, sigma: float = 3.0) -> Instance:
    return grid_points(side, seed, eta, tol, sigma).build()


def gmm_points(m: int, n: int, seed: int, eta: float = 5e-3, tol: float = 1e-7) -> PointInstance:
    """Config 3: two 8-component 3-D Gaussian mixtures (std 0.05),
    normalised squared distance, uniform marginals."""
    rng = np.random.default_rng(seed)
    x = _gmm(rng, m, 8, 3, 0.05)
    y = _gmm(rng, n, 8, 3, 0.05)
    return PointInstance(f"gmm3d-{m}x{n}-s{seed}", x, y, np.full(m, 1.0 / m), np.full(n, 1.0 / n), True, eta, tol)


def gmm_clouds(m: int, n: int, seed: int, eta: float = 5e-3, tol: float = 1e-7) -> Instance:
    return gmm_points(m, n, seed, eta, tol).build()


def colour_points(m: int, n: int, seed: int, eta: float = 1e-2, tol: float = 1e-6) -> PointInstance:
    """Config 4: source RGB from a 16-component GMM (std 0.05) clipped to
    [0,1]^3, target RGB uniform, unnormalised squared distance, uniform
    marginals."""
    rng = np.random.default_rng(seed)
    x = np.clip(_gmm(rng, m, 16, 3, 0.05), 0.0, 1.0)
    y = rng.random((n, 3))
    return PointInstance(f"colour-{m}x{n}-s{seed}", x, y, np.full(m, 1.0 / m), np.full(n, 1.0 / n), False, eta, tol)


def colour_transfer(m: int, n: int, seed: int, eta: float = 1e-2, tol: float = 1e-6) -> Instance:
    return colour_points(m, n, seed, eta, tol).build()


def config_points(idx: int, seed: int = 0) -> PointInstance:
    """The points and marginals of BASELINE.json configuration ``idx``."""
    c = CONFIGS[idx]
    name = f"{c['name']}-s{seed}"
    if idx == 1:
        p = uniform2d_points(1000, 1000, seed, c["eta"], c["tol"])
    elif idx == 2:
        p = grid_points(64, seed, c["eta"], c["tol"])
    elif idx == 3:
        p = gmm_points(10000, 10000, seed, c["eta"], c["tol"])
    elif idx == 4:
        p = colour_points(65536, 16384, seed, c["eta"], c["tol"])
    elif idx == 5:
        p = uniform2d_points(50000, 50000, seed, c["eta"], c["tol"])
    else:
        raise KeyError(idx)
    return PointInstance(name, p.x, p.y, p.a, p.b, p.normalised, p.eta, p.kkt_tol)


def config(idx: int, seed: int = 0) -> Instance:
    """The BASELINE.json configuration ``idx`` (1-based) at ``seed``, built on the host."""
    return config_points(idx, seed).build()


def device_cost(points: PointInstance, device, rows: tuple[int, int] | None = None, ld: int | None = None,
                comm=None):
    """Rows [r0, r1) of the instance's cost matrix built on the GPU by libotb
    (otb_sq_dist + otb_scale_cost): bit-identical to ``points.build().cost``
    without the m x n host array.  Returns a (r1 - r0, n) float64 CUDA
    tensor (a view of an (r1 - r0, ld) buffer when ld > n).  Multi-rank:
    the normalising peak is max-reduced over `comm` (torch.distributed)."""
    import ctypes as C

    import torch

    from . import _lib

    m, n = points.x.shape[0], points.y.shape[0]
    r0, r1 = rows if rows is not None else (0, m)
    ld = n if ld is None else ld
    dim = points.x.shape[1]
    x = torch.from_numpy(np.ascontiguousarray(points.x)).to(device)
    y = torch.from_numpy(np.ascontiguousarray(points.y)).to(device)
    buf = torch.empty((r1 - r0, ld), dtype=torch.float64, device=device)
    if ld > n:
        buf[:, n:].zero_()
    stream = torch.cuda.current_stream(device).cuda_stream
    peak = C.c_double()
    _lib.check(_lib.lib.otb_sq_dist(x.data_ptr(), y.data_ptr(), r1 - r0, n, dim, r0, buf.data_ptr(), ld,
                                    C.byref(peak), C.c_void_p(stream)))
    if points.normalised:
        p = peak.value
        if comm is not None and getattr(comm, "world", 1) > 1:
            t = torch.tensor([p], dtype=torch.float64, device=device)
            comm.all_reduce_(t, op="max")
            p = float(t.item())
        _lib.check(_lib.lib.otb_scale_cost(buf.data_ptr(), r1 - r0, n, ld, p, C.c_void_p(stream)))
    return buf[:, :n] if ld > n else buf


def small_uniform(m: int, n: int, seed: int) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Uniform random cost entries + positive marginals, the recipe of the
    reference's ``gen_uniform`` (data.py:38-43), for small parity cases."""
    rng = np.random.default_rng(seed)
    cost = normalise(rng.random((m, n)))
    a = positive_uniform(rng, m)
    b = positive_uniform(rng, n)
    return cost, a / a.sum(), b / b.sum()
