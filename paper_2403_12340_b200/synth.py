"""Seeded synthetic workloads with the BASELINE.json configs' shapes.

BASELINE.json names no public dataset (the paper's KSSOLV Si8/Si64/C60 inputs
are not in this container), so every run uses seeded synthetic orbitals and
energies with the stated grids, band counts and energy ranges:

  orbitals  first N_v / next N_c columns of the QR of a seeded N(0,1)
            N_r x (N_v+N_c) matrix (unit L2 columns on the grid); for C60,
            QR of seeded combinations of 4 Gaussians (widths 0.6/0.9/1.3/1.9
            bohr) on each of 60 centres drawn in a 7-bohr ball (the literal
            60-Gaussian recipe spans only 60 dimensions; builder's choice,
            SURVEY §8d)
  energies  seeded uniform occupied / virtual draws, sorted, HOMO pinned to
            the top of the occupied range and LUMO to the bottom of the
            virtual range (q = stated gap exactly)
  probe     seeded N(0,1) N_r x 8 block

Input generation is plumbing (numpy on host for small grids, torch on the
device for large ones); it is never timed.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    dims: tuple
    cell: float
    n_v: int
    n_c: int
    occ: tuple
    virt: tuple
    k_mu: float
    n_lambda: int
    kind: str = "si"

    @property
    def n_r(self):
        return self.dims[0] * self.dims[1] * self.dims[2]

    @property
    def cell3(self):
        return (self.cell, self.cell, self.cell)


CONFIGS = {
    "si8": Config("si8", (24, 24, 24), 10.26, 16, 16, (-0.50, -0.10), (0.05, 0.80), 8.0, 16),
    "si64": Config("si64", (48, 48, 48), 20.52, 128, 128, (-0.50, -0.10), (0.05, 0.80), 8.0, 24),
    "c60": Config("c60", (80, 80, 80), 30.0, 120, 120, (-0.80, -0.22), (-0.12, 0.60), 8.0, 32, "c60"),
    "si216": Config("si216", (72, 72, 72), 30.78, 432, 432, (-0.50, -0.10), (0.02, 0.80), 8.0, 32),
    "si512": Config("si512", (96, 96, 96), 41.04, 1024, 1024, (-0.50, -0.10), (0.00, 0.80), 8.0, 40),
}


def energies(cfg: Config, seed: int = 2) -> np.ndarray:
    rng = np.random.default_rng(seed)
    ev = np.sort(rng.uniform(cfg.occ[0], cfg.occ[1], cfg.n_v))
    ec = np.sort(rng.uniform(cfg.virt[0], cfg.virt[1], cfg.n_c))
    ev[-1] = cfg.occ[1]
    ec[0] = cfg.virt[0]
    return np.concatenate([ev, ec])


def orbitals_host(cfg: Config, seed: int = 1) -> np.ndarray:
    """N_r x (N_v + N_c) Fortran-order orthonormal columns (numpy QR)."""
    rng = np.random.default_rng(seed)
    g = rng.standard_normal((cfg.n_r, cfg.n_v + cfg.n_c))
    q, _ = np.linalg.qr(g)
    return np.asfortranarray(q)


def orbitals_device(cfg: Config, seed: int = 1, device="cuda"):
    """Same recipe on the GPU (torch QR); returns a column-major float64 tensor."""
    import torch

    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    nb = cfg.n_v + cfg.n_c
    if cfg.kind == "c60":
        g = _c60_basis(cfg, seed, device)
    else:
        g = torch.randn(cfg.n_r, nb, generator=gen, dtype=torch.float64, device=device)
    q, _ = torch.linalg.qr(g)
    return q.t().contiguous().t()  # column-major (stride(0) == 1)


def _c60_basis(cfg: Config, seed: int, device):
    import torch

    rng = np.random.default_rng(seed + 2)
    centres = []
    c0 = np.full(3, cfg.cell / 2.0)
    while len(centres) < 60:
        p = rng.uniform(-7.0, 7.0, 3)
        if np.linalg.norm(p) <= 7.0:
            centres.append(c0 + p)
    widths = (0.6, 0.9, 1.3, 1.9)
    n1, n2, n3 = cfg.dims
    h = cfg.cell / np.array([n1, n2, n3])
    x = torch.arange(n1, device=device, dtype=torch.float64) * h[0]
    y = torch.arange(n2, device=device, dtype=torch.float64) * h[1]
    z = torch.arange(n3, device=device, dtype=torch.float64) * h[2]
    funcs = []
    for c in centres:
        dx = torch.remainder(x - c[0] + cfg.cell / 2, cfg.cell) - cfg.cell / 2
        dy = torch.remainder(y - c[1] + cfg.cell / 2, cfg.cell) - cfg.cell / 2
        dz = torch.remainder(z - c[2] + cfg.cell / 2, cfg.cell) - cfg.cell / 2
        r2 = dz[:, None, None] ** 2 + dy[None, :, None] ** 2 + dx[None, None, :] ** 2
        for w in widths:
            funcs.append(torch.exp(-r2 / (2 * w * w)).reshape(-1))
    basis = torch.stack(funcs, dim=1)  # N_r x 240, flat index i1 + n1 (i2 + n2 i3)
    coef = torch.as_tensor(np.random.default_rng(seed + 3).standard_normal((basis.shape[1], cfg.n_v + cfg.n_c)),
                           device=device)
    return basis @ coef


def probe_host(n_r: int, m: int = 8, seed: int = 0xA5A5A5A4) -> np.ndarray:
    return np.asfortranarray(np.random.default_rng(seed).standard_normal((n_r, m)))
