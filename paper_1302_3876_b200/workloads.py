"""Seeded synthetic inputs for the five BASELINE.json configurations.

No public dataset is involved: every config is synthetic.  Host (numpy)
generation uses Philox-4x64 exactly like the reference's `make_rng`
(rng.py:13-20) so the same seeds give the same arrays on any host; the
full-size bench inputs of configs 4/5 are drawn on the device with torch's
Philox (same shapes and distributions, different stream) because the host
would need minutes and 70+ GiB to draw them.

Config summary (BASELINE.json "configs"):
  1  Lorenz-96 Ns=40, N=20, every other component observed (Nobs=20), R=0.01 I
  2  Lorenz-96 Ns=Nobs=4096 (identity H), N=64, R=0.1^2 I, 5 RK4 steps/cycle, 100 cycles
  3  QG-shaped 129x129 field (Ns=16641), N=96, stride-4 subgrid (Nobs=1089),
     k^-3 Gaussian random fields, R diagonal with std ~ U[0.5, 1.5]
  4  Ns=2^24, N=128, Nobs=2^20 random distinct indices, X = mu + sigma eps
  5  Ns=2^26, N=128, Nobs=2^23, as config 4, sharded over 1/2/4/8 GPUs
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

SEEDS = {
    1: dict(truth=101, ens=102, obs=103),
    2: dict(truth=201, ens=202, obs=203),
    3: dict(field=301, ens=302, obs=303, h=304),
    4: dict(state=401, h=402, obs=403),
    5: dict(state=501, h=502, obs=503),
}

SIZES = {
    1: dict(ns=40, nens=20, nobs=20),
    2: dict(ns=4096, nens=64, nobs=4096),
    3: dict(ns=129 * 129, nens=96, nobs=33 * 33),
    4: dict(ns=1 << 24, nens=128, nobs=1 << 20),
    5: dict(ns=1 << 26, nens=128, nobs=1 << 23),
}

CHUNK_ROWS = 1 << 20  # generation granularity of configs 4/5 (G-invariant sharding)


def make_rng(seed: int) -> np.random.Generator:
    """rng.py:13-20 — Philox-4x64 generator."""
    return np.random.Generator(np.random.Philox(seed))


def gaussian_matrix(rng, rows, cols, mean=0.0, std=1.0):
    """rng.py:23-62 — N(mean, std_i^2) entries, std scalar or per row."""
    std = np.asarray(std, dtype=float)
    scale = std if std.ndim == 0 else std[:, None]
    return mean + rng.standard_normal((rows, cols)) * scale


def uniform_stride_indices(nstate: int, pobs: float):
    """observations.py:70-101, "uniform-stride": index k = floor(k Ns / Nobs);
    None when every component is observed (identity)."""
    nobs = max(1, int(pobs * nstate))
    if nobs == nstate:
        return None
    return (np.arange(nobs) * nstate) // nobs


def random_indices(nstate: int, pobs: float, seed: int):
    """observations.py:95-96, "random": sorted sample without replacement from
    make_rng(seed) — the same draw the reference makes, so the observed set is
    identical."""
    nobs = max(1, int(pobs * nstate))
    idx = np.sort(make_rng(seed).choice(nstate, size=nobs, replace=False))
    if nobs == nstate:
        return None
    return idx


# --------------------------------------------------------------------------
# Lorenz-96 (models/lorenz96.py:31-49), host numpy: used only to spin up and
# advance the config 1/2 inputs.
def l96_tendency(x, forcing=8.0):
    return (np.roll(x, -1, axis=0) - np.roll(x, 2, axis=0)) * np.roll(x, 1, axis=0) - x + forcing


def l96_rk4(x, dt=0.05, forcing=8.0):
    k1 = l96_tendency(x, forcing)
    k2 = l96_tendency(x + 0.5 * dt * k1, forcing)
    k3 = l96_tendency(x + 0.5 * dt * k2, forcing)
    k4 = l96_tendency(x + dt * k3, forcing)
    return x + (dt / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)


@dataclass
class Problem:
    """One analysis problem in the reference's array layout."""

    x: np.ndarray            # (Ns, N) C order
    perturbed: np.ndarray    # (Nobs, N)
    y: np.ndarray            # (Nobs,)
    indices: np.ndarray | None  # sorted int64 or None (identity)
    r: np.ndarray            # (Nobs,)
    name: str = ""

    @property
    def shape(self):
        return (self.x.shape[0], self.perturbed.shape[0], self.x.shape[1])


def _perturb(rng, y, r, nens):
    """enkf.py:95-111 — Y_j = y + eps_j, eps_j ~ N(0, diag(r))."""
    eps = gaussian_matrix(rng, y.shape[0], nens, 0.0, np.sqrt(r))
    return y[:, None] + eps


def config1() -> Problem:
    s = SEEDS[1]
    ns, nens = SIZES[1]["ns"], SIZES[1]["nens"]
    truth = gaussian_matrix(make_rng(s["truth"]), ns, 1, 8.0, 0.01)[:, 0]
    for _ in range(1000):
        truth = l96_rk4(truth)
    x = truth[:, None] + gaussian_matrix(make_rng(s["ens"]), ns, nens, 0.0, 1.0)
    idx = uniform_stride_indices(ns, 0.5)
    r = np.full(idx.size, 0.01)
    rng = make_rng(s["obs"])
    y = truth[idx] + gaussian_matrix(rng, idx.size, 1, 0.0, np.sqrt(r))[:, 0]
    return Problem(np.ascontiguousarray(x), _perturb(rng, y, r, nens), y, idx, r, "config1")


class Config2Cycler:
    """Config 2: L96-4096, identity H, 5 RK4 steps between analyses.  The
    forecast is host numpy (input generation); `cycle()` returns the problem
    of the next analysis given the current analysis ensemble."""

    def __init__(self, ns=None, nens=None):
        s = SEEDS[2]
        self.ns = ns or SIZES[2]["ns"]
        self.nens = nens or SIZES[2]["nens"]
        truth = gaussian_matrix(make_rng(s["truth"]), self.ns, 1, 8.0, 0.01)[:, 0]
        for _ in range(1000):
            truth = l96_rk4(truth)
        self.truth = truth
        self.x = truth[:, None] + gaussian_matrix(make_rng(s["ens"]), self.ns, self.nens, 0.0, 1.0)
        self.r = np.full(self.ns, 0.1 ** 2)
        self.rng = make_rng(s["obs"])

    def cycle(self, xa=None) -> Problem:
        if xa is not None:
            self.x = np.asarray(xa)
        for _ in range(5):
            self.truth = l96_rk4(self.truth)
            self.x = l96_rk4(self.x)
        y = self.truth + gaussian_matrix(self.rng, self.ns, 1, 0.0, np.sqrt(self.r))[:, 0]
        return Problem(np.ascontiguousarray(self.x), _perturb(self.rng, y, self.r, self.nens),
                       y, None, self.r, "config2")


def gaussian_random_field(rng, n: int, slope: float = -3.0) -> np.ndarray:
    """Smooth periodic GRF on an n x n grid with power spectrum ~ k^slope,
    normalised to zero mean and unit variance."""
    white = rng.standard_normal((n, n))
    kx = np.fft.fftfreq(n)[:, None]
    ky = np.fft.rfftfreq(n)[None, :]
    k = np.sqrt(kx * kx + ky * ky)
    amp = np.zeros_like(k)
    amp[k > 0] = k[k > 0] ** (slope / 2.0)
    f = np.fft.irfft2(np.fft.rfft2(white) * amp, s=(n, n))
    f -= f.mean()
    return f / f.std()


def config3() -> Problem:
    s = SEEDS[3]
    g, nens = 129, SIZES[3]["nens"]
    rf = make_rng(s["field"])
    mean = gaussian_random_field(rf, g).ravel()
    truth = mean + gaussian_random_field(rf, g).ravel()
    re = make_rng(s["ens"])
    x = np.stack([mean + gaussian_random_field(re, g).ravel() for _ in range(nens)], axis=1)
    sub = np.arange(0, g, 4)
    idx = np.sort((sub[:, None] * g + sub[None, :]).ravel()).astype(np.int64)
    ro = make_rng(s["obs"])
    std = ro.uniform(0.5, 1.5, idx.size)
    r = std * std
    y = truth[idx] + std * ro.standard_normal(idx.size)
    return Problem(np.ascontiguousarray(x), _perturb(ro, y, r, nens), y, idx, r, "config3")


def _chunked_normals(seed: int, rows: int, cols: int, chunk: int = 1 << 16, threads: int = 8):
    """Standard normals from independent Philox streams per row chunk
    (Philox(seed).jumped(c)); multithreaded, deterministic."""
    out = np.empty((rows, cols))

    def fill(c):
        lo = c * chunk
        hi = min(rows, lo + chunk)
        g = np.random.Generator(np.random.Philox(seed).jumped(c))
        out[lo:hi] = g.standard_normal((hi - lo, cols))

    nchunks = (rows + chunk - 1) // chunk
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(fill, range(nchunks)))
    return out


def large_problem(ns: int, nobs: int, nens: int = 128, seed_state=401, seed_h=402, seed_obs=403,
                  name="large") -> Problem:
    """Configs 4/5 value distributions at any size (host numpy):
    X_ij = mu_i + sigma_i eps_ij, mu ~ N(0,1), sigma ~ U[0.5, 2]; H = sorted
    random distinct indices; r ~ U[0.25, 1]; y = H(mu + sigma eps_truth) +
    sqrt(r) eta; Y_j = y + sqrt(r) xi_j."""
    rs = make_rng(seed_state)
    mu = rs.standard_normal(ns)
    sigma = rs.uniform(0.5, 2.0, ns)
    x = _chunked_normals(seed_state + 7919, ns, nens)
    x *= sigma[:, None]
    x += mu[:, None]
    idx = random_indices(ns, nobs / ns, seed_h)
    idx_arr = np.arange(ns) if idx is None else idx
    ro = make_rng(seed_obs)
    r = ro.uniform(0.25, 1.0, nobs)
    truth_obs = mu[idx_arr] + sigma[idx_arr] * ro.standard_normal(nobs)
    y = truth_obs + np.sqrt(r) * ro.standard_normal(nobs)
    xi = _chunked_normals(seed_obs + 7919, nobs, nens)
    xi *= np.sqrt(r)[:, None]
    xi += y[:, None]
    return Problem(x, xi, y, idx, r, name)


def config4(scale_log2: int = 0) -> Problem:
    s, z = SEEDS[4], SIZES[4]
    return large_problem(z["ns"] >> scale_log2, z["nobs"] >> scale_log2, z["nens"],
                         s["state"], s["h"], s["obs"], f"config4/2^{scale_log2}")


def config5(scale_log2: int = 0) -> Problem:
    s, z = SEEDS[5], SIZES[5]
    return large_problem(z["ns"] >> scale_log2, z["nobs"] >> scale_log2, z["nens"],
                         s["state"], s["h"], s["obs"], f"config5/2^{scale_log2}")


# --------------------------------------------------------------------------
# Device generation of the config 4/5 shapes (bench), sharded by state rows.
from .distributed import obs_slice, shard_rows  # noqa: E402  (one definition of the sharding)


def device_problem_shard(cfg: int, world: int = 1, rank: int = 0, device=None,
                         scale_log2: int = 0, indices=None):
    """Config 4/5 inputs for state rows [lo, hi) of this rank, drawn on the GPU
    in CHUNK_ROWS state chunks seeded by chunk id (so the global problem does
    not depend on the GPU count).  Returns dict of CUDA tensors + metadata."""
    import torch

    z, s = SIZES[cfg], SEEDS[cfg]
    ns, nobs, nens = z["ns"] >> scale_log2, z["nobs"] >> scale_log2, z["nens"]
    if indices is None:
        indices = random_indices(ns, nobs / ns, s["h"])
    lo, hi = shard_rows(ns, world, rank)
    o_lo, o_hi = obs_slice(indices, lo, hi)
    device = device or torch.device("cuda", torch.cuda.current_device())
    x = torch.empty((hi - lo, nens), dtype=torch.float64, device=device)
    m = o_hi - o_lo
    yv = torch.empty((m, nens), dtype=torch.float64, device=device)
    r = torch.empty(m, dtype=torch.float64, device=device)
    loc_idx = torch.from_numpy(np.ascontiguousarray(indices[o_lo:o_hi] - lo, dtype=np.int64)).to(device)
    chunk = min(CHUNK_ROWS, ns)
    gen = torch.Generator(device=device)
    c0 = lo // chunk
    c1 = (hi + chunk - 1) // chunk
    for c in range(c0, c1):
        a, b = max(lo, c * chunk), min(hi, (c + 1) * chunk)
        gen.manual_seed(s["state"] * 1_000_003 + c)
        mu = torch.randn(chunk, dtype=torch.float64, device=device, generator=gen)
        sigma = torch.rand(chunk, dtype=torch.float64, device=device, generator=gen) * 1.5 + 0.5
        eps = torch.randn((chunk, nens), dtype=torch.float64, device=device, generator=gen)
        rows = slice(a - c * chunk, b - c * chunk)
        x[a - lo:b - lo] = mu[rows, None] + sigma[rows, None] * eps[rows]
        # observations whose index lies in this chunk
        ca, cb = obs_slice(indices, c * chunk, (c + 1) * chunk)
        if cb > ca:
            gen.manual_seed(s["obs"] * 1_000_003 + c)
            k = cb - ca
            rr = torch.rand(k, dtype=torch.float64, device=device, generator=gen) * 0.75 + 0.25
            tr = torch.randn(k, dtype=torch.float64, device=device, generator=gen)
            eta = torch.randn(k, dtype=torch.float64, device=device, generator=gen)
            xi = torch.randn((k, nens), dtype=torch.float64, device=device, generator=gen)
            loc = torch.from_numpy(np.ascontiguousarray(indices[ca:cb] - c * chunk)).to(device)
            yy = mu[loc] + sigma[loc] * tr + rr.sqrt() * eta
            sa, sb = max(ca, o_lo), min(cb, o_hi)
            if sb > sa:
                sel = slice(sa - ca, sb - ca)
                r[sa - o_lo:sb - o_lo] = rr[sel]
                yv[sa - o_lo:sb - o_lo] = yy[sel, None] + rr[sel].sqrt()[:, None] * xi[sel]
        del mu, sigma, eps
    return dict(x=x, perturbed=yv, r=r, idx=loc_idx, lo=lo, hi=hi, o_lo=o_lo, o_hi=o_hi,
                ns=ns, nobs=nobs, nens=nens, identity=False)
