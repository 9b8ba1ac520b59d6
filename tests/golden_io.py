"""Loaders for the committed golden fixtures (tests/golden/*.npz, produced by
running the reference itself: tests/golden/make_golden.py)."""

import hashlib
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def make_rng(seed):
    return np.random.Generator(np.random.Philox(seed))


def ism_cases():
    """Yield (seed, r, v, d, z_ref, z_level_ref, ops_ref)."""
    g = load("ism_systems")
    for i in range(int(g["ncases"])):
        seed, nobs, nens, ops = (int(t) for t in g[f"c{i}_meta"])
        rng = make_rng(seed)
        r = rng.uniform(0.5, 2.0, nobs)
        v = rng.standard_normal((nobs, nens))
        d = rng.standard_normal((nobs, nens))
        assert sha(np.concatenate([r, v.ravel(), d.ravel()])) == str(g[f"c{i}_inputs_sha"])
        yield seed, r, v, d, g[f"c{i}_z"], g[f"c{i}_zlevel"], ops


def kalman_cases():
    g = load("analysis_small")
    for i in range(int(g["nkalman"])):
        yield tuple(g[f"k{i}_{k}"] for k in ("x", "idx", "r", "perturbed", "xa"))


def rel_err(a, b):
    """Normwise max convention of the reference tests: max|a-b| / max|b|."""
    a, b = np.asarray(a), np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def localized_cases():
    """Yield dicts with x, idx (None = identity), r, perturbed, delta, kind, scale, xa."""
    g = load("localized")
    for i in range(int(g["ncases"])):
        c = {k: g[f"l{i}_{k}"] for k in ("x", "r", "perturbed", "delta", "xa")}
        c["idx"] = None if bool(g[f"l{i}_identity"]) else g[f"l{i}_idx"].astype(np.int64)
        c["kind"] = str(g[f"l{i}_kind"])
        sc = float(g[f"l{i}_scale"])
        c["scale"] = None if np.isnan(sc) else sc
        yield c


def l96_cases():
    """Yield (ns, nens, steps, x, xf_sha, xf_rows, row_stride) of the Lorenz96.advance fixture."""
    g = load("lorenz96")
    for i in range(int(g["nforecast"])):
        seed, ns, nens, steps = (int(t) for t in g[f"f{i}_meta"])
        x = 8.0 + make_rng(seed).standard_normal((ns, nens))
        yield ns, nens, steps, x, str(g[f"f{i}_xf_sha"]), g[f"f{i}_xf_rows"], max(1, ns // 64)
