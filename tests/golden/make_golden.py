"""Generate the golden fixtures by running the REFERENCE itself.

Run in the build container (the reference is importable only there):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [fixture ...]
It imports `enkfkit` from /root/reference/pkg/src (read-only) and writes
small .npz files next to this script.  The GPU box never reads the reference;
tests compare the oracle restatement (CPU tests) and the CUDA path (GPU tests)
against these files.  Inputs are regenerated from the recorded Philox seeds
where storing them would be large; a checksum of every regenerated input is
stored so drift is detected.
"""

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)
sys.dont_write_bytecode = True

import enkfkit  # noqa: E402  (the reference)
from enkfkit import enkf as ref_enkf  # noqa: E402
from enkfkit import sherman as ref_sherman  # noqa: E402
from enkfkit.models import Lorenz96, Lorenz96Config  # noqa: E402
from enkfkit.observations import build_selection_operator  # noqa: E402
from enkfkit.rng import gaussian_matrix, make_rng  # noqa: E402

from paper_1302_3876_b200 import workloads as W  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ism_systems():
    """solve_sherman on random systems: the reference tests' shapes
    (tests/test_sherman.py:41-53, 85-94; test_acceptance.py:44-61)."""
    out = {}
    cases = [(31, 5, 3), (90, 50, 2), (56, 200, 16), (168, 2000, 128), (57, 150, 1),
             (59, 150, 3), (64, 150, 8), (65, 150, 9), (72, 150, 16), (87, 150, 31)]
    rng = make_rng(0xA1)
    for _ in range(12):  # C1-style: Nobs log-uniform 10-500, N log-uniform 2-64
        nobs = int(round(np.exp(rng.uniform(np.log(10), np.log(500)))))
        nens = int(round(np.exp(rng.uniform(np.log(2), np.log(64)))))
        cases.append((int(rng.integers(1000, 10**6)), nobs, nens))
    for i, (seed, nobs, nens) in enumerate(cases):
        g = make_rng(seed)
        r = g.uniform(0.5, 2.0, nobs)
        v = g.standard_normal((nobs, nens))
        d = g.standard_normal((nobs, nens))
        res = ref_sherman.solve_sherman(r, v, d)
        zl, ops = ref_sherman._sweep_reference(r, v, d, count_ops=True, verify_frozen=False)
        out[f"c{i}_meta"] = np.array([seed, nobs, nens, ops])
        out[f"c{i}_z"] = res.z
        out[f"c{i}_zlevel"] = zl
        out[f"c{i}_inputs_sha"] = np.array(sha(np.concatenate([r, v.ravel(), d.ravel()])))
    out["ncases"] = np.array(len(cases))
    out["opcount"] = np.array([[n, m, ref_sherman.long_op_count(n, m)] for n, m in
                               [(3, 3), (1, 1), (4, 10), (2, 7), (5, 40), (16, 320), (128, 1 << 20)]])
    return out


def analysis_small():
    """analysis_step on the Kalman-gain oracle instances (test_acceptance.py:88-115),
    zero spread (test_enkf.py:208-213), uninformative obs (:203-206)."""
    out = {}
    rng = make_rng(0xA3)
    for i in range(20):
        nstate = int(rng.integers(6, 21))
        nens = int(rng.integers(3, 7))
        nobs = int(rng.integers(2, min(nstate, 10) + 1))
        x = rng.standard_normal((nstate, nens))
        idx = np.sort(rng.choice(nstate, size=nobs, replace=False))
        h = ref_enkf.SelectionOperator.from_indices(idx)
        r = rng.uniform(0.2, 1.0, nobs)
        y = rng.standard_normal(nobs)
        eps = 0.2 * rng.standard_normal((nobs, nens))
        obs = ref_enkf.ObservationBatch(y=y, perturbed=y[:, None] + eps, perturbations=eps)
        xa = ref_enkf.analysis_step(x, obs, h, r, "sherman")
        for k, val in dict(x=x, idx=idx, r=r, perturbed=obs.perturbed, xa=xa).items():
            out[f"k{i}_{k}"] = val
    out["nkalman"] = np.array(20)
    x = np.tile(np.arange(6.0)[:, None], (1, 4))
    h = ref_enkf.SelectionOperator.from_indices([1, 4])
    yb = np.array([5.0, -2.0])
    obs = ref_enkf.ObservationBatch(y=yb, perturbed=yb[:, None] + np.zeros((2, 4)), perturbations=np.zeros((2, 4)))
    out["zero_x"], out["zero_xa"] = x, ref_enkf.analysis_step(x, obs, h, np.ones(2), "sherman")
    return out


def config_fixtures():
    out = {}
    # config 1 built with the reference's own model/observation code
    ns, nens = 40, 20
    s = W.SEEDS[1]
    truth = gaussian_matrix(make_rng(s["truth"]), ns, 1, 8.0, 0.01)[:, 0]
    model = Lorenz96(Lorenz96Config(nstate=ns, forcing=8.0, dt=0.05))
    truth = model.advance(truth, 0.0, 1000 * 0.05)
    x = truth[:, None] + gaussian_matrix(make_rng(s["ens"]), ns, nens, 0.0, 1.0)
    h = build_selection_operator(ns, 0.5)
    r = np.full(h.nobs(ns), 0.01)
    rng = make_rng(s["obs"])
    y = h.apply(truth) + gaussian_matrix(rng, r.size, 1, 0.0, np.sqrt(r))[:, 0]
    obs = ref_enkf.perturb_observations(y, r, nens, rng)
    xa = ref_enkf.analysis_step(x, obs, h, r, "sherman")
    out.update(c1_x=x, c1_idx=h.indices, c1_r=r, c1_perturbed=obs.perturbed, c1_xa=xa)

    # configs 2 (first cycle), 3 and a scaled config 4: inputs from our seeded
    # generators (checksummed), outputs from the reference's analysis_step.
    cyc = W.Config2Cycler()
    p2 = cyc.cycle()
    p3 = W.config3()
    p4 = W.config4(8)
    for tag, p in (("c2", p2), ("c3", p3), ("c4s8", p4)):
        h = ref_enkf.SelectionOperator.identity() if p.indices is None else \
            ref_enkf.SelectionOperator.from_indices(p.indices)
        ob = ref_enkf.ObservationBatch(y=p.y, perturbed=p.perturbed, perturbations=p.perturbed - p.y[:, None])
        xa = ref_enkf.analysis_step(p.x, ob, h, p.r, "sherman")
        stride = max(1, p.x.shape[0] // 512)
        out[f"{tag}_input_sha"] = np.array(sha(np.concatenate([p.x.ravel(), p.perturbed.ravel(), p.r])))
        out[f"{tag}_stride"] = np.array(stride)
        out[f"{tag}_xa_rows"] = xa[::stride]
        out[f"{tag}_xa_colsum"] = xa.sum(axis=0)
        out[f"{tag}_xa_absmax"] = np.array(np.abs(xa).max())
    return out


def selections():
    """'Identical observation-index selection': the reference's
    build_selection_operator for every config's H."""
    out = {}
    h1 = build_selection_operator(40, 0.5)
    out["c1"] = h1.indices
    h2 = build_selection_operator(4096, 1.0)
    out["c2_identity"] = np.array(h2.indices is None)
    for cfg in (4, 5):
        z, s = W.SIZES[cfg], W.SEEDS[cfg]
        h = build_selection_operator(z["ns"], z["nobs"] / z["ns"], "random", s["h"])
        out[f"c{cfg}_sha"] = np.array(sha(h.indices.astype(np.int64)))
        out[f"c{cfg}_head"] = h.indices[:512]
        out[f"c{cfg}_tail"] = h.indices[-512:]
        out[f"c{cfg}_n"] = np.array(h.indices.size)
    for sl in (8, 6):
        z, s = W.SIZES[4], W.SEEDS[4]
        ns, nobs = z["ns"] >> sl, z["nobs"] >> sl
        h = build_selection_operator(ns, nobs / ns, "random", s["h"])
        out[f"c4s{sl}_sha"] = np.array(sha(h.indices.astype(np.int64)))
    return out


def localized():
    """Localized analysis (enkf.py:193-199) with the reference's own
    influence_matrix_cyclic (enkf.py:138-164): the lorenz-small preset shape
    (40 x 20, fully observed, scale 8), a partially observed ring, a random
    dense influence matrix (test_enkf.py:235-252 style) and unit influence
    (test_enkf.py:254-260)."""
    out = {}
    rng = make_rng(0xA5)
    cases = [(40, 20, None, 8.0, "cyclic"), (64, 12, 16, 5.0, "cyclic"), (9, 4, 5, None, "uniform"),
             (10, 4, 6, None, "ones"), (130, 33, 40, None, "cyclic"), (50, 7, 50, 3.0, "cyclic")]
    for i, (nstate, nens, nobs, scale, kind) in enumerate(cases):
        x = rng.standard_normal((nstate, nens)) + 8.0
        if nobs is None:
            h = ref_enkf.SelectionOperator.identity()
            m = nstate
        else:
            idx = np.sort(rng.choice(nstate, size=nobs, replace=False))
            h = ref_enkf.SelectionOperator.from_indices(idx)
            m = nobs
        r = rng.uniform(0.2, 1.0, m)
        y = rng.standard_normal(m) + 8.0
        eps = 0.5 * rng.standard_normal((m, nens))
        obs = ref_enkf.ObservationBatch(y=y, perturbed=y[:, None] + eps, perturbations=eps)
        if kind == "cyclic":
            delta = ref_enkf.influence_matrix_cyclic(nstate, h, scale=scale)
        elif kind == "uniform":
            delta = rng.uniform(0.0, 1.0, (nstate, m))
        else:
            delta = np.ones((nstate, m))
        xa = ref_enkf.analysis_step(x, obs, h, r, "sherman", localization=delta)
        out[f"l{i}_x"] = x
        out[f"l{i}_idx"] = np.array([]) if h.indices is None else h.indices
        out[f"l{i}_identity"] = np.array(h.indices is None)
        out[f"l{i}_r"] = r
        out[f"l{i}_perturbed"] = obs.perturbed
        out[f"l{i}_delta"] = delta
        out[f"l{i}_kind"] = np.array(kind)
        out[f"l{i}_scale"] = np.array(np.nan if scale is None else scale)
        out[f"l{i}_xa"] = xa
    out["ncases"] = np.array(len(cases))
    # influence_matrix_cyclic known answers (test_enkf.py:160-190)
    for tag, (ns, idx, sc) in {"i0": (10, [0, 5], None), "i1": (10, [5], None), "i2": (10, [9], None),
                               "i3": (17, None, None), "i4": (10, [5], 2.0), "i5": (40, None, 8.0)}.items():
        h = ref_enkf.SelectionOperator.identity() if idx is None else ref_enkf.SelectionOperator.from_indices(idx)
        out[f"{tag}_delta"] = ref_enkf.influence_matrix_cyclic(ns, h, scale=sc)
    return out


def lorenz96():
    """Lorenz96.advance (models/lorenz96.py:31-78) on seeded ensembles, the
    DivergenceError member, and a short closed-loop cycle of forecast_step +
    analysis_step (experiment.py:457-479) at a reduced config-2 shape."""
    from enkfkit.enkf import forecast_step, perturb_observations
    from enkfkit.errors import DivergenceError
    out = {}
    rng = make_rng(0xA7)
    # inputs regenerated from the per-case seed (tests/golden_io.l96_input); outputs
    # pinned bitwise by sha256 plus a strided row sample for diagnostics
    cases = [(40, 20, 10), (4096, 8, 5), (7000, 3, 2), (4, 2, 3), (33, 1, 7), (1000, 64, 1)]
    for i, (ns, nens, steps) in enumerate(cases):
        x = 8.0 + make_rng(0xB000 + i).standard_normal((ns, nens))
        model = Lorenz96(Lorenz96Config(nstate=ns, forcing=8.0, dt=0.05))
        xf = model.advance(x, 0.0, steps * 0.05)
        out[f"f{i}_meta"] = np.array([0xB000 + i, ns, nens, steps])
        out[f"f{i}_xf_sha"] = np.array(sha(xf))
        out[f"f{i}_xf_rows"] = xf[::max(1, ns // 64)]
    out["nforecast"] = np.array(len(cases))
    x1 = 8.0 + rng.standard_normal(40)
    out["single_x"], out["single_xf"] = x1, Lorenz96(Lorenz96Config(nstate=40)).advance(x1, 0.0, 0.25)
    # divergence: huge members overflow; the reference names the first bad column
    xd = 8.0 + rng.standard_normal((16, 6))
    xd[:, 4] *= 1e120
    xd[:, 2] *= 1e160
    try:
        Lorenz96(Lorenz96Config(nstate=16)).advance(xd, 0.0, 0.5)
        member = -1
    except DivergenceError as exc:
        member = exc.member
    out["div_x"], out["div_member"] = xd, np.array(member)
    # closed loop: ns=128, N=16, identity H, R = 0.1^2 I, 5 steps per cycle, 8 cycles
    ns, nens, cycles = 128, 16, 8
    model = Lorenz96(Lorenz96Config(nstate=ns))
    truth = model.advance(8.0 + 0.01 * rng.standard_normal(ns), 0.0, 500 * 0.05)
    x = truth[:, None] + rng.standard_normal((ns, nens))
    r = np.full(ns, 0.01)
    h = ref_enkf.SelectionOperator.identity()
    out["cyc_x0"] = x
    ys, mf, ma = [], [], []
    for c in range(cycles):
        truth = model.advance(truth, 0.0, 0.25)
        y = truth + 0.1 * rng.standard_normal(ns)
        ob = perturb_observations(y, r, nens, rng)
        x = forecast_step(model, x, c * 0.25, (c + 1) * 0.25)
        mf.append(x.mean(axis=1))
        x = ref_enkf.analysis_step(x, ob, h, r, "sherman")
        ma.append(x.mean(axis=1))
        ys.append(ob.perturbed)
    out["cyc_r"], out["cyc_ys"] = r, np.stack(ys)
    out["cyc_mean_f"], out["cyc_mean_a"], out["cyc_xa"] = np.stack(mf), np.stack(ma), x
    # inflate (enkf.py:123-135) on seeded ensembles, and the same loop with inflation 1.05
    # (experiment.py:466-467: after the forecast error, before the analysis)
    from enkfkit.enkf import inflate
    for i, (ns_, ne_, a_) in enumerate([(40, 20, 1.05), (256, 16, 1.3), (7, 3, 2.0)]):
        xi = 8.0 + make_rng(0xB100 + i).standard_normal((ns_, ne_))
        out[f"inf{i}_meta"] = np.array([0xB100 + i, ns_, ne_])
        out[f"inf{i}_alpha"] = np.array(a_)
        out[f"inf{i}_out"] = inflate(xi, a_)
    x = out["cyc_x0"].copy()
    mf, ma = [], []
    for c in range(cycles):
        x = forecast_step(model, x, c * 0.25, (c + 1) * 0.25)
        mf.append(x.mean(axis=1))
        x = inflate(x, 1.05)
        ob = ref_enkf.ObservationBatch(y=None, perturbed=out["cyc_ys"][c], perturbations=None)
        x = ref_enkf.analysis_step(x, ob, h, r, "sherman")
        ma.append(x.mean(axis=1))
    out["cycinf_mean_f"], out["cycinf_mean_a"], out["cycinf_xa"] = np.stack(mf), np.stack(ma), x
    # the lorenz-small preset's loop (presets/lorenz-small.ini: ns=40, N=20, R = I, analysis
    # every 2 RK4 steps, inflation 1.05, cyclic localization scale 8), 8 cycles, with the
    # identity H (pobs = 1) and with a stride-2 H
    for tag, idxs in (("lcA", None), ("lcB", np.arange(0, 40, 2))):
        ns, nens, cycles = 40, 20, 8
        model = Lorenz96(Lorenz96Config(nstate=ns))
        rng2 = make_rng(0xC3 if idxs is None else 0xC4)
        truth = model.advance(8.0 + 0.01 * rng2.standard_normal(ns), 0.0, 500 * 0.05)
        x = truth[:, None] + 0.4 * rng2.standard_normal((ns, nens))
        h = ref_enkf.SelectionOperator.identity() if idxs is None else ref_enkf.SelectionOperator.from_indices(idxs)
        nobs = ns if idxs is None else len(idxs)
        r = np.ones(nobs)
        delta = ref_enkf.influence_matrix_cyclic(ns, h, scale=8.0)
        out[f"{tag}_x0"] = x
        out[f"{tag}_idx"] = np.array([], dtype=np.int64) if idxs is None else np.asarray(idxs, dtype=np.int64)
        ys, mf, ma = [], [], []
        for c in range(cycles):
            truth = model.advance(truth, 0.0, 0.1)
            y = h.apply(truth) + rng2.standard_normal(nobs)
            ob = perturb_observations(y, r, nens, rng2)
            x = forecast_step(model, x, c * 0.1, (c + 1) * 0.1)
            mf.append(x.mean(axis=1))
            x = inflate(x, 1.05)
            x = ref_enkf.analysis_step(x, ob, h, r, "sherman", localization=delta)
            ma.append(x.mean(axis=1))
            ys.append(ob.perturbed)
        out[f"{tag}_r"], out[f"{tag}_ys"] = r, np.stack(ys)
        out[f"{tag}_mean_f"], out[f"{tag}_mean_a"], out[f"{tag}_xa"] = np.stack(mf), np.stack(ma), x
    return out


if __name__ == "__main__":
    for name, fn in (("lorenz96", lorenz96), ("localized", localized), ("ism_systems", ism_systems), ("analysis_small", analysis_small),
                     ("configs", config_fixtures), ("selection", selections)):
        if len(sys.argv) > 1 and name not in sys.argv[1:]:
            continue  # e.g. `make_golden.py localized` regenerates one fixture
        data = fn()
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **data)
        print(name, os.path.getsize(path) // 1024, "KiB")
    print("reference", enkfkit.__version__)
