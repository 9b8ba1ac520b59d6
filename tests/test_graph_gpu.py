"""CUDA-graph capture of the device-resident step (`enkf_analysis_async_f64`, the
header's "graph-capturable" claim): the status reset, Gram pass, levels and
anomaly update of one plan captured once on a side stream and replayed on new
input contents give the same X^A, bit for bit, as the direct call — on the
single-CTA path (config 1), the FP64 DMMA path (configs 2, 3) and the int8
tensor-core path (N = 128).  A replay with a non-finite observation reports
the same ValueError status through `enkf_plan_sync_status`.
"""

import ctypes

import numpy as np
import pytest

from golden_io import make_rng
from paper_1302_3876_b200 import _native

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_1302_3876_b200.build import build
    build()
    import torch
    assert torch.cuda.is_available()


def _inputs(rng, ns, nobs, n, identity):
    x = rng.standard_normal((ns, n)) * rng.uniform(0.5, 2.0, (ns, 1)) + rng.standard_normal((ns, 1))
    idx = None if identity else np.sort(rng.choice(ns, size=nobs, replace=False)).astype(np.int64)
    hx = x if identity else x[idx]
    y = hx.mean(axis=1)[:, None] + rng.standard_normal((nobs, n))
    r = rng.uniform(0.25, 1.0, nobs)
    return x, y, idx, r


@pytest.mark.parametrize("ns,nobs,n,identity", [(40, 20, 20, False), (4096, 4096, 64, True),
                                                (16641, 1089, 96, False), (1 << 16, 1 << 13, 128, False)])
def test_graph_replay_equals_direct_call(ns, nobs, n, identity):
    import torch
    dev = torch.device("cuda", 0)
    lib = _native.lib()
    rng = make_rng(ns + n)
    a = _inputs(rng, ns, nobs, n, identity)
    b = _inputs(rng, ns, nobs, n, identity)
    if not identity:
        b = (b[0], b[1], a[2], b[3])  # same H: the index buffer is part of the captured graph
    xd, yd, rd = (torch.from_numpy(v).to(dev) for v in (a[0], a[1], a[3]))
    idd = None if identity else torch.from_numpy(a[2]).to(dev)
    ip = 0 if idd is None else idd.data_ptr()
    out = torch.empty_like(xd)
    plan = _native.Plan(ns, nobs, n, 0)
    side = torch.cuda.Stream(dev)
    st = _native.EnkfStatus()

    # warm-up call on the side stream: lazily allocated workspace exists before capture
    with torch.cuda.stream(side):
        assert lib.enkf_analysis_async_f64(plan.handle, xd.data_ptr(), yd.data_ptr(), ip, rd.data_ptr(),
                                           out.data_ptr(), side.cuda_stream) == 0
        assert lib.enkf_plan_sync_status(plan.handle, side.cuda_stream, ctypes.byref(st)) == 0, st.message
    torch.cuda.synchronize(dev)

    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=side):
        cs = torch.cuda.current_stream(dev).cuda_stream
        assert lib.enkf_analysis_async_f64(plan.handle, xd.data_ptr(), yd.data_ptr(), ip, rd.data_ptr(),
                                           out.data_ptr(), cs) == 0

    def direct(x, y, r):
        ref = torch.empty_like(xd)
        s2 = _native.EnkfStatus()
        rc = lib.enkf_analysis_f64(plan.handle, x.data_ptr(), y.data_ptr(), ip, r.data_ptr(), ref.data_ptr(),
                                   torch.cuda.current_stream(dev).cuda_stream, ctypes.byref(s2))
        assert rc == 0, s2.message
        return ref.cpu()

    for xs, ys, rs in ((a[0], a[1], a[3]), (b[0], b[1], b[3]), (a[0], a[1], a[3])):
        xd.copy_(torch.from_numpy(xs))
        yd.copy_(torch.from_numpy(ys))
        rd.copy_(torch.from_numpy(rs))
        graph.replay()
        torch.cuda.synchronize(dev)
        assert lib.enkf_plan_sync_status(plan.handle, torch.cuda.current_stream(dev).cuda_stream,
                                         ctypes.byref(st)) == 0, st.message
        got = out.cpu()
        ref = direct(xd, yd, rd)
        assert torch.equal(got, ref)

    # a non-finite observation: the captured status reset + device flags report it on replay
    bad = b[1].copy()
    bad[nobs // 2, 1] = np.nan
    yd.copy_(torch.from_numpy(bad))
    graph.replay()
    torch.cuda.synchronize(dev)
    rc = lib.enkf_plan_sync_status(plan.handle, torch.cuda.current_stream(dev).cuda_stream, ctypes.byref(st))
    assert rc == 1  # ENKF_INVALID_ARGUMENT -> ValueError
    # and a clean replay afterwards is clean again
    yd.copy_(torch.from_numpy(b[1]))
    graph.replay()
    torch.cuda.synchronize(dev)
    assert lib.enkf_plan_sync_status(plan.handle, torch.cuda.current_stream(dev).cuda_stream,
                                     ctypes.byref(st)) == 0, st.message
    del graph
