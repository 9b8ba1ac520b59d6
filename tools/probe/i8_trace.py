"""Per-tile event trace of anomaly_i8_kernel (CTA 0), ENKF_I8_DBG=8."""
import ctypes, os, subprocess, sys
import numpy as np, torch
if os.environ.get("ENKF_LIB_VARIANT", "") == "":
    # the event stamps are compiled in only with -DI8_TRACE_ON (variant "trace")
    subprocess.run([sys.executable, "tools/build_variant.py", "trace", "-DI8_TRACE_ON=1", "-DI8_DBG_BUILD"], check=True,
                   stdout=subprocess.DEVNULL)
    os.environ["ENKF_LIB_VARIANT"] = "trace"
os.environ["ENKF_I8_DBG"] = str(8 | int(sys.argv[1] if len(sys.argv) > 1 else 0))
sys.path.insert(0, '.')
from paper_1302_3876_b200 import _native
dev = torch.device('cuda', 0)
lib = _native.lib()
n, ns = 128, (1 << 22)
x = torch.randn((ns, n), dtype=torch.float64, device=dev)
t = torch.eye(n, dtype=torch.float64, device=dev) + 0.01 * torch.randn((n, n), dtype=torch.float64, device=dev)
out = torch.empty_like(x)
plan = _native.Plan(ns, 1, n, 0)
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    lib.enkf_anomaly_update_f64(plan.handle, x.data_ptr(), t.data_ptr(), out.data_ptr(), ns, s)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
lib.enkf_anomaly_update_f64(plan.handle, x.data_ptr(), t.data_ptr(), out.data_ptr(), ns, s)
e1.record(); torch.cuda.synchronize()
print("dbg", os.environ["ENKF_I8_DBG"], "kernel ms (2^22 rows)", e0.elapsed_time(e1))
buf = (ctypes.c_ulonglong * (256 * 16))()
fn = lib.enkf_debug_i8_trace
fn.argtypes = [ctypes.c_void_p]
assert fn(ctypes.addressof(buf)) == 0
tr = np.array(buf, dtype=np.float64).reshape(256, 16)
t0 = tr[0, 0]
tr = (tr - t0) / 1000.0  # us
names = ["tma_issue", "landed", "slice_done", "mma_start", "mma_end", "epi_ready", "epi_done", "xempty_ok"]
print("tile " + " ".join(f"{n:>10s}" for n in names))
for i in (list(range(0, 12)) + list(range(100, 108))) if len(sys.argv) > 2 else []:
    print(f"{i:4d} " + " ".join(f"{v:10.2f}" for v in tr[i]))
d = np.diff(tr[20:200, 6])
print("steady epi_done interval us: mean", d.mean(), "tiles/us", 1 / d.mean())
for a, b, lab in [(0, 1, "tma latency"), (1, 2, "land->slice done"), (2, 3, "slice->mma start"), (3, 4, "mma issue"), (4, 5, "mma end->epi ready"), (5, 6, "epi duration"), (1, 7, "land->xempty ok")]:
    v = tr[20:200, b] - tr[20:200, a]
    print(f"{lab:22s} mean {v.mean():7.2f} us  median {np.median(v):7.2f}")

print("per chunk (us, relative to tile's tma issue):  mma0_start mma0_commit mma1_start mma1_commit | epi0_ready epi0_end epi1_ready epi1_end")
for i in range(100, 110):
    b = tr[i, 0]
    print(f"{i:4d} " + " ".join(f"{tr[i, k] - b:7.2f}" for k in (8, 9, 10, 11)) + " | " + " ".join(f"{tr[i, k] - b:7.2f}" for k in (12, 14, 13, 15)))
