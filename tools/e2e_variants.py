"""e2e (host buffers) throughput of several library builds. usage: python tools/e2e_variants.py CFG N CHUNK lib.so ..."""
import ctypes
import os
import sys

# chunked (staged) transport: pinned buffers would otherwise take the zero-copy one
os.environ["BLK_HOST_PIPELINE"] = "1"

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import workloads  # noqa: E402

cfg, n, ch = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
v, x = workloads.generate(cfg, 0, n)
hv, hx = torch.from_numpy(v).pin_memory(), torch.from_numpy(x).pin_memory()
ho = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(3)]
vp = ctypes.c_void_p
for path in sys.argv[4:]:
    L = ctypes.CDLL(os.path.abspath(path))
    L.bessel_logk_host_workspace_bytes.restype = ctypes.c_size_t
    L.bessel_logk_host_workspace_bytes.argtypes = [ctypes.c_size_t, ctypes.c_size_t]
    f = L.bessel_logk_f64_host
    f.restype = ctypes.c_int
    f.argtypes = [vp, vp, ctypes.c_size_t, vp, vp, vp, ctypes.c_int, vp, ctypes.c_size_t, ctypes.c_size_t, vp]
    wsb = L.bessel_logk_host_workspace_bytes(ch, 8)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    args = [vp(hv.data_ptr()), vp(hx.data_ptr()), n] + [vp(t.data_ptr()) for t in ho] + \
           [128, vp(ws.data_ptr()), wsb, ch, vp(st.cuda_stream)]
    for _ in range(3):
        assert f(*args) == 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(10):
        f(*args)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{os.path.basename(path):10s} {cfg} n={n} chunk={ch} {ms:.3f} ms/step {n / ms * 1e3:.3e} evals/s", flush=True)
