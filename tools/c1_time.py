import sys, os, ctypes, torch, numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, 'tools')
from _timing import device_time
import workloads
v, x = workloads.generate("c1", 0, 10000)
dev = torch.device("cuda"); vt, xt = torch.from_numpy(v).to(dev), torch.from_numpy(x).to(dev)
o = [torch.empty_like(vt) for _ in range(3)]
vp = ctypes.c_void_p
for path in sys.argv[1:]:
    L = ctypes.CDLL(os.path.abspath(path)); f = L.bessel_logk_f64
    f.argtypes = [vp, vp, ctypes.c_size_t, vp, vp, vp, ctypes.c_int, vp]
    P = [vp(t.data_ptr()) for t in (vt, xt, *o)]; s = vp(torch.cuda.current_stream().cuda_stream)
    ms = device_time(lambda: f(P[0], P[1], 10000, P[2], P[3], P[4], 128, s), reps=50)
    print(path, f"c1 {ms*1e3:.1f} us")
