"""Memory-safety checks of every entry point without compute-sanitizer (the
tool is closed on the GPU pool: profiles/r02i_compute_sanitizer_refused.log).

Every device array is a window into a larger buffer whose guard regions
before and after hold a sentinel bit pattern; after the call the guards
must be unchanged (no out-of-bounds or stray write), the inputs must be
unchanged (no write to them), and every output element must have been
written (no element skipped: the windows are prefilled with a tiny positive
value no result can take).  Sizes cover single elements, partial warps, ragged
blocks and empty lanes; the same results must come out of every block size
(the exp-table copy and its barrier)."""
import numpy as np
import pytest
import torch

import paper_2108_11560_b200 as blk
import workloads

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")
GUARD = 4099
# guard sentinel and window prefill: values no output can take
SENT = {torch.float64: -2.718281828459045e300, torch.float32: -3.1e38}
FILL = {torch.float64: 1.2345e-300, torch.float32: 1.2345e-37}


class Guarded:
    """n elements inside [GUARD | n | GUARD] of a device (or pinned host) buffer."""

    def __init__(self, n, dtype, data=None, pinned=False, device=DEV):
        self.n = n
        self.dtype = dtype
        buf = torch.full((n + 2 * GUARD,), SENT[dtype], dtype=dtype)
        if pinned:
            buf = buf.pin_memory()
        elif device is not None:
            buf = buf.to(device)
        self.buf = buf
        self.t = buf[GUARD:GUARD + n]
        if data is not None:
            self.t.copy_(torch.as_tensor(data, dtype=dtype))
        else:
            self.t.fill_(FILL[dtype])

    def guards_ok(self):
        b = self.buf.cpu()
        s = torch.tensor(SENT[self.dtype], dtype=b.dtype)
        return bool((b[:GUARD] == s).all()) and bool((b[GUARD + self.n:] == s).all())

    def all_written(self):
        t = self.t.cpu()
        return not bool((t == torch.tensor(FILL[self.dtype], dtype=t.dtype)).any())


def _inputs(cfg, n, dtype):
    v, x = workloads.generate(cfg, 7, n)
    v = v.astype(np.float64)
    x = x.astype(np.float64)
    if n >= 8:   # special values, negative orders, invalid arguments
        v[:4] = [-3.5, 0.0, np.nan, 2.0]
        x[:4] = [1.0, 0.5, 1.0, -1.0]
    return v.astype(dtype), x.astype(dtype)


@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("n", [1, 31, 33, 127, 129, 1037])
@pytest.mark.parametrize("lanes,nbins", [(1, 128), (2, 16), (8, 2), (32, 3), (32, 128), (0, 64)])
def test_guards_logk(prec, n, lanes, nbins):
    dt = torch.float64 if prec == 64 else torch.float32
    v, x = _inputs("c1" if prec == 64 else "c4", n, np.float64 if prec == 64 else np.float32)
    gv, gx = Guarded(n, dt, data=v), Guarded(n, dt, data=x)
    outs = [Guarded(n, dt) for _ in range(3)]
    f = blk.bessel_logk_f64 if prec == 64 else blk.bessel_logk_f32
    f(gv.t, gx.t, *[o.t for o in outs], nbins=nbins, lanes_per_element=lanes)
    torch.cuda.synchronize()
    for g in (gv, gx, *outs):
        assert g.guards_ok()
    assert np.array_equal(gv.t.cpu().numpy(), v, equal_nan=True)
    assert np.array_equal(gx.t.cpu().numpy(), x, equal_nan=True)
    for o in outs:
        assert o.all_written()
    # one output only: the others untouched
    only = [Guarded(n, dt) for _ in range(3)]
    f(gv.t, gx.t, None, only[1].t, None, nbins=nbins, lanes_per_element=lanes)
    torch.cuda.synchronize()
    assert only[1].all_written() and torch.equal(only[1].t.nan_to_num(7.0), outs[1].t.nan_to_num(7.0))
    for o in (only[0], only[2]):
        assert o.guards_ok() and bool((o.t.cpu() == FILL[dt]).all())


@pytest.mark.parametrize("threads", [32, 64, 96, 128])
def test_block_sizes_bitwise(threads):
    """The table copy (strided by blockDim) and its barrier: every block size
    gives the same bits, including a ragged last block."""
    v, x = _inputs("c3", 5000 + 17, np.float64)
    vt, xt = torch.from_numpy(v).to(DEV), torch.from_numpy(x).to(DEV)
    ref = blk.log_bessel_k(vt, xt, lanes_per_element=1)
    got = blk.log_bessel_k(vt, xt, lanes_per_element=1, block_threads=threads)
    for a, b in zip(ref, got):
        assert torch.equal(a.nan_to_num(7.0), b.nan_to_num(7.0))


@pytest.mark.parametrize("n", [1, 33, 1037])
def test_guards_hess_plan_nig(n):
    v, x = _inputs("c2", n, np.float64)
    gv, gx = Guarded(n, torch.float64, data=v), Guarded(n, torch.float64, data=x)
    for lanes in (1, 8):
        outs = [Guarded(n, torch.float64) for _ in range(6)]
        o = blk._Options(lanes, 0, 0, 0)
        import ctypes
        st = blk.lib().bessel_logk_hess_f64(
            ctypes.c_void_p(gv.t.data_ptr()), ctypes.c_void_p(gx.t.data_ptr()), n,
            *[ctypes.c_void_p(g.t.data_ptr()) for g in outs], 128, ctypes.byref(o),
            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        assert st == blk.BLK_OK
        torch.cuda.synchronize()
        for g in outs:
            assert g.guards_ok() and g.all_written()
    import ctypes
    plan = [Guarded(n, torch.float64) for _ in range(4)]
    st = blk.lib().bessel_logk_plan_f64(
        ctypes.c_void_p(gv.t.data_ptr()), ctypes.c_void_p(gx.t.data_ptr()), n,
        *[ctypes.c_void_p(g.t.data_ptr()) for g in plan], 16, None,
        ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert st == blk.BLK_OK
    torch.cuda.synchronize()
    for g in plan:
        assert g.guards_ok() and g.all_written()
    for g in (gv, gx):
        assert g.guards_ok()
    # NIG: 5 outputs, a workspace of exactly the required size inside guards
    y = Guarded(n, torch.float64, data=np.random.default_rng(n).normal(0, 3, n))
    out = Guarded(5, torch.float64)
    wsb = blk.lib().bessel_nig_workspace_bytes(n)
    ws = Guarded(wsb // 8, torch.float64)
    blk.nig_loglik(y.t, 2.0, 0.5, 1.5, 0.3, out=out.t, workspace=ws.t.view(torch.uint8))
    torch.cuda.synchronize()
    for g in (y, out, ws):
        assert g.guards_ok()
    assert out.all_written()


@pytest.mark.parametrize("n,chunk", [(1, 0), (1037, 256), (70001, 16384)])
def test_guards_host_paths(n, chunk):
    """Zero-copy (pinned) and staged (pageable, chunked) host transports write
    exactly the n host outputs; the staged path's device workspace of exactly
    the required size is not overrun."""
    v, x = _inputs("c2", n, np.float64)
    ref = blk.log_bessel_k(torch.from_numpy(v).to(DEV), torch.from_numpy(x).to(DEV),
                           lanes_per_element=1)
    ref = [r.cpu() for r in ref]
    # zero-copy
    hv, hx = Guarded(n, torch.float64, data=v, pinned=True), Guarded(n, torch.float64, data=x, pinned=True)
    ho = [Guarded(n, torch.float64, pinned=True) for _ in range(3)]
    blk.bessel_logk_f64_host(hv.t, hx.t, *[g.t for g in ho], nbins=128)
    for g, r in zip(ho, ref):
        assert g.guards_ok() and g.all_written() and torch.equal(g.t.nan_to_num(7.0), r.nan_to_num(7.0))
    # staged
    pv, px = Guarded(n, torch.float64, data=v, device=None), Guarded(n, torch.float64, data=x, device=None)
    po = [Guarded(n, torch.float64, device=None) for _ in range(3)]
    wsb = blk.host_workspace_bytes(chunk)
    ws = Guarded(wsb // 8, torch.float64)
    blk.bessel_logk_f64_host(pv.t, px.t, *[g.t for g in po], nbins=128,
                             workspace=ws.t.view(torch.uint8), chunk=chunk)
    assert ws.guards_ok()
    for g, r in zip(po, ref):
        assert g.guards_ok() and g.all_written() and torch.equal(g.t.nan_to_num(7.0), r.nan_to_num(7.0))
