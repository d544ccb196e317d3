"""PCIe floor of the e2e step: H2D of the inputs and D2H of the outputs of one c2
batch (2^20 FP64: 16 MiB in, 24 MiB out), alone and concurrently on two streams."""
import torch

n = 1 << 20
hin = torch.empty(2 * n, dtype=torch.float64).pin_memory()
hout = torch.empty(3 * n, dtype=torch.float64).pin_memory()
din = torch.empty(2 * n, dtype=torch.float64, device="cuda")
dout = torch.empty(3 * n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d():
    din.copy_(hin, non_blocking=True)


def d2h():
    hout.copy_(dout, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        din.copy_(hin, non_blocking=True)
    with torch.cuda.stream(s2):
        hout.copy_(dout, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
print(f"H2D 16 MiB {t1:.3f} ms ({16.777216 / t1:.1f} GB/s); D2H 24 MiB {t2:.3f} ms "
      f"({25.165824 / t2:.1f} GB/s); both concurrently {t3:.3f} ms")
