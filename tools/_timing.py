"""Device-side timing of one enqueue of `fn` with CUDA events on the current stream.
Before the start event a ~50 us spin kernel keeps the GPU busy while Python
enqueues the event and the launch, so the measured interval is the kernel
(plus the event granularity), not the host launch overhead."""
import torch


def device_time(fn, reps=10, warm=3, spin_cycles=100_000):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.cuda._sleep(spin_cycles)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]
