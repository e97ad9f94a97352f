"""PCIe bandwidth of pinned host <-> device copies: H2D alone, D2H alone, both at once
(two streams), 1 GiB each way, CUDA events.  Context for the streamed e2e step."""
import torch

N = 2 ** 27          # doubles = 1 GiB
h_in = torch.empty(N, dtype=torch.float64).pin_memory()
h_out = torch.empty(N, dtype=torch.float64).pin_memory()
d_a = torch.empty(N, dtype=torch.float64, device="cuda")
d_b = torch.ones(N, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    for s in (s1, s2):
        torch.cuda.current_stream().wait_stream(s)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


def h2d():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


def both():
    h2d()
    d2h()


for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    fn()
    ms = min(timed(fn) for _ in range(3))
    gb = 8 * N / 1e9 * (2 if name == "both" else 1)
    print(f"{name}: {ms:.2f} ms, {gb / ms * 1e3:.1f} GB/s total")
