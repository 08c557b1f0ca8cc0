"""PCIe copy-engine probe: H2D alone, D2H alone, both at once on two streams (pinned)."""
import time
import torch

MB = 1 << 20
n_in, n_out = 50 * MB, 96 * MB
h_in = torch.empty(n_in, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(n_out, dtype=torch.uint8, pin_memory=True)
d_in = torch.empty(n_in, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n_out, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(f, reps=10):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d(); d2h()


a, b, c = t(h2d), t(d2h), t(both)
print(f"H2D {n_in/MB:.0f} MB {a:.3f} ms ({n_in/a/1e6:.1f} GB/s); D2H {n_out/MB:.0f} MB {b:.3f} ms ({n_out/b/1e6:.1f} GB/s); "
      f"both {c:.3f} ms (serial would be {a+b:.3f})")
print(torch.cuda.get_device_properties(0))
