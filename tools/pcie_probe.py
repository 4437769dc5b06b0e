"""PCIe probe (diagnostics): pinned H2D / D2H copy rates alone and together,
for the e2e leg's bound (bench.py e2e)."""
import torch

n_h2d = 1258389504  # configs[2] depth maps per step (4096 x 240 x 320 x 4 B)
n_d2h = 945913856
h = torch.empty(n_h2d, dtype=torch.uint8).pin_memory()
ho = torch.empty(n_d2h, dtype=torch.uint8).pin_memory()
d = torch.empty(n_h2d, dtype=torch.uint8, device="cuda")
do = torch.empty(n_d2h, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    for s in (s1, s2):
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        ho.copy_(do, non_blocking=True)


def both():
    h2d()
    d2h()


for name, fn, nb in (("h2d", h2d, n_h2d), ("d2h", d2h, n_d2h)):
    ms = timed(fn)
    print(f"{name}: {nb / ms / 1e6:.1f} GB/s ({ms:.2f} ms)")
ms = timed(both)
print(f"h2d+d2h concurrent: {ms:.2f} ms per step -> h2d {n_h2d / ms / 1e6:.1f} GB/s, d2h {n_d2h / ms / 1e6:.1f} GB/s; "
      f"e2e bound {4096 / ms * 1e3:.0f} frames/s")
