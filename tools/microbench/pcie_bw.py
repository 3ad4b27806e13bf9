"""Host<->device copy bandwidth from pinned memory on the GPU box: one stream vs two streams,
chunk sizes, and H2D concurrent with D2H (the e2e path's link budget)."""
import torch

dev = torch.device("cuda", 0)
N = 268435456 // 16  # c1 tensor: 268 MB of complex128
h = torch.empty(N * 2, dtype=torch.float64).pin_memory()
h2 = torch.empty(N * 2, dtype=torch.float64).pin_memory()
d = torch.empty(N * 2, dtype=torch.float64, device=dev)
d2 = torch.empty(N * 2, dtype=torch.float64, device=dev)
bytes_ = h.numel() * 8
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def chunked(dst, src, k, streams):
    n = src.numel() // k
    for i in range(k):
        with torch.cuda.stream(streams[i % len(streams)]):
            dst[i * n:(i + 1) * n].copy_(src[i * n:(i + 1) * n], non_blocking=True)
    for s in streams:
        torch.cuda.current_stream().wait_stream(s)


for k in (1, 8, 32):
    for ns in (1, 2):
        ms = timed(lambda: chunked(d, h, k, [s1, s2][:ns]))
        print(f"H2D chunks {k:3d} streams {ns}: {bytes_ / ms / 1e6:7.1f} GB/s")
        ms = timed(lambda: chunked(h, d, k, [s1, s2][:ns]))
        print(f"D2H chunks {k:3d} streams {ns}: {bytes_ / ms / 1e6:7.1f} GB/s")


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


ms = timed(both)
print(f"H2D + D2H concurrent: {2 * bytes_ / ms / 1e6:7.1f} GB/s total")
