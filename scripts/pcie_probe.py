"""PCIe probe for the e2e SpMV: pinned H2D, D2H and both at once (separate
streams), at the C1 vector size (6.19 MB) and at 64 MB, CUDA-event timed."""
import torch

for nbytes in (6193152, 64 << 20):
    n = nbytes // 8
    hs = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(2)]
    ds = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(2)]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    reps = 50

    def run(mode):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            if mode in ("h2d", "both"):
                with torch.cuda.stream(s1):
                    ds[0].copy_(hs[0], non_blocking=True)
            if mode in ("d2h", "both"):
                with torch.cuda.stream(s2):
                    hs[1].copy_(ds[1], non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 1e3 / reps

    for mode in ("h2d", "d2h", "both"):
        run(mode)
        t = run(mode)
        print(f"{nbytes / 1e6:7.2f} MB {mode:5s}: {t * 1e6:8.1f} us per rep, "
              f"{nbytes / t / 1e9:6.1f} GB/s per direction")

# H2D of the C1 vector split into k pieces on k streams
nbytes = 6193152
n = nbytes // 8
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
streams = [torch.cuda.Stream() for _ in range(8)]
for k in (1, 2, 4, 8):
    for rep in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            for i in range(k):
                a, b = i * n // k, (i + 1) * n // k
                streams[i].wait_event(e0) if False else None
                with torch.cuda.stream(streams[i]):
                    d[a:b].copy_(h[a:b], non_blocking=True)
        for i in range(k):
            torch.cuda.current_stream().wait_stream(streams[i])
        e1.record()
        torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / 50
    print(f"H2D 6.19 MB in {k} pieces: {t * 1e6:7.1f} us, {nbytes / t / 1e9:5.1f} GB/s")
