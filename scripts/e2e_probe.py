"""e2e SpMV pipeline probe (C1): copies only, kernel only, and the full
H2D -> SpMV -> D2H pipeline over per-engine streams, CUDA-event timed."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2202_09056_b200 as pb  # noqa: E402

p = pb.generate_hex(nx=63, ny=63, nz=63, dirichlet="eliminate", noise=0.01, seed=2022)
A = pb.Bsr3.from_host(p.nbrows, p.nbrows, p.ptr, p.col, p.val.reshape(-1))
n, P, K = p.n, 4, 100
xh = torch.empty((K, n), dtype=torch.float64).pin_memory()
yh = torch.empty((K, n), dtype=torch.float64).pin_memory()
xh.uniform_(-1, 1)
bx = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(P)]
by = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(P)]
sh, sk, sd = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
nbytes = A.spmv_bytes()


def run(h2d, kern, d2h):
    ev_h = [torch.cuda.Event() for _ in range(P)]
    ev_k = [torch.cuda.Event() for _ in range(P)]
    ev_d = [torch.cuda.Event() for _ in range(P)]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in (sh, sk, sd):
        s.wait_event(e0)
    for k in range(K):
        b = k % P
        if h2d:
            if k >= P:
                sh.wait_event(ev_k[b])
            with torch.cuda.stream(sh):
                bx[b].copy_(xh[k], non_blocking=True)
            ev_h[b].record(sh)
            sk.wait_event(ev_h[b])
        if k >= P:
            sk.wait_event(ev_d[b])
        if kern:
            A.spmv_device(bx[b].data_ptr(), by[b].data_ptr(), stream=sk.cuda_stream)
        ev_k[b].record(sk)
        if d2h:
            sd.wait_event(ev_k[b])
            with torch.cuda.stream(sd):
                yh[k].copy_(by[b], non_blocking=True)
        ev_d[b].record(sd)
    for s in (sh, sk, sd):
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / K


for name, cfg in [("h2d+d2h", (1, 0, 1)), ("full", (1, 1, 1))]:
    run(*cfg)
    t = min(run(*cfg) for _ in range(3))
    print(f"{name:12s}: {t * 1e6:7.1f} us/step  ({nbytes / t / 1e9:7.1f} GB/s-eq)", flush=True)

# variants of the full pipeline
def run2(P2, ahead, d2h_on_k):
    ev_h = [torch.cuda.Event() for _ in range(P2)]
    ev_k = [torch.cuda.Event() for _ in range(P2)]
    ev_d = [torch.cuda.Event() for _ in range(P2)]
    bx2 = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(P2)]
    by2 = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(P2)]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s_ in (sh, sk, sd):
        s_.wait_event(e0)
    def issue_h(k):
        b = k % P2
        if k >= P2:
            sh.wait_event(ev_k[b])
        with torch.cuda.stream(sh):
            bx2[b].copy_(xh[k], non_blocking=True)
        ev_h[b].record(sh)
    for k in range(min(ahead, K)):
        issue_h(k)
    for k in range(K):
        b = k % P2
        if k + ahead < K and ahead > 0:
            issue_h(k + ahead)
        elif ahead == 0:
            issue_h(k)
        sk.wait_event(ev_h[b])
        if k >= P2 and not d2h_on_k:
            sk.wait_event(ev_d[b])
        A.spmv_device(bx2[b].data_ptr(), by2[b].data_ptr(), stream=sk.cuda_stream)
        ev_k[b].record(sk)
        if d2h_on_k:
            with torch.cuda.stream(sk):
                yh[k].copy_(by2[b], non_blocking=True)
        else:
            sd.wait_event(ev_k[b])
            with torch.cuda.stream(sd):
                yh[k].copy_(by2[b], non_blocking=True)
            ev_d[b].record(sd)
    for s_ in (sh, sk, sd):
        torch.cuda.current_stream().wait_stream(s_)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / K

for P2, ahead, dk in [(4, 0, False), (4, 2, False), (8, 4, False), (4, 0, True), (4, 2, True), (8, 6, True)]:
    run2(P2, ahead, dk)
    t = min(run2(P2, ahead, dk) for _ in range(3))
    print(f"P={P2} ahead={ahead} d2h_on_kernel_stream={dk}: {t * 1e6:7.1f} us/step ({nbytes / t / 1e9:7.1f} GB/s-eq)", flush=True)
