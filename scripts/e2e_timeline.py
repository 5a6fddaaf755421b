import os, sys
sys.path.insert(0, "/root/repo")
import torch, numpy as np
import paper_2202_09056_b200 as pb
p = pb.generate_hex(nx=63, ny=63, nz=63, dirichlet="eliminate", noise=0.01, seed=2022)
A = pb.Bsr3.from_host(p.nbrows, p.nbrows, p.ptr, p.col, p.val.reshape(-1))
n, P, K = p.n, 4, 40
xh = torch.empty((K, n), dtype=torch.float64).pin_memory(); yh = torch.empty((K, n), dtype=torch.float64).pin_memory()
bx = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(P)]
by = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(P)]
sh, sk, sd = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
for rep in range(2):
    E = lambda: torch.cuda.Event(enable_timing=True)
    t = [[E() for _ in range(6)] for _ in range(K)]
    ev_h = [torch.cuda.Event() for _ in range(P)]; ev_k = [torch.cuda.Event() for _ in range(P)]; ev_d = [torch.cuda.Event() for _ in range(P)]
    torch.cuda.synchronize()
    e0 = E(); e0.record()
    for s_ in (sh, sk, sd): s_.wait_event(e0)
    for k in range(K):
        b = k % P
        if k >= P: sh.wait_event(ev_k[b])
        t[k][0].record(sh)
        with torch.cuda.stream(sh): bx[b].copy_(xh[k], non_blocking=True)
        t[k][1].record(sh); ev_h[b].record(sh)
        sk.wait_event(ev_h[b])
        if k >= P: sk.wait_event(ev_d[b])
        t[k][2].record(sk)
        A.spmv_device(bx[b].data_ptr(), by[b].data_ptr(), stream=sk.cuda_stream)
        t[k][3].record(sk); ev_k[b].record(sk)
        sd.wait_event(ev_k[b])
        t[k][4].record(sd)
        with torch.cuda.stream(sd): yh[k].copy_(by[b], non_blocking=True)
        t[k][5].record(sd); ev_d[b].record(sd)
    torch.cuda.synchronize()
for k in range(10, 20):
    print(k, " ".join("%8.1f" % (e0.elapsed_time(x) * 1e3) for x in t[k]),
          " h2d %.1f ker %.1f d2h %.1f" % ((t[k][0].elapsed_time(t[k][1]))*1e3, t[k][2].elapsed_time(t[k][3])*1e3, t[k][4].elapsed_time(t[k][5])*1e3))
