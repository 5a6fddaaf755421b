"""bench.py -- B200 SA-AMG NS-Block hot path benchmark (one JSON line).

Metric (BASELINE.json): "BSR SpMV HBM GB/s (% roofline); AMG setup+solve
seconds at 1/2/4/8 B200".  ``value`` is the 3x3-BSR SpMV throughput in
algorithmic GB/s on the C1 fine matrix (64^3-node cube, free-DOF form,
774,144 unknowns, 6,750,700 blocks = 527 MB > 126 MB L2, so no L2 flush is
needed); one step = one y = A x over the whole matrix, inputs resident in
HBM, timed with CUDA events on the launching stream.  ``amg`` carries the
full ns_block setup + SPAI0-preconditioned CG solve seconds on the same
problem.  ``e2e`` is the SpMV through the C-ABI with host vectors (H2D of x
and D2H of y inside the timed region).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

For N>1 (torchrun, one rank per GPU) every rank runs the same per-GPU
workload (replicas, weak scaling); the timed region is bracketed by a
barrier + synchronize and the max over ranks is reported.
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BSR SpMV HBM GB/s (% roofline); AMG setup+solve seconds at 1/2/4/8 B200"
C1 = dict(nx=63, ny=63, nz=63, dirichlet="eliminate", noise=0.01, seed=2022)
WORKLOAD = ("C1: 64x64x64-node unit cube, trilinear hex8 elasticity (E=1, nu=0.3), x=0 face "
            "clamped (free-DOF form: 774,144 unknowns), body force -z + U[-0.01,0.01] noise, "
            "3x3 BSR fp64; SA-AMG ns_block + SPAI0, CG rtol 1e-8")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--amg-repeats", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c4", action="store_true", help="skip the C4 setup+solve leg")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--force-dist", action="store_true",
                    help="use the row-partitioned (NCCL halo) path even on one GPU")
    return ap.parse_args()


_OUT_FD = None


def emit(line):
    """The one JSON line, on the real stdout (fd 1 is pointed at stderr for
    the rest of the run, so library log lines such as NCCL's version banner
    cannot land on stdout)."""
    data = (json.dumps(line) + "\n").encode()
    if _OUT_FD is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        os.write(_OUT_FD, data)


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# Read-only HBM stream on a round-2 B200 (scripts/micro/read_bw.cu, best of
# 10 over 4 GiB, profiles/r02_read_bw.txt): the SpMV moves ~99 % reads,
# while MEASURED_PEAKS' copy figure is half reads and half writes (a copy
# measured 6141 GB/s on the same box), so a read stream can exceed it.
READ_PEAK_GBS = 7199.0


def read_peak_fields(achieved):
    return {"peak_read_only": READ_PEAK_GBS, "frac_read_only": achieved / READ_PEAK_GBS,
            "peak_read_only_source": "16-byte grid-stride loads over 4 GiB, scripts/micro/read_bw.cu "
                                     "(profiles/r02_read_bw.txt)"}


def dist_init(args):
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    dist = None
    if world > 1 or args.force_dist:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl" if args.impl == "b200" else "gloo", rank=rank,
                                world_size=world)
    return rank, world, local, dist


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    def __init__(self, device):
        self.samples, self.reasons = [], set()
        self.stop_ev = threading.Event()
        self.ok = False
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(device)
            self.max = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max = None

    NAMES = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
             0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
             0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
             0x100: "display_clock_setting"}

    def _run(self):
        nv = self.nv
        while not self.stop_ev.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.NAMES.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self.stop_ev.set()
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def ncu_traffic():
    """dram bytes per launch of the SpMV kernel from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "r02_ncu_full_spmv_tma_c1.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f).get("dram_bytes_per_launch")
    return None


def make_problem(pb):
    return pb.generate_hex(**C1)


def config_dict(p, world):
    """The `config` object, identical in both arms (same workload, same sizes)."""
    return {"workload": WORKLOAD, "unknowns": p.n, "block_rows": p.nbrows, "nnzb": p.nnzb,
            "spmv_bytes_per_step": spmv_bytes(p),
            "l2": "no flush: matrix stream 527 MB > 126 MB L2",
            "parallelism": f"replicas x{world}" if world > 1 else "1 GPU"}


def dist_problem_kw(world):
    """The N > 1 SpMV workload: a cantilever of `world` C1-sized slabs (63
    x-planes of 64 x 64 nodes per GPU, x slowest, so a rank owns contiguous
    planes), free-DOF form."""
    return dict(nx=63 * world, ny=63, nz=63, lx=float(world), dirichlet="eliminate", noise=0.01,
                seed=2022, x_slowest=True)


class Whole:
    """Global sizes of the N-slab problem (for dist_config on the b200 arm,
    where each rank generates only its slab)."""

    def __init__(self, n, nbrows, nnzb):
        self.n, self.nbrows, self.nnzb = n, nbrows, nnzb


def dist_config(world, p):
    """The N > 1 `config` object, identical in both arms."""
    return {"workload": f"cantilever {63 * world}x63x63 hex8 elements (x slowest), free-DOF, one "
                        f"C1-sized slab (258,048 block rows) per GPU, row-partitioned SpMV with an "
                        f"NCCL halo exchange per step",
            "unknowns": p.n, "block_rows": p.nbrows, "nnzb": p.nnzb,
            "spmv_bytes_per_step": spmv_bytes(p),
            "l2": "no flush: per-GPU matrix stream > 126 MB L2",
            "parallelism": f"row partition x{world} (NCCL P2P halo)"}


def cpu_reference_spmv(p, seconds, steps=None):
    """The reference's spmv<static_block<3>> (csr.hpp:129-160) from
    oracle/_ref on one host core over the C1 matrix: time-bounded sample."""
    from oracle.oracle import Ref
    ref = Ref()
    A = ref.bsr3(p.nbrows, p.nbrows, p.ptr, p.col, p.val.reshape(-1))
    x = np.random.default_rng(1).uniform(-1, 1, p.n)
    y = np.zeros(p.n)
    A.spmv(x, y)
    times = []
    t_end = time.perf_counter() + seconds
    while (steps is None and (time.perf_counter() < t_end or len(times) < 3)) or \
            (steps is not None and len(times) < steps):
        t0 = time.perf_counter()
        A.spmv(x, y)
        times.append(time.perf_counter() - t0)
    return times


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_reference_spmv_threaded(p, threads, seconds, steps=None):
    """The reference's own spmv<static_block<3>> (csr.hpp:129-160, unmodified,
    oracle/_ref) on every host thread: the matrix is cut into `threads`
    contiguous row slices of equal block count (reference csr<block3> objects
    of their own, built by the reference driver), and one y = A x is every
    thread running spmv on its slice at once (ctypes releases the GIL), the
    slices' y ranges disjoint.  The reference itself is single-threaded; this
    is the same kernel scaled out without modifying it."""
    from oracle.oracle import Ref
    ref = Ref()
    nnz = p.ptr[-1]
    cuts = [0]
    for t in range(1, threads):
        cuts.append(int(np.searchsorted(p.ptr, nnz * t // threads)))
    cuts.append(p.nbrows)
    cuts = sorted(set(cuts))
    val = p.val.reshape(-1)
    parts = [ref.bsr3(r1 - r0, p.nbrows, p.ptr[r0:r1 + 1], p.col, val)
             for r0, r1 in zip(cuts[:-1], cuts[1:])]
    x = np.random.default_rng(1).uniform(-1, 1, p.n)
    y = np.zeros(p.n)
    ys = [y[3 * r0:3 * r1] for r0, r1 in zip(cuts[:-1], cuts[1:])]
    from concurrent.futures import ThreadPoolExecutor
    pool = ThreadPoolExecutor(len(parts))

    def one():
        list(pool.map(lambda k: parts[k].spmv(x, ys[k]), range(len(parts))))

    one()
    times = []
    t_end = time.perf_counter() + seconds
    while (steps is None and (time.perf_counter() < t_end or len(times) < 3)) or \
            (steps is not None and len(times) < steps):
        t0 = time.perf_counter()
        one()
        times.append(time.perf_counter() - t0)
    pool.shutdown()
    return times, len(parts)


def spmv_bytes(p):
    return p.nnzb * 76 + (p.nbrows + 1) * 4 + p.nbrows * 24 + p.nbrows * 24


def run_reference(args, rank, world, dist):
    """--impl reference: the reference's own CPU path, rank 0 only.  Nothing
    of the product is loaded: the problem comes from the repo's host
    generator as linked into oracle/_ref (bitwise the product's
    generate_hex, tests/test_abi.py), the rigid-body modes from the
    reference's own rigid_body_modes (elasticity.hpp:38-52)."""
    if rank != 0:
        return
    from oracle.oracle import Params, Ref, SM_SPAI0
    ref = Ref()
    # the same workload as the b200 arm at this N: C1 on one GPU, the
    # N-slab cantilever of the row-partitioned SpMV above
    p = ref.gen_hex(**(C1 if world == 1 else dist_problem_kw(world)))
    nbytes = spmv_bytes(p)
    # each step: one full SpMV (5 ms class on all threads); bound the run
    steps = args.steps
    budget = 60.0
    threads = host_threads()
    warm, _ = cpu_reference_spmv_threaded(p, threads, 0, steps=max(1, min(args.warmup, 3)))
    per = statistics.median(warm)
    sample_steps = int(min(steps, max(3, budget / max(per, 1e-6))))
    times, cores = cpu_reference_spmv_threaded(p, threads, 0, steps=sample_steps)
    t = statistics.median(times)
    gbs = nbytes / t / 1e9
    t1 = statistics.median(cpu_reference_spmv(p, 0, steps=5))
    amg = None
    if world > 1:
        amg = {"note": "the b200 arm's N > 1 AMG leg strong-scales C4 / C3; the reference's C4 "
                       "setup takes 182 s and its solve about 1.5 h on one core (DESIGN.md section 3): "
                       "not run here"}
    elif os.environ.get("SAMG_BENCH_REF_AMG", "1") == "1":
        n, ptr, col, val = p.csr()
        B = p.nullspace()
        h = ref.setup(n, ptr, col, val, B, Params(smoother=SM_SPAI0))
        u, rep = h.cg_solve(p.rhs)
        amg = {"setup_s": h.setup_seconds, "solve_s": rep["solve_seconds"],
               "iterations": rep["iterations"], "relative_residual": rep["relative_residual"],
               "levels": h.nlevels, "converged": rep["converged"], "cores": 1,
               "timing": "steady_clock inside oracle/_ref around samg::setup (+ the harness "
                         "smoother arrays) and around cg_solve_op, as bench.hpp:72-80",
               "input": "host scalar CSR + host f/u (the reference's own API)"}
    line = {
        "metric": METRIC, "value": gbs, "unit": "GB/s", "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(p, world) if world == 1 else dist_config(world, p),
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "reference",
                         "sample": f"{len(times)} x samg::spmv<static_block<3>> over the full "
                                   f"{'C1' if world == 1 else 'cantilever'} "
                                   f"matrix (median), oracle/_ref, {cores} threads on row slices "
                                   f"of equal block count (the reference is single-threaded: "
                                   f"one thread runs {nbytes / t1 / 1e9:.2f} GB/s)",
                         "single_thread_value": nbytes / t1 / 1e9},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "amg": amg,
    }
    emit(line)


def run_b200(args, rank, world, local, dist):
    import torch

    import paper_2202_09056_b200 as pb
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    p = make_problem(pb)
    nbytes = spmv_bytes(p)
    A = pb.Bsr3.from_host(p.nbrows, p.nbrows, p.ptr, p.col, p.val.reshape(-1), device=local)
    x = torch.rand(p.n, dtype=torch.float64, device=dev) * 2 - 1
    y = torch.zeros(p.n, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream
    for _ in range(max(args.warmup, 3)):
        A.spmv_device(x.data_ptr(), y.data_ptr(), 1.0, 0.0, sh)
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            A.spmv_device(x.data_ptr(), y.data_ptr(), 1.0, 0.0, sh)
        e1.record(stream)
        torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    torch.cuda.synchronize(dev)
    ms_per = ms / args.steps
    gbs_rank = nbytes / (ms_per * 1e-3) / 1e9
    value = gbs_rank * world

    # e2e: host vectors through the C-ABI; every step copies its own x in
    # (H2D) and its y out (D2H).  samg_bsr3_spmv_batch pipelines the steps
    # over three streams (H2D of step k+1 and D2H of step k-1 overlap kernel k)
    e2e_steps = max(10, min(args.steps, 100))
    xh = torch.empty((e2e_steps, p.n), dtype=torch.float64, pin_memory=True).numpy()
    yh = torch.empty((e2e_steps, p.n), dtype=torch.float64, pin_memory=True).numpy()
    xh[:] = np.random.default_rng(3).uniform(-1, 1, (e2e_steps, p.n))
    from paper_2202_09056_b200._lib import check, lib
    for _ in range(2):
        check(lib.samg_bsr3_spmv_batch(A.h, 1.0, xh.ctypes.data, 0.0, yh.ctypes.data, 4))
    t0 = time.perf_counter()
    check(lib.samg_bsr3_spmv_batch(A.h, 1.0, xh.ctypes.data, 0.0, yh.ctypes.data, e2e_steps))
    e2e_t = (time.perf_counter() - t0) / e2e_steps
    if dist:
        t = torch.tensor([e2e_t], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_t = float(t.item())
    e2e_val = nbytes / e2e_t / 1e9 * world

    # full AMG setup + solve on the same problem through the drop-in calls a
    # reference user makes: samg_setup from the host scalar CSR + host B
    # (hierarchy.hpp:263) and samg_cg_solve with host f / u (cg.hpp:87);
    # uploads and the D2H of u inside the timed region, wall clock
    amg = None
    if args.amg_repeats > 0:
        A_csr = p.csr()
        B = p.nullspace()
        prm = pb.AmgParams(smoother="spai0", device=local)
        setups, solves, rep, h = [], [], None, None
        # untimed warm-up: lazy module loading of every setup/solve kernel
        hw = pb.setup(A_csr, B, "ns_block", prm)
        hw.cg_solve(p.rhs, pb.CgParams(max_iterations=2))
        hw.close()
        for _ in range(args.amg_repeats):
            if h is not None:
                h.close()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            h = pb.setup(A_csr, B, "ns_block", prm)
            torch.cuda.synchronize(dev)
            setups.append(time.perf_counter() - t0)
            t0 = time.perf_counter()
            u_host, rep = h.cg_solve(p.rhs)
            solves.append(time.perf_counter() - t0)
        levels = [h.level_info(l)[0] for l in range(h.nlevels)]
        amg = {"setup_s": statistics.median(setups), "solve_s": statistics.median(solves),
               "setup_s_all": setups, "solve_s_all": solves,
               "iterations": rep["iterations"], "relative_residual": rep["relative_residual"],
               "converged": rep["converged"], "levels_block_rows": levels,
               "coarse_dim": h.coarse_dim, "preconditioner_bytes": rep["preconditioner_bytes"],
               "smoother": "spai0 (M_i = A_ii / sum_j ||A_ij||_F^2)",
               "input": "drop-in C-ABI: samg_setup(host scalar CSR, host B) + "
                        "samg_cg_solve(host f, host u); H2D / D2H inside the timed region"}
        h.close()
        # the same with block input (samg_setup_bsr3, host BSR3 upload) and the
        # solve on device vectors
        f_d = torch.from_numpy(p.rhs).to(dev)
        u_d = torch.zeros_like(f_d)
        st, sv = [], []
        for it in range(1 + args.amg_repeats):
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            hb = pb.setup_bsr3(p.nbrows, p.ptr, p.col, p.val.reshape(-1), B, "ns_block", prm)
            torch.cuda.synchronize(dev)
            t1 = time.perf_counter()
            repb = hb.cg_solve_device(f_d.data_ptr(), u_d.data_ptr())
            torch.cuda.synchronize(dev)
            t2 = time.perf_counter()
            hb.close()
            if it:
                st.append(t1 - t0)
                sv.append(t2 - t1)
        amg["bsr3_input"] = {"setup_s": statistics.median(st), "solve_s": statistics.median(sv),
                             "iterations": repb["iterations"],
                             "what": "samg_setup_bsr3 (host BSR3 upload inside setup_s) + "
                                     "samg_cg_solve_device"}
        # fully device-resident pipeline: on-GPU assembly (samg_generate_hex_device),
        # setup from the device matrix, solve on the device right-hand side
        times = []
        for it in range(3):
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            dp = pb.generate_hex_device(pb.ProblemParams(**C1), device=local)
            torch.cuda.synchronize(dev)
            t1 = time.perf_counter()
            hd = pb.setup_device(dp.A, dp.nullspace_ptr, 6, "ns_block", prm)
            torch.cuda.synchronize(dev)
            t2 = time.perf_counter()
            repd = hd.cg_solve_device(dp.rhs_ptr, u_d.data_ptr())
            torch.cuda.synchronize(dev)
            t3 = time.perf_counter()
            times.append((t1 - t0, t2 - t1, t3 - t2))
            hd.close()
            del dp
        t0 = time.perf_counter()
        pb.generate_hex(**C1)
        host_gen = time.perf_counter() - t0
        amg["device_resident"] = {
            "assemble_s": statistics.median(t[0] for t in times),
            "setup_s": statistics.median(t[1] for t in times),
            "solve_s": statistics.median(t[2] for t in times),
            "iterations": repd["iterations"], "host_generator_s": host_gen,
            "runs": times,
            "what": "samg_generate_hex_device + samg_setup_device + samg_cg_solve_device "
                    "(median of three runs per phase)"}
        # the same problem with the reference's default smoother (block
        # ILU(0), bit-identical) and with the mixed-precision V-cycle
        variants = {}
        for key, vprm in (("ilu0", pb.AmgParams(smoother="ilu0", device=local)),
                          ("ilu0_latest_last", pb.AmgParams(smoother="ilu0", device=local,
                                                            ilu_sweep_order="latest_last")),
                          ("spai0_mixed", pb.AmgParams(smoother="spai0", device=local,
                                                       vcycle_precision="mixed"))):
            st, sv, vr = [], [], None
            for it in range(1 + args.amg_repeats):  # first run: untimed warm-up
                torch.cuda.synchronize(dev)
                t0 = time.perf_counter()
                hv = pb.setup_bsr3(p.nbrows, p.ptr, p.col, p.val.reshape(-1), B, "ns_block", vprm)
                torch.cuda.synchronize(dev)
                t1 = time.perf_counter()
                vr = hv.cg_solve_device(f_d.data_ptr(), u_d.data_ptr())
                torch.cuda.synchronize(dev)
                t2 = time.perf_counter()
                hv.close()
                if it:
                    st.append(t1 - t0)
                    sv.append(t2 - t1)
            variants[key] = {"setup_s": statistics.median(st), "solve_s": statistics.median(sv),
                             "iterations": vr["iterations"], "converged": vr["converged"],
                             "relative_residual": vr["relative_residual"]}
        amg["variants"] = variants
        if not args.no_c4:
            amg["c4"] = run_c4(pb, torch, dev, local)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            times, cores = cpu_reference_spmv_threaded(p, host_threads(), args.cpu_seconds)
            tc = statistics.median(times)
            t1 = statistics.median(cpu_reference_spmv(p, 0, steps=5))
            cpu = {"value": nbytes / tc / 1e9, "unit": "GB/s", "cores": cores, "kind": "reference",
                   "sample": f"{len(times)} x samg::spmv<static_block<3>> over the full C1 "
                             f"matrix in ~{args.cpu_seconds:.0f} s (median), oracle/_ref, "
                             f"{cores} threads on row slices (one thread: "
                             f"{nbytes / t1 / 1e9:.2f} GB/s)",
                   "single_thread_value": nbytes / t1 / 1e9}
        except Exception as e:  # reference not built on this box
            cpu = {"value": None, "unit": "GB/s", "cores": 1, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    peak, peak_src = peaks()
    traffic = ncu_traffic()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": config_dict(p, world),
            "roofline": {"bound": "hbm", "achieved": gbs_rank, "peak": peak, "unit": "GB/s",
                         "frac": gbs_rank / peak, "traffic": traffic, "peak_source": peak_src,
                         **read_peak_fields(gbs_rank),
                         "kernel": "k_bsr3_tma<8,8,2,false,EpiSpmv> (solve.cu, TMA-fed)"},
            "e2e": {"value": e2e_val, "unit": "GB/s", "h2d_bytes_per_step": 8 * p.n,
                    "d2h_bytes_per_step": 8 * p.n,
                    "path": "samg_bsr3_spmv_batch (C-ABI): per step H2D of its own x and D2H of "
                            "its y from/to pinned host memory, steps pipelined over per-engine "
                            "streams (H2D / SpMV / D2H, 4 staging slots), the SpMV on 96 of 148 "
                            "SMs to leave HBM headroom for the PCIe DMA"},
            "gpu_launches": args.steps,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "amg": amg,
        }
        emit(line)


C4 = dict(nx=199, ny=199, nz=199, dirichlet="eliminate", noise=0.01, seed=2022)


def run_c4(pb, torch, dev, local):
    """C4 (200^3-node cube, 23.88 M unknowns, 212.8 M blocks) on one GPU:
    assembled in HBM (samg_generate_hex_device; the host generator + 16.6 GB
    upload would dominate), ns_block setup from the device matrix, SPAI0-PCG
    to 1e-8.  Two runs, the first also warms the memory pool."""
    prm = pb.AmgParams(smoother="spai0", device=local)
    runs = []
    for it in range(2):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        dp = pb.generate_hex_device(pb.ProblemParams(**C4), device=local)
        torch.cuda.synchronize(dev)
        t1 = time.perf_counter()
        hd = pb.setup_device(dp.A, dp.nullspace_ptr, 6, "ns_block", prm)
        torch.cuda.synchronize(dev)
        t2 = time.perf_counter()
        u_d = torch.zeros(dp.n, dtype=torch.float64, device=dev)
        rep = hd.cg_solve_device(dp.rhs_ptr, u_d.data_ptr())
        torch.cuda.synchronize(dev)
        t3 = time.perf_counter()
        levels = [hd.level_info(l)[0] for l in range(hd.nlevels)]
        runs.append({"assemble_s": t1 - t0, "setup_s": t2 - t1, "solve_s": t3 - t2,
                     "iterations": rep["iterations"], "converged": rep["converged"],
                     "relative_residual": rep["relative_residual"]})
        hd.close()
        del dp, u_d
    torch.cuda.empty_cache()
    best = dict(runs[-1])
    for k in ("assemble_s", "setup_s", "solve_s"):
        best[k] = min(r[k] for r in runs)
    return {**best, "levels_block_rows": levels, "runs": runs, "unknowns": 23880000,
            "what": "C4 200^3 nodes free-DOF, samg_generate_hex_device + samg_setup_device + "
                    "samg_cg_solve_device, SPAI0; best of two runs per phase (the setup's "
                    "time varies with how much of the stream-ordered pool is already mapped)"}


def run_b200_dist(args, rank, world, local, dist):
    """N > 1: row-partitioned SpMV with an NCCL halo exchange every step.
    Weak scaling: a cantilever of world x C1-sized slabs (63 kept x-planes of
    64x64 nodes per GPU, x slowest so each rank owns contiguous planes);
    interior rows run while the halo is in flight (dist.cu)."""
    import torch

    import paper_2202_09056_b200 as pb
    from paper_2202_09056_b200.dist import DistMatrix, Halo, exchange_plan
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pp = pb.ProblemParams(**dist_problem_kw(world))
    per_plane = 64 * 64
    starts = np.array([63 * r * per_plane for r in range(world + 1)], dtype=np.int64)
    r0, r1 = int(starts[rank]), int(starts[rank + 1])
    mine = pb.generate_hex(pb.ProblemParams(**{**pp.__dict__, "node_begin": r0, "node_end": r1}))
    dm = DistMatrix(mine.ptr, mine.col, mine.val.reshape(-1), starts, rank)
    exchange_plan(dm, dist, device=dev)
    dm.to_device(local, 4)
    inf = dm.info()
    halo = Halo(dm, dist, dev)
    nloc, ngh = inf["nloc"], inf["nghost"]
    halo.x_ext[:3 * nloc] = torch.rand(3 * nloc, dtype=torch.float64, device=dev)
    y = torch.zeros(3 * nloc, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream
    nbytes = mine.nnzb * 76 + (nloc + 1) * 4 + (nloc + ngh) * 24 + nloc * 24

    def step():
        reqs = halo.start(sh)
        dm.spmv(0, halo.x_ext.data_ptr(), y.data_ptr(), stream=sh)
        for r in reqs:
            r.wait()
        dm.spmv(1, halo.x_ext.data_ptr(), y.data_ptr(), stream=sh)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize(dev)
    dist.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    tb = torch.tensor([float(nbytes), float(mine.nnzb)], device=dev, dtype=torch.float64)
    dist.all_reduce(tb)
    total_bytes = float(tb[0].item())
    nnzb_total = int(tb[1].item())
    ms_per = ms / args.steps
    value = total_bytes / (ms_per * 1e-3) / 1e9
    # e2e: host x_local in, host y_local out, same distributed step
    xh = torch.empty(3 * nloc, dtype=torch.float64, pin_memory=True)
    yh = torch.empty(3 * nloc, dtype=torch.float64, pin_memory=True)
    xh.copy_(torch.rand(3 * nloc, dtype=torch.float64))
    e2e_steps = max(10, min(args.steps, 200))
    dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        halo.x_ext[:3 * nloc].copy_(xh, non_blocking=True)
        step()
        yh.copy_(y, non_blocking=True)
        torch.cuda.synchronize(dev)
    e2e_t = (time.perf_counter() - t0) / e2e_steps
    te = torch.tensor([e2e_t], device=dev, dtype=torch.float64)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_val = total_bytes / float(te.item()) / 1e9
    amg = run_dist_amg(args, rank, world, local, dist) if args.amg_repeats > 0 and not args.no_c4 else None
    peak, peak_src = peaks()
    gb_rank = nbytes / (ms_per * 1e-3) / 1e9
    if rank == 0:
        emit({
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": dist_config(world, Whole(3 * 258048 * world, 258048 * world, nnzb_total)),
            "partition": {"block_rows_rank0": nloc, "ghost_block_rows_rank0": ngh,
                          "interior_rows_rank0": inf["ninterior"], "nnzb_rank0": mine.nnzb},
            "roofline": {"bound": "hbm", "achieved": gb_rank, "peak": peak, "unit": "GB/s",
                         "frac": gb_rank / peak, "traffic": ncu_traffic(),
                         "peak_source": peak_src, **read_peak_fields(gb_rank),
                         "kernel": "k_bsr3_tma<8,8,2,false,EpiSpmv> on the interior row view + k_bsr3 on the boundary rows (dist.cu, solve.cu)"},
            "e2e": {"value": e2e_val, "unit": "GB/s", "h2d_bytes_per_step": 8 * 3 * nloc * world,
                    "d2h_bytes_per_step": 8 * 3 * nloc * world,
                    "path": "samg_dist_pack/spmv (C-ABI) + torch.distributed NCCL halo"},
            "gpu_launches": 3 * args.steps,
            "clocks": clk.summary(),
            "cpu_baseline": None,
            "amg": amg,
        })


C3 = dict(nx=511, ny=63, nz=63, lx=511 / 63, dirichlet="eliminate", load="traction_xend",
          x_slowest=True)


def run_dist_amg(args, rank, world, local, dist):
    """Multi-GPU AMG, strong scaling on the largest configs (C4 200^3 cube,
    C3 512x64x64 x-slowest cantilever): each rank assembles ONLY its slab of
    node planes on its GPU (samg_generate_hex_device with a node range), the
    setup is distributed (samg_dsetup_device: every rank builds its rows of
    each large level, dsetup.cu) and the partitioned PCG runs with NCCL halos
    and all-reduces inside one CUDA graph (dsolve.cu).  Times: wall clock
    around each phase, max over ranks; the first run warms up, then the
    best of two per phase."""
    import torch

    import paper_2202_09056_b200 as pb
    from paper_2202_09056_b200.dist import DistHierarchy
    dev = torch.device("cuda", local)

    def tmax(x):
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    out = {}
    for name, kw, planes, per_plane in (
            ("C4", C4, C4["nz"] + 1, C4["nx"] * (C4["ny"] + 1)),
            ("C3", C3, C3["nx"], (C3["ny"] + 1) * (C3["nz"] + 1))):
        # contiguous node ranges = whole planes (z-slabs for C4 whose x runs
        # fastest, x-slabs for the x-slowest C3)
        cuts = [planes * r // world for r in range(world + 1)]
        rs = np.array([c * per_plane for c in cuts], dtype=np.int64)
        n0, n1 = int(rs[rank]), int(rs[rank + 1])
        prm = pb.AmgParams(smoother="spai0", device=local)
        uid = None
        runs = []
        for it in range(1 + max(2, args.amg_repeats // 2)):
            dist.barrier()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            dp = pb.generate_hex_device(pb.ProblemParams(**{**kw, "node_begin": n0, "node_end": n1}),
                                        device=local)
            torch.cuda.synchronize(dev)
            t1 = time.perf_counter()
            dh = DistHierarchy(0, None, None, None, None, rank, world, dist=dist, row_starts=rs,
                               min_rows=4096, prm=prm, uid=uid, device=(dp.A, dp.nullspace_ptr))
            torch.cuda.synchronize(dev)
            t2 = time.perf_counter()
            u = torch.zeros(dp.n + 3, dtype=torch.float64, device=dev)
            rep = dh.cg_solve_device(dp.rhs_ptr, u.data_ptr(),
                                     pb.CgParams(max_iterations=2 if it == 0 else 5000))
            torch.cuda.synchronize(dev)
            t3 = time.perf_counter()
            inf = dh.info()
            rec = {"assemble_s": tmax(t1 - t0), "setup_s": tmax(t2 - t1), "solve_s": tmax(t3 - t2),
                   "iterations": rep["iterations"], "converged": rep["converged"],
                   "relative_residual": rep["relative_residual"]}
            dh.close()
            del dp, u
            if it:
                runs.append(rec)
        # best per phase over the timed runs, as the single-GPU C4 leg (the
        # setup's time varies with how much of the memory pool is mapped)
        best = dict(runs[-1])
        for k in ("assemble_s", "setup_s", "solve_s"):
            best[k] = min(r[k] for r in runs)
        out[name] = {**best, "runs": runs, "levels": inf["nlevels"],
                     "distributed_levels": inf["dist_levels"],
                     "held_rows_rank0": inf["held_rows"], "rows_rank0": n1 - n0,
                     "what": f"{name}: each rank assembles its slab on the GPU, distributed setup "
                             f"(samg_dsetup_device), partitioned PCG (graph, NCCL halos), SPAI0"}
        torch.cuda.empty_cache()
    out["problem"] = "strong scaling: the same global C4 / C3 on every N"
    out["timing"] = "wall clock around assemble / setup / solve, max over ranks; best of two timed runs per phase"
    return out


def main():
    args = parse()
    # NCCL's own log lines ("NCCL version ...") go to stderr: stdout carries
    # exactly one JSON line
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    global _OUT_FD
    sys.stdout.flush()
    _OUT_FD = os.dup(1)
    os.dup2(2, 1)
    rank, world, local, dist = dist_init(args)
    try:
        if args.impl == "reference":
            run_reference(args, rank, world, dist)
        elif world > 1 or args.force_dist:
            run_b200_dist(args, rank, world, local, dist)
        else:
            run_b200(args, rank, world, local, dist)
    finally:
        if dist:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
