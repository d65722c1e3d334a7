"""Benchmark of the Fortran array path of arXiv 2409.18824 on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--rows all|none|...] [--impl reference]

Headline (BASELINE.json configs[1]): the 2-D 5-point Jacobi of real(8) 8192^2, one step =
100 sweeps (ftn_jacobi); value = GLUPS = interior points x sweeps / time.  With N > 1
(torchrun) every rank owns an 8192 x 8192 slab of an 8192 x (8192 N) grid and exchanges one
halo column per sweep over NCCL (ftn_jacobi_dist): weak scaling.

"rows" reports every other SURVEY §8 row on its BASELINE config, each with a roofline
fraction: C4 element-wise / reductions (GB/s), C3 MATMUL (TFLOP/s), C5 3-D Jacobi (GLUPS),
and the paper's Table III shapes.  Inputs are synthetic (splitmix64, seed 18824) and
generated on the device by ftn_gen_fill; every working set is larger than the 126 MB L2.

--impl reference times the oracle (oracle/, plain C) on the host cores on a bounded sample
of the same workload (there is no reference code base for this paper).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 18824
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0          # GB/s, B200_PROFILING.md fallback
FP64_PEAK_TFLOPS = 148 * 1.965 * 128 / 1000.0   # 37.2: SMs x max clock x DMMA FLOP/clk/SM (probe: 37.1 measured)


def load_peaks():
    try:
        with open(PEAKS_FILE) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


# ----------------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed regions."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None
        self.active = False
        self.lock = threading.Lock()

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            with self.lock:
                if self.active:
                    self.samples.append(parts)

    def timing(self, on: bool):
        with self.lock:
            self.active = on

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        with self.lock:
            s = list(self.samples)
        if not s:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = sorted(float(x[0]) for x in s if x[0].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for x in s for k in range(4) if x[2 + k].lower().startswith("active")})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": float(s[0][1]), "reasons": reasons,
                "samples": len(s)}


# ----------------------------------------------------------------------------------- timing helpers
LAST_LAUNCHES = [0]
LAST_STEP_MS = [0.0, 0.0]   # min, median of the last timed() call's steps (this rank)


def timed(torch, fn, steps, warmup, clocks=None, dist=None, counter=None):
    """W untimed runs, then `steps` runs bracketed by barrier + synchronize; CUDA events on the
    current stream.  Returns seconds for all steps (max over ranks); LAST_LAUNCHES[0] gets the
    number of libftn kernel launches inside the timed region (when `counter` is given)."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    if clocks:
        clocks.timing(True)
    c0 = counter() if counter else 0
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(steps - 1)]
    a.record()
    for k in range(steps):
        fn()
        if k < steps - 1:
            marks[k].record()
    b.record()
    LAST_LAUNCHES[0] = (counter() - c0) if counter else 0
    torch.cuda.synchronize()
    if clocks:
        clocks.timing(False)
    t = a.elapsed_time(b) / 1e3
    ev = [a] + marks + [b]   # per-step device times (median and min beside the mean)
    per = sorted(ev[k].elapsed_time(ev[k + 1]) for k in range(steps))
    LAST_STEP_MS[:] = [per[0], per[len(per) // 2]]
    if dist is not None:
        tt = torch.tensor([t], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
        dist.barrier()
    return t


def c5_checksum(torch, ftn, R, p_lo, p_hi, comm):
    """Decomposition-independent checksum of the C5 result: the integer SUM (mod 2^64, order
    free) of the bit patterns of the global interior planes 2..2047 -- on one GPU the section
    R(:, :, 2:2047), on N ranks the owned planes p_lo..p_hi of each slab, combined by the
    global integer SUM.  Equal across N iff every owned value is bit-identical (the result is
    the same whatever the slab count: R#16 + the exchange)."""
    bits = ftn.FArray(R.tensor.view(torch.int64))
    sec = bits.section((1, bits.shape[0]), (1, bits.shape[1]), (p_lo, p_hi))
    v = comm.sum(sec) if comm is not None else ftn.sum(sec)
    return {"kind": "SUM of int64 bit patterns of global planes 2..2047 (mod 2^64)",
            "value": int(v.item()) & 0xFFFFFFFFFFFFFFFF}


def jacobi_faces(ftn, U, n1, n2):
    """synth.jacobi_init recipe on the device: interior U[0,1), j=1 face 1.0, other faces 0.
    --mode intvalued: interior integers in [-8, 8]; --mode closed: the whole array is the
    linear (discrete-harmonic) field u(i,j) = (i-1) + n1 (j-1), a fixed point of the sweep:
    every step must return it bit for bit (checked after the timed region)."""
    if MODE == "closed":
        ftn.gen_fill(U, SEED, 0, ftn.GEN_LINEAR)
        return
    ftn.gen_fill(U, SEED, 0, ftn.GEN_INT8 if MODE == "intvalued" else ftn.GEN_U01)
    for tr in (((1, n1), (n2, n2)), ((1, 1), (1, n2)), ((n1, n1), (1, n2))):
        ftn.fill(U.section(*tr), 0.0)
    ftn.fill(U.section((1, n1), (1, 1)), 1.0)


# ----------------------------------------------------------------------------------- headline
def bench_jacobi2d(torch, ftn, args, ctx):
    n, sweeps = 8192, SWEEPS
    N, rank = ctx["world"], ctx["rank"]
    if N == 1 and not ctx.get("force_dist"):
        U, W = ftn.FArray.empty((n, n)), ftn.FArray.empty((n, n))
        jacobi_faces(ftn, U, n, n)
        ftn.assign(W, U)
        step = lambda: ftn.jacobi(U, W, sweeps)  # noqa: E731
        interior = (n - 2) * (n - 2)
    else:
        # weak scaling: global grid 8192 x (8192 N + 2); rank r owns global columns
        # [1 + r n, (r+1) n] (Fortran dim 2) and keeps `halo` halo planes per side, so
        # ftn_jacobi_dist exchanges T planes and runs T fused sweeps per step (T = halo)
        halo = max(1, ftn.jacobi_fusion())
        nl = n + 2 * halo
        U, W = ftn.FArray.empty((n, nl)), ftn.FArray.empty((n, nl))
        if MODE == "closed":   # the linear field (i-1) + n (global column + halo - 1): harmonic
            ftn.gen_fill(U, SEED, 0, ftn.GEN_LINEAR, t0=n * n * rank)
        else:
            ftn.gen_fill(U, SEED, 1 + rank, ftn.GEN_INT8 if MODE == "intvalued" else ftn.GEN_U01)
            ftn.fill(U.section((1, 1), (1, nl)), 0.0)
            ftn.fill(U.section((n, n), (1, nl)), 0.0)
            if rank == 0:
                ftn.fill(U.section((1, n), (halo, halo)), 1.0)            # global boundary plane j = 1
            if rank == N - 1:
                ftn.fill(U.section((1, n), (nl - halo + 1, nl - halo + 1)), 0.0)   # global plane j = N
        ftn.assign(W, U)
        comm = ctx["comm"]
        step = lambda: comm.jacobi(U, W, sweeps, halo=halo)  # noqa: E731
        interior = (n - 2) * n * N
    t = timed(torch, step, args.steps, args.warmup, ctx["clocks"], ctx["dist"], counter=ftn.launch_count)
    launches = LAST_LAUNCHES[0]
    step_min, step_med = LAST_STEP_MS
    glups = interior * sweeps * args.steps / t / 1e9
    # launch plan of ftn_jacobi: F launches of T fused sweeps + S1 single sweeps per step
    halo_T = max(1, ftn.jacobi_fusion())
    plan = ftn.jacobi_plan(sweeps, halo_T)
    per_launch_bytes = 16 * (n - 2) * (n - 2 if N == 1 else n)       # algorithmic: read u once, write once
    stencil_launches = len(plan) * args.steps
    achieved = per_launch_bytes * stencil_launches / t / 1e9          # GB/s, launches back to back
    res = {"value": glups, "ms_per_step": t / args.steps * 1e3, "launches": launches,
           "ms_step_min": step_min, "ms_step_median": step_med,
           "achieved_gbs": achieved, "per_launch_bytes": per_launch_bytes,
           "plan": {"max_sweeps_per_launch": halo_T, "launches_per_step": len(plan),
                    "sweeps_per_launch": {str(k): plan.count(k) for k in sorted(set(plan))}}}
    if MODE == "closed":
        # the harmonic field is a fixed point: after every step the result array must hold the
        # initial field bit for bit (MAXVAL(ABS(result - initial)) over the owned planes = 0)
        R = U if sweeps % 2 == 0 else W
        G = ftn.FArray.empty(tuple(U.shape))
        if N == 1 and not ctx.get("force_dist"):
            ftn.gen_fill(G, SEED, 0, ftn.GEN_LINEAR)
            diff = float(ftn.maxval_absdiff(R, G).item())
        else:
            ftn.gen_fill(G, SEED, 0, ftn.GEN_LINEAR, t0=n * n * rank)
            own = ((1, n), (halo + 1, U.shape[1] - halo))
            d = ftn.maxval_absdiff(R.section(*own), G.section(*own)).reshape(1)
            if ctx["dist"] is not None:
                ctx["dist"].all_reduce(d, op=ctx["dist"].ReduceOp.MAX)
            diff = float(d.item())
        res["check"] = {"mode": "closed", "field": "u(i,j) = (i-1) + 8192 (j-1) (discrete-harmonic)",
                        "max_abs_diff_vs_initial": diff, "bit_exact": diff == 0.0}
        del G, R
    # ---- e2e: through the C ABI from pinned host buffers (H2D of u, D2H of the result inside);
    # at N > 1 every rank moves its own slab, timed as the max over ranks
    shape = tuple(U.shape)
    host_u = torch.empty(shape[::-1], dtype=torch.float64, pin_memory=True).t()   # Fortran layout
    host_u.copy_(U.tensor)
    dist_path = not (N == 1 and not ctx.get("force_dist"))
    halo_e2e = max(1, ftn.jacobi_fusion())
    ne = max(6, args.steps)
    if not dist_path:
        # ftn_jacobi_host (host in -> device -> sweeps -> host out) per step; consecutive steps
        # rotate over NSTR streams and buffer sets, so one step's device-to-host copy overlaps
        # the next steps' host-to-device copies (PCIe is full duplex) and kernels; every step
        # still moves its full input and result
        NSTR = int(os.environ.get("FTN_E2E_STREAMS", "3"))
        sets = [(ftn.FArray.empty(shape), ftn.FArray.empty(shape),
                 torch.empty(shape[::-1], dtype=torch.float64, pin_memory=True).t()) for _ in range(NSTR)]
        streams = [torch.cuda.Stream() for _ in range(NSTR)]

        def e2e_run(k):
            cur = torch.cuda.current_stream()
            ev = torch.cuda.Event()
            ev.record(cur)
            for st in streams:
                st.wait_event(ev)
            for i in range(k):
                U2, W2, hout = sets[i % NSTR]
                ftn.jacobi_host(host_u, hout, U2, W2, sweeps, stream=streams[i % NSTR])
            for st in streams:
                e = torch.cuda.Event()
                e.record(st)
                cur.wait_event(e)

        e2e_run(NSTR)
        torch.cuda.synchronize()
        te = timed(torch, lambda: e2e_run(ne), 1, 0, None, ctx["dist"])
        host_out = sets[0][2]
        note = ("per step: ftn_jacobi_host = H2D of u from pinned host memory, device copy u -> unew "
                "(boundary), the 100 sweeps, D2H of the result; consecutive steps rotate over 3 streams "
                "(copies of one step overlap the next steps')")
        del sets
    else:
        # the distributed step keeps its NCCL exchanges on one stream (the caller's); the copies
        # of neighbouring steps run beside it on two copy streams over NB buffer sets: the H2D of
        # step i+1 and the D2H of step i-1 overlap the sweeps of step i, and every step still
        # moves its full slab in and its full result out
        NB = 3
        sets = [(ftn.FArray.empty(shape), ftn.FArray.empty(shape),
                 torch.empty(shape[::-1], dtype=torch.float64, pin_memory=True).t()) for _ in range(NB)]
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()

        def e2e_run(k):
            main = torch.cuda.current_stream()
            start = torch.cuda.Event()
            start.record(main)
            s_in.wait_event(start)
            s_out.wait_event(start)
            outs = [None] * NB            # D2H done event of the last step that used each set
            for i in range(k):
                U2, W2, hout = sets[i % NB]
                if outs[i % NB] is not None:
                    s_in.wait_event(outs[i % NB])
                with torch.cuda.stream(s_in):
                    U2.tensor.copy_(host_u, non_blocking=True)
                e_in = torch.cuda.Event()
                e_in.record(s_in)
                main.wait_event(e_in)
                ftn.assign(W2, U2)
                new = ctx["comm"].jacobi(U2, W2, sweeps, halo=halo_e2e)
                e_c = torch.cuda.Event()
                e_c.record(main)
                s_out.wait_event(e_c)
                with torch.cuda.stream(s_out):
                    hout.copy_((W2 if new else U2).tensor, non_blocking=True)
                outs[i % NB] = torch.cuda.Event()
                outs[i % NB].record(s_out)
            done = torch.cuda.Event()
            done.record(s_out)
            main.wait_event(done)

        e2e_run(NB)
        torch.cuda.synchronize()
        te = timed(torch, lambda: e2e_run(ne), 1, 0, None, ctx["dist"])
        host_out = sets[0][2]
        note = ("per step: H2D of the rank's slab from pinned host memory, device copy u -> unew (boundary), "
                "the 100 sweeps (ftn_jacobi_dist, halos over the communicator), D2H of the result; the copies of "
                "neighbouring steps overlap the sweeps on two copy streams over 3 buffer sets; bytes summed over ranks")
        del sets
    res["e2e"] = {"value": interior * sweeps * ne / te / 1e9, "unit": "GLUPS",
                  "h2d_bytes_per_step": host_u.numel() * 8 * N, "d2h_bytes_per_step": host_out.numel() * 8 * N,
                  "note": note}
    del host_u, host_out
    del U, W
    torch.cuda.empty_cache()
    return res


# ----------------------------------------------------------------------------------- §8 rows
def bench_rows(torch, ftn, args, ctx, hbm_peak):
    rows = {}
    N, rank = ctx["world"], ctx["rank"]
    steps, warm = max(3, args.steps // 2), 2
    dist = ctx["dist"]
    comm = ctx.get("comm")
    distmode = N > 1 or bool(ctx.get("force_dist"))   # the NCCL code paths (also at N = 1 with --dist)

    def gbs_row(name, nbytes, fn, units=None):
        t = timed(torch, fn, steps, warm, None, dist)
        gbs = nbytes * N * steps / t / 1e9
        rows[name] = {"value": gbs, "unit": "GB/s", "ms": t / steps * 1e3, "ms_min": LAST_STEP_MS[0],
                      "ms_median": LAST_STEP_MS[1],
                      "roofline": {"bound": "hbm", "frac": gbs / N / hbm_peak,
                                   "frac_of_8TBps_spec": gbs / N / HBM_SPEC_GBS}}

    # C1: real(8) a(0:63,1:48) = its 0-based offset, s = a(::2,:); latency of each call (median of
    # 1000, CUDA events around the call: host launch overhead included) and the closed forms of
    # SURVEY §8(c.4) checked on the results (not a roofline case: 24 KiB)
    if "c1" in args.rows and N == 1:
        a = ftn.FArray.empty((64, 48), lbounds=[0, 1])
        ftn.gen_fill(a, SEED, 0, ftn.GEN_LINEAR)          # a(i,j) = i + 64(j-1)
        s = a.section((0, 63, 2), (1, 48))
        c = a.section((1, 63, 2), (1, 48))
        e = ftn.FArray.empty((32, 48), lbounds=[-5, 10])
        ftn.gen_fill(e, SEED, 1, ftn.GEN_U01)
        r = ftn.FArray.empty((32, 48))
        st = ftn.FArray.empty((48, 32))
        m48 = ftn.FArray.empty((48, 48))
        b48 = [ftn.FArray.empty((48, 48)) for _ in range(2)]
        for q, x in enumerate(b48):
            ftn.gen_fill(x, SEED, 2 + q, ftn.GEN_U11)
        out = torch.empty((), dtype=torch.float64, device="cuda")
        ops = {"muladd_r=s*c+d": lambda: ftn.muladd(r, s, c, e, contract=CONTRACT),
               "sum_s": lambda: ftn.sum(s, out),
               "maxval_s": lambda: ftn.maxval(s, out),
               "minval_s": lambda: ftn.minval(s, out),
               "transpose_s": lambda: ftn.transpose(st, s),
               "matmul_transpose(s)_s_48x48x32": lambda: ftn.matmul(m48, s, s, transpose_a=True),
               "matmul_48^3": lambda: ftn.matmul(m48, b48[0], b48[1])}
        lat = {}
        for name, fn in ops.items():
            for _ in range(20):
                fn()
            torch.cuda.synchronize()
            ts = []
            for _ in range(1000):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            ts.sort()
            lat[name] = round(ts[len(ts) // 2], 2)
        # device-side latency: 100 calls captured in one CUDA graph, replayed (no host overhead)
        lat_graph = {}
        gs = torch.cuda.Stream()
        for name, fn in ops.items():
            with torch.cuda.stream(gs):
                fn()
                gs.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=gs):
                    for _ in range(100):
                        fn()
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            lat_graph[name] = round(e0.elapsed_time(e1) * 1e3 / 1000, 2)
            del g
        # closed forms: SUM(s) = 2357760, MAXVAL = 3070 (s holds the even i),
        # MINVAL = 0; MATMUL(TRANSPOSE(s), s)(p,q) = 41664 + 63488(p+q-2) + 131072(p-1)(q-1)
        checks = {"sum": ftn.sum(s).item() == 2357760.0, "maxval": ftn.maxval(s).item() == 3070.0,
                  "minval": ftn.minval(s).item() == 0.0}
        ftn.matmul(m48, s, s, transpose_a=True)
        p_ = torch.arange(1, 49, dtype=torch.float64, device="cuda")
        cf = 41664 + 63488 * (p_[:, None] + p_[None, :] - 2) + 131072 * (p_[:, None] - 1) * (p_[None, :] - 1)
        checks["matmul_transpose"] = bool(torch.equal(m48.tensor, cf))
        ftn.transpose(st, s)
        checks["transpose"] = bool(torch.equal(st.tensor, s.view_tensor().t()))
        # the same calls from plain C through the ABI (examples/c1_latency.c): no Python in the loop
        c_abi = None
        try:
            import tempfile
            cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
            lib = os.path.join(ROOT, "paper_2409_18824_b200")
            with tempfile.TemporaryDirectory() as td:
                exe = os.path.join(td, "c1_latency")
                subprocess.run(["gcc", "-O2", os.path.join(ROOT, "examples", "c1_latency.c"), "-I",
                                os.path.join(ROOT, "include"), "-I", os.path.join(cuda, "include"), "-L", lib, "-lftn",
                                "-L", os.path.join(cuda, "lib64"), "-lcudart", f"-Wl,-rpath,{lib}",
                                f"-Wl,-rpath,{os.path.join(cuda, 'lib64')}", "-o", exe], check=True,
                               capture_output=True, timeout=120)
                out_c = subprocess.run([exe], capture_output=True, text=True, timeout=120, check=True)
                c_abi = json.loads(out_c.stdout.strip().splitlines()[-1])
        except Exception as e:  # report, do not fail the bench line
            c_abi = {"unavailable": str(e)[:200]}
        rows["c1_latency"] = {"value": lat["sum_s"], "unit": "us (median of 1000, SUM(a(::2,:)))",
                              "c_abi": c_abi,
                              "latency_us": lat, "latency_graph_us": lat_graph,
                              "note": "latency_us: one Python call each (ctypes marshalling + launch + kernel); "
                                      "latency_graph_us: per call inside a CUDA graph of 100 calls (device time)",
                              "closed_forms_ok": checks}
        del a, s, c, e, r, st, m48, b48

    # C4: 1024^3 arrays x(-511:512, 0:1023, 1:1024); at N>1 slabs of 1024/N planes (strong scaling)
    if "c4" in args.rows:
        nk = 1024 // N
        shape = (1024, 1024, nk)
        lbs = [-511, 0, 1 + rank * nk]
        arrs = [ftn.FArray.empty(shape, lbounds=lbs) for _ in range(4)]
        for k, a in enumerate(arrs):
            ftn.gen_fill(a, SEED, 10 + k, ftn.GEN_U01)
        b, c, d, r = arrs
        n_el = 1024 * 1024 * nk
        gbs_row("c4_muladd_r=b*c+d", 32 * n_el, lambda: ftn.muladd(r, b, c, d, contract=CONTRACT))
        gbs_row("hbm_copy_r=b", 16 * n_el, lambda: ftn.assign(r, b))      # the in-run copy ceiling
        out = torch.empty((), dtype=torch.float64, device="cuda")
        if not distmode:
            gbs_row("c4_sum", 8 * n_el, lambda: ftn.sum(b, out))
            gbs_row("c4_maxval", 8 * n_el, lambda: ftn.maxval(b, out))
            gbs_row("c4_minval", 8 * n_el, lambda: ftn.minval(b, out))
            fx = ftn.FArray(b.tensor.permute(2, 1, 0).reshape(-1))
            fy = ftn.FArray(c.tensor.permute(2, 1, 0).reshape(-1))
            gbs_row("c4_dot_product", 16 * n_el, lambda: ftn.dot_product(fx, fy, out))
            # PRODUCT and DIM= reductions (results are 8 MiB: not counted)
            gbs_row("f1_product", 8 * n_el, lambda: ftn.product(b, out))
            rd = [ftn.FArray.empty((1024, 1024)) for _ in range(3)]
            for dd in (1, 2, 3):
                gbs_row(f"f1_sum_dim{dd}", 8 * n_el, lambda dd=dd: ftn.sum_dim(b, dd, rd[dd - 1]))
            gbs_row("f1_maxval_dim3", 8 * n_el, lambda: ftn.maxval_dim(b, 3, rd[2]))
            del rd
        else:
            gbs_row("c4_sum_global", 8 * n_el, lambda: comm.sum(b, out))
            gbs_row("c4_maxval_global", 8 * n_el, lambda: comm.maxval(b, out))
            fx = ftn.FArray(b.tensor.permute(2, 1, 0).reshape(-1))
            fy = ftn.FArray(c.tensor.permute(2, 1, 0).reshape(-1))
            gbs_row("c4_dot_product_global", 16 * n_el, lambda: comm.dot_product(fx, fy, out))
        del arrs, b, c, d, r, fx, fy
        torch.cuda.empty_cache()
        # section variant: parents (1:1024,1:1024,1:2048/N), sections (:,:,1::2)
        parents = [ftn.FArray.empty((1024, 1024, 2 * nk)) for _ in range(4)]
        for k, p in enumerate(parents):
            ftn.gen_fill(p, SEED, 20 + k, ftn.GEN_U01)
        secs = [p.section((1, 1024), (1, 1024), (1, 2 * nk, 2)) for p in parents]
        gbs_row("c4_section_muladd", 32 * n_el, lambda: ftn.muladd(secs[3], secs[0], secs[1], secs[2], contract=CONTRACT))
        if N == 1:
            gbs_row("c4_section_sum", 8 * n_el, lambda: ftn.sum(secs[0], out))
        del parents, secs
        torch.cuda.empty_cache()
        # dim-1-strided variant: parents (0:2047,1024,1024/N), sections (0:2047:2,:,:):
        # every 32-byte sector carries 2 used elements of 4, so DRAM moves ~2x the algorithmic bytes
        if N == 1:
            parents = [ftn.FArray.empty((2048, 1024, nk), lbounds=[0, 1, 1]) for _ in range(4)]
            for k, p in enumerate(parents):
                ftn.gen_fill(p, SEED, 30 + k, ftn.GEN_U01)
            secs = [p.section((0, 2047, 2), (1, 1024), (1, nk)) for p in parents]
            gbs_row("c4_dim1_strided_muladd", 32 * n_el, lambda: ftn.muladd(secs[3], secs[0], secs[1], secs[2], contract=CONTRACT))
            gbs_row("c4_dim1_strided_sum", 8 * n_el, lambda: ftn.sum(secs[0], out))
            for nm in ("c4_dim1_strided_muladd", "c4_dim1_strided_sum"):
                rows[nm]["roofline"]["note"] = "sector-limited: 2 of every 4 elements of a 32-byte sector are used"
            del parents, secs
            torch.cuda.empty_cache()

    # C3: MATMUL 8192^3, column blocks of b and c over the ranks (a replicated)
    if "c3" in args.rows:
        n = 8192
        nc = n // N
        A = ftn.FArray.empty((n, n))
        B = ftn.FArray.empty((n, nc))
        C = ftn.FArray.empty((n, nc))
        ftn.gen_fill(A, SEED, 1, ftn.GEN_U11)
        ftn.gen_fill(B, SEED, 2 + rank, ftn.GEN_U11)
        fn = (lambda: ftn.matmul(C, A, B)) if not distmode else (lambda: comm.matmul(C, A, B))
        t = timed(torch, fn, steps, warm, ctx["clocks"], dist)
        tf = 2.0 * n * n * n * steps / t / 1e12
        rows["c3_matmul_8192"] = {"value": tf, "unit": "TFLOP/s", "ms": t / steps * 1e3,
                                  "roofline": {"bound": "fp64 tensor (DMMA)", "frac": tf / N / FP64_PEAK_TFLOPS,
                                               "peak": FP64_PEAK_TFLOPS}}
        if N == 1:
            Ac, Bc = A.tensor, B.tensor
            tc = timed(torch, lambda: torch.matmul(Ac, Bc), 3, 1, None, None)
            rows["c3_matmul_8192"]["cublas_dgemm_tflops_context"] = 2.0 * n ** 3 * 3 / tc / 1e12
            # MATMUL(TRANSPOSE(a), b) without forming the transpose, and the
            # rank-1 forms (HBM-bound: 8 B per matrix element)
            t = timed(torch, lambda: ftn.matmul(C, A, B, transpose_a=True), steps, warm, None, None)
            tf = 2.0 * n ** 3 * steps / t / 1e12
            rows["f3_matmul_transpose_a_8192"] = {"value": tf, "unit": "TFLOP/s", "ms": t / steps * 1e3,
                                                  "roofline": {"bound": "fp64 tensor (DMMA)",
                                                               "frac": tf / FP64_PEAK_TFLOPS}}
            xv, yv = ftn.FArray.empty((n,)), ftn.FArray.empty((n,))
            ftn.gen_fill(xv, SEED, 9, ftn.GEN_U11)
            gbs_row("f3_matvec_8192", 8 * n * n, lambda: ftn.matmul(yv, A, xv))
            gbs_row("f3_vecmat_8192", 8 * n * n, lambda: ftn.matmul(yv, xv, A))
            del xv, yv
        del A, B, C
        torch.cuda.empty_cache()

    # paper Table III shapes (1 GPU): transpose int32 32768^2, sum 32768^2, dot 2^27, matmul 4096^3
    # f2: Jacobi to convergence on the headline grid -- 100 sweeps in blocks of 20, the residual
    # MAXVAL(ABS(u_s - u_{s-1})) fused into each block's last launch and read back by the host
    # (tol = 0: all 100 sweeps run, 5 checks), against the plain 100 sweeps of the headline
    if "f2" in args.rows and N == 1:
        n, sweeps, every = 8192, SWEEPS, 20
        U, W = ftn.FArray.empty((n, n)), ftn.FArray.empty((n, n))
        jacobi_faces(ftn, U, n, n)
        ftn.assign(W, U)
        out = {}

        def solve_step():
            out["r"] = ftn.jacobi_solve(U, W, sweeps, every, 0.0)
        t = timed(torch, solve_step, max(2, steps // 2), 1, ctx["clocks"], dist)
        ns = max(2, steps // 2)
        done, resid, _ = out["r"]
        gl = (n - 2) ** 2 * done * ns / t / 1e9
        rows["f2_jacobi_solve_8192"] = {"value": gl, "unit": "GLUPS", "sweeps_per_call": done,
                                        "check_every": every, "last_residual": resid,
                                        "note": "residual fused into the last launch of each block; one host read "
                                                "per block; compare the headline's plain sweeps"}
        del U, W
        torch.cuda.empty_cache()

    if "paper" in args.rows and N == 1:
        n = 32768
        a = ftn.FArray.empty((n, n), dtype=torch.int32)
        ftn.gen_fill(a, SEED, 1, ftn.GEN_LINEAR)
        r = ftn.FArray.empty((n, n), dtype=torch.int32)
        gbs_row("paper_transpose_int32_32768", 8 * n * n, lambda: ftn.transpose(r, a))
        del a, r
        torch.cuda.empty_cache()
        s = ftn.FArray.empty((n, n))
        ftn.gen_fill(s, SEED, 2, ftn.GEN_U01)
        out = torch.empty((), dtype=torch.float64, device="cuda")
        gbs_row("paper_sum_32768", 8 * n * n, lambda: ftn.sum(s, out))
        del s
        torch.cuda.empty_cache()
        m = 1 << 27
        x, y = ftn.FArray.empty((m,)), ftn.FArray.empty((m,))
        ftn.gen_fill(x, SEED, 3, ftn.GEN_U11)
        ftn.gen_fill(y, SEED, 4, ftn.GEN_U11)
        gbs_row("paper_dot_2^27", 16 * m, lambda: ftn.dot_product(x, y, out))
        del x, y
        k = 4096
        A, B, C = (ftn.FArray.empty((k, k)) for _ in range(3))
        ftn.gen_fill(A, SEED, 5, ftn.GEN_U11)
        ftn.gen_fill(B, SEED, 6, ftn.GEN_U11)
        t = timed(torch, lambda: ftn.matmul(C, A, B), steps, warm, None, None)
        tf = 2.0 * k ** 3 * steps / t / 1e12
        rows["paper_matmul_4096"] = {"value": tf, "unit": "TFLOP/s", "ms": t / steps * 1e3,
                                     "roofline": {"bound": "fp64 tensor (DMMA)", "frac": tf / FP64_PEAK_TFLOPS}}
        del A, B, C
        torch.cuda.empty_cache()
        # jacobi 1024^2 x 10^5 sweeps: the 16 MiB working set stays in L2, so GLUPS only (no HBM fraction)
        nj, sw = 1024, 100000
        U, W = ftn.FArray.empty((nj, nj)), ftn.FArray.empty((nj, nj))
        ftn.gen_fill(U, SEED, 0, ftn.GEN_U01)
        jacobi_faces(ftn, U, nj, nj)
        ftn.assign(W, U)
        t = timed(torch, lambda: ftn.jacobi(U, W, sw), 1, 1, None, None)
        rows["paper_jacobi_1024_1e5"] = {"value": (nj - 2) ** 2 * sw / t / 1e9, "unit": "GLUPS", "ms": t * 1e3,
                                         "roofline": {"bound": "l2-resident (16 MiB working set): not an HBM case",
                                                      "frac": None}}
        del U, W

    # C5: 3-D 7-point Jacobi 2048^3 (slabs of 2048/N planes + halos at N > 1), 100 sweeps per step
    # (an even number of 2-sweep launches, so no single sweep in the plan)
    if "c5" in args.rows:
        n, sweeps = 2048, 100
        probe = ftn.FArray.empty((8, 8, 8))
        T3 = ftn.jacobi_fusion(probe)   # the rank-3 sweeps per launch (3 by default)
        del probe
        free = torch.cuda.mem_get_info()[0]
        plane = n * n
        checksum = None
        if not distmode:
            need = 2 * n ** 3 * 8
            if free > need + (2 << 30):
                U, W = ftn.FArray.empty((n, n, n)), ftn.FArray.empty((n, n, n))
                ftn.gen_fill(U, SEED, 7, ftn.GEN_U01)
                ftn.assign(W, U)
                new = [False]

                def c5_step():
                    new[0] = ftn.jacobi(U, W, sweeps)
                t = timed(torch, c5_step, max(2, steps // 2), 1, ctx["clocks"], dist)
                interior = (n - 2) ** 3
                R = W if new[0] else U
                checksum = c5_checksum(torch, ftn, R, 2, n - 1, None)
                del U, W, R
            else:
                t, interior = None, 0
        else:
            from paper_2409_18824_b200 import dist as D
            halo = 3                                     # 3 halo planes: 3 fused sweeps per exchange
            g0, nl = D.jacobi_slab(n, N, rank, halo=halo)
            U, W = ftn.FArray.empty((n, n, nl)), ftn.FArray.empty((n, n, nl))
            # the global array's values where they live (decomposition-independent input):
            # local plane q holds global plane g0 + q; planes beyond the global array are never read
            q0, q1 = max(0, -g0), min(nl, n - g0)
            ftn.fill(U, 0.0)
            ftn.gen_fill(U.section((1, n), (1, n), (q0 + 1, q1)), SEED, 7, ftn.GEN_U01, t0=(g0 + q0) * plane)
            ftn.assign(W, U)
            new = [False]

            def c5_step():
                new[0] = comm.jacobi(U, W, sweeps, halo=halo)
            t = timed(torch, c5_step, max(2, steps // 2), 1, ctx["clocks"], dist)
            interior = (n - 2) ** 3
            R = W if new[0] else U
            checksum = c5_checksum(torch, ftn, R, halo + 1, nl - halo, comm)
            del U, W, R
        torch.cuda.empty_cache()
        if t:
            ns = max(2, steps // 2)
            gl = interior * sweeps * ns / t / 1e9
            # algorithmic bytes: 16 B per interior point per launch (ftn_jacobi_plan with T = 3:
            # jacobi3d_wr<3>, and jacobi3d_tb2 for the plan's 2-sweep launches; 3-halo slabs at N > 1)
            nl3 = len(ftn.jacobi_plan(sweeps, T3))
            gbs = 16 * interior * nl3 * ns / t / 1e9 / N
            rows["c5_jacobi3d_2048"] = {"value": gl, "unit": "GLUPS", "ms_per_sweep": t / ns / sweeps * 1e3,
                                        "launches_per_step": nl3, "sweeps_per_launch_max": T3,
                                        "roofline": {"bound": "hbm", "achieved_gbs_per_gpu": gbs,
                                                     "frac": gbs / hbm_peak},
                                        "checksum": dict(checksum or {}, sweeps_done=(1 + ns) * sweeps)}

    # f4: pw-advection, three fields (k, j, i) = 2048 x 1024 x 1024 (R#26/R#27); at N > 1
    # every rank owns 1024/N i-planes plus one halo plane per side (inputs do not change
    # between calls, so there is no exchange in the timed loop: weak slabs, no collective)
    if "f4" in args.rows:
        nz, ny, nx = 2048, 1024, 1024
        nxl = nx if N == 1 else nx // N + 2
        need = 6 * nz * ny * nxl * 8
        if torch.cuda.mem_get_info()[0] > need + (2 << 30):
            F = [ftn.FArray.empty((nz, ny, nxl)) for _ in range(3)]
            for q, f in enumerate(F):
                ftn.gen_fill(f, SEED, 50 + q + 3 * rank, ftn.GEN_U11)
            O = [ftn.FArray.empty((nz, ny, nxl)) for _ in range(3)]
            Z = [ftn.FArray.empty((nz,)) for _ in range(4)]
            for q, z in enumerate(Z):
                ftn.gen_fill(z, SEED, 60 + q, ftn.GEN_U11)
            t = timed(torch, lambda: ftn.pw_advection(*O, *F, *Z, 0.1, 0.2), steps, warm, None, dist)
            cells = (nz - 2) * (ny - 2) * (nxl - 2) * N
            gcs = cells * steps / t / 1e9
            gbs = 48 * cells * steps / t / 1e9
            rows["f4_pw_advection_2048x1024x1024"] = {
                "value": gcs, "unit": "Gcells/s", "ms": t / steps * 1e3, "achieved_gbs": gbs,
                "roofline": {"bound": "hbm", "bytes_per_cell": 48, "frac": gbs / N / hbm_peak}}
            del F, O, Z
            torch.cuda.empty_cache()
        # tra-adv (R#28): the NEMO tracer advection, 1024 x 512 x 512, 20 iterations
        # per step.  Algorithmic: 72 B per cell and iteration (md read and written, the seven
        # other 3-D fields read once); the two fused passes move ~115 B (ncu: the horizontal
        # pass writes md6 and zind, the vertical pass reads them back), which the line states
        ni, nj, nk, iters = 1024, 512 // N if N > 1 else 512, 512, 20
        if torch.cuda.mem_get_info()[0] > 14 * ni * nj * nk * 8 + (2 << 30):
            D = [ftn.FArray.empty((ni, nj, nk)) for _ in range(8)]
            for q, d in enumerate(D[:5]):
                ftn.gen_fill(d, SEED, 70 + q + 10 * rank, ftn.GEN_U11)
            for q, d in enumerate(D[5:]):
                ftn.gen_fill(d, SEED, 80 + q, ftn.GEN_U01)
            D2 = [ftn.FArray.empty((ni, nj)) for _ in range(3)]
            for q, d in enumerate(D2):
                ftn.gen_fill(d, SEED, 90 + q, ftn.GEN_U01)
            RZ = ftn.FArray.empty((nk,))
            ftn.gen_fill(RZ, SEED, 95, ftn.GEN_U01)
            t = timed(torch, lambda: ftn.tra_adv(*D, *D2, RZ, iters), max(2, steps // 4), 1, None, dist)
            ns = max(2, steps // 4)
            cells = ni * nj * nk * N
            gcs = cells * iters * ns / t / 1e9
            gbs = 72 * cells * iters * ns / t / 1e9
            rows["f4_tra_adv_1024x512x512_x20"] = {
                "value": gcs, "unit": "Gcell-iterations/s", "ms_per_step": t / ns * 1e3, "achieved_gbs": gbs,
                "note": ("one GPU" if N == 1 else
                         "N independent jj-slabs without halo exchange: aggregate throughput of replicas, "
                         "not a distributed tra-adv (its fields change every iteration)"),
                "roofline": {"bound": "hbm", "algorithmic_bytes_per_cell_iteration": 72,
                             "implementation_bytes_per_cell_iteration": 115, "frac": gbs / N / hbm_peak,
                             "frac_of_moved_bytes": 115 / 72 * gbs / N / hbm_peak}}
            del D, D2, RZ
            torch.cuda.empty_cache()
    # SURVEY §8(e) strong scaling, predicted on one GPU: each rank's share at p = 8 run alone
    # (no exchange), against the same kernel on the whole 1-GPU problem: the compute side of
    # the 1 -> 8 efficiency (wave quantisation, halo recompute, shorter streams)
    if "shares" in args.rows and N == 1:
        P8 = 8
        shares = {}
        # C3: c(:, J_r) = MATMUL(a, b(:, J_r)), 8192 x 8192 x 1024 (512 tiles of 128 x 128)
        n = 8192
        A, B, C = ftn.FArray.empty((n, n)), ftn.FArray.empty((n, n // P8)), ftn.FArray.empty((n, n // P8))
        ftn.gen_fill(A, SEED, 1, ftn.GEN_U11)
        ftn.gen_fill(B, SEED, 2, ftn.GEN_U11)
        t = timed(torch, lambda: ftn.matmul(C, A, B), steps, warm, None, None)
        tf = 2.0 * n * n * (n // P8) * steps / t / 1e12
        shares["c3_matmul_share_8192x8192x1024"] = {"value": tf, "unit": "TFLOP/s", "ms": t / steps * 1e3,
                                                    "frac_of_fp64_peak": tf / FP64_PEAK_TFLOPS}
        if "c3_matmul_8192" in rows:
            shares["c3_matmul_share_8192x8192x1024"]["vs_full_problem"] = tf / rows["c3_matmul_8192"]["value"]
        del A, B, C
        torch.cuda.empty_cache()
        # C5: a rank's slab 2048 x 2048 x (256 owned + 2) planes, 100 sweeps (the local compute of
        # one rank; the 3 halo planes per side only add the exchange)
        n, sw = 2048, 100
        nl = (n - 2) // P8 + 1 + 2
        U, W = ftn.FArray.empty((n, n, nl)), ftn.FArray.empty((n, n, nl))
        ftn.gen_fill(U, SEED, 7, ftn.GEN_U01)
        ftn.assign(W, U)
        t = timed(torch, lambda: ftn.jacobi(U, W, sw), 2, 1, None, None)
        gl = (n - 2) ** 2 * (nl - 2) * sw * 2 / t / 1e9
        shares["c5_jacobi3d_slab_2048x2048x258"] = {"value": gl, "unit": "GLUPS", "ms": t / 2 * 1e3}
        if "c5_jacobi3d_2048" in rows:
            shares["c5_jacobi3d_slab_2048x2048x258"]["vs_full_problem"] = gl / rows["c5_jacobi3d_2048"]["value"]
        del U, W
        torch.cuda.empty_cache()
        # C4: a rank's slab 1024 x 1024 x 128 (SUM and b*c+d)
        arrs = [ftn.FArray.empty((1024, 1024, 1024 // P8)) for _ in range(4)]
        for k, a in enumerate(arrs):
            ftn.gen_fill(a, SEED, 10 + k, ftn.GEN_U01)
        b, c, d, r = arrs
        n_el = 1024 * 1024 * (1024 // P8)
        out = torch.empty((), dtype=torch.float64, device="cuda")
        for name, nb, fn, full in (("c4_sum_share_1024x1024x128", 8 * n_el, lambda: ftn.sum(b, out), "c4_sum"),
                                   ("c4_muladd_share_1024x1024x128", 32 * n_el, lambda: ftn.muladd(r, b, c, d, contract=CONTRACT),
                                    "c4_muladd_r=b*c+d")):
            t = timed(torch, fn, steps, warm, None, None)
            g = nb * steps / t / 1e9
            shares[name] = {"value": g, "unit": "GB/s", "ms": t / steps * 1e3, "frac": g / hbm_peak}
            if full in rows:
                shares[name]["vs_full_problem"] = g / rows[full]["value"]
        del arrs, b, c, d, r
        torch.cuda.empty_cache()
        rows["p8_shares_on_one_gpu"] = shares

    return rows


# ----------------------------------------------------------------------------------- CPU oracle
def cpu_oracle_jacobi(budget_s=12.0, max_sweeps=100):
    """The oracle's Jacobi (oracle/ftn_oracle.c, OpenMP over independent rows) on the full 8192^2
    grid of the headline workload, for as many sweeps as fit the budget."""
    import numpy as np
    import oracle
    import synth
    n = 8192
    u = synth.jacobi_init((n, n))
    w = u.copy(order="F")
    U, Wd = oracle.FArray(u), oracle.FArray(w)
    t0 = time.perf_counter()
    oracle.jacobi(U, Wd, 1, 0.25)
    t1 = time.perf_counter() - t0
    sweeps = int(max(1, min(max_sweeps, budget_s / max(t1, 1e-6))))
    t0 = time.perf_counter()
    oracle.jacobi(U, Wd, sweeps, 0.25)
    t = time.perf_counter() - t0
    cores = len(os.sched_getaffinity(0))
    threads = int(os.environ.get("OMP_NUM_THREADS", cores))
    # the plain single-thread oracle: one full sweep
    prev = oracle.set_threads(1)
    t0 = time.perf_counter()
    oracle.jacobi(U, Wd, 1, 0.25)
    t1s = time.perf_counter() - t0
    oracle.set_threads(prev)
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            model = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), "")
    except OSError:
        pass
    del u, w, np
    return {"value": (n - 2) ** 2 * sweeps / t / 1e9, "unit": "GLUPS", "cores": threads, "kind": "oracle",
            "sample": f"full 8192^2 grid, {sweeps} of the 100 sweeps ({t:.1f} s), OpenMP over rows",
            "single_thread": {"value": (n - 2) ** 2 / t1s / 1e9, "unit": "GLUPS",
                              "sample": f"one full 8192^2 sweep ({t1s:.2f} s), 1 thread"},
            "cpu_model": model}


def run_reference(args):
    """--impl reference: the oracle (oracle/ftn_oracle.c, OpenMP over independent rows) timed on
    the host cores on the SAME workload and config as the headline: each step is the full 100
    sweeps of the 8192^2 grid (N = 1) or of the weak-scaled global grid 8192 x (8192 N + 2) that
    the N GPUs advance together (N > 1).  Rank 0 alone runs it; no reference code base exists."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import numpy as np
    import oracle
    import synth
    N = max(1, args.gpus)
    n, sweeps = 8192, SWEEPS
    n2 = n if N == 1 else n * N + 2
    if MODE == "closed":
        u = np.asfortranarray(np.add.outer(np.arange(n, dtype=np.float64), n * np.arange(n2, dtype=np.float64)))
    else:
        u = synth.jacobi_init((n, n2), seed=SEED)
        if MODE == "intvalued":
            u[1:-1, 1:-1] = synth.farray((n - 2, n2 - 2), seed=SEED, mode=synth.INT8, array_id=0)
    w = u.copy(order="F")
    U, Wd = oracle.FArray(u), oracle.FArray(w)
    for _ in range(args.warmup):
        oracle.jacobi(U, Wd, 1, 0.25)        # warm-up: one sweep each (page-in, thread start)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.jacobi(U, Wd, sweeps, 0.25)   # one step = the full 100 sweeps
    t = time.perf_counter() - t0
    interior = (n - 2) * (n2 - 2)
    glups = interior * sweeps * args.steps / t / 1e9
    cores = int(os.environ.get("OMP_NUM_THREADS", len(os.sched_getaffinity(0))))
    cpu = {"value": glups, "unit": "GLUPS", "cores": cores, "kind": "oracle",
           "sample": f"the whole workload: {args.steps} steps of {sweeps} sweeps of the {n}x{n2} grid, OpenMP over rows"}
    line = {"impl": "reference", "metric": metric(), "value": glups, "unit": "GLUPS", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(config(), parallelism=f"slab{N}" if N > 1 else "1 GPU",
                           global_grid=f"{n}x{n2}"),
            "cpu_baseline": cpu,
            "e2e": {"value": glups, "unit": "GLUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    del np
    print(json.dumps(line), flush=True)
    return 0


SWEEPS = 100          # sweeps per step of the C2 headline (BASELINE: 100; --sweeps)
MODE = "random"       # C2 input (--mode): random U[0,1) interior | closed (a harmonic field) | intvalued
CONTRACT = False      # MULADD rows as one fused multiply-add (--contract, R#6)


def metric():
    return f"Jacobi GLUPS (2-D 5-point, real(8) 8192^2, {SWEEPS} sweeps per step)"


def config():
    c = {"workload": f"BASELINE configs[1]: 2-D 5-point Jacobi stencil, real(8) 8192x8192, {SWEEPS} sweeps",
         "l2": "working set 2 x 512 MiB > 126 MB L2 (no flush needed)", "seed": SEED}
    if MODE != "random":
        c["input_mode"] = MODE
    return c


HBM_SPEC_GBS = 8000.0   # B200 datasheet HBM3e bandwidth (BASELINE's ~8 TB/s)


def in_run_ceilings(rows, hbm_peak):
    """the HBM ceilings measured in this run beside the denominators --
    read-only (C4 SUM, 8 B/elem), copy (r = b, 16 B/elem), triad (b*c+d, 32 B/elem), the
    MEASURED_PEAKS copy figure and the 8 TB/s spec."""
    get = lambda k: rows.get(k, {}).get("value") if isinstance(rows.get(k), dict) else None  # noqa: E731
    return {"read_gbs": get("c4_sum"), "copy_gbs": get("hbm_copy_r=b"), "triad_gbs": get("c4_muladd_r=b*c+d"),
            "measured_peaks_copy_gbs": hbm_peak, "spec_gbs": HBM_SPEC_GBS, "unit": "GB/s"}


def fused_kernel_name(sizes):
    """The 2-D kernels of a launch plan ({sweeps per launch: count}): jacobi2d_wq<k> for k >= 7
    (and any k under FTN_WF_WQ=1), jacobi2d_wf<k> for 2 <= k <= 6, jacobi2d_tma for k = 1."""
    wq_all = os.environ.get("FTN_WF_WQ", "0") not in ("", "0")
    names = []
    for k in sorted((int(x) for x in sizes), reverse=True):
        names.append("jacobi2d_tma" if k == 1 else (f"jacobi2d_wq<{k}>" if k >= 7 or wq_all else f"jacobi2d_wf<{k}>"))
    return " + ".join(names)


def traffic_from_profiles():
    p = os.path.join(ROOT, "profiles", "jacobi2d_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get("dram_bytes_per_launch")
    except Exception:
        return None


def main():
    global SEED, SWEEPS, MODE, CONTRACT
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ftn", choices=["ftn", "reference"])
    ap.add_argument("--rows", default="c1,c4,c3,f2,paper,c5,f4,shares", help="comma list of extra rows, or 'none'")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--dist", action="store_true",
                    help="use the multi-GPU code path (NCCL communicator, ftn_jacobi_dist) even at N=1")
    # SURVEY §5 bench CLI
    ap.add_argument("--config", default=None,
                    help="which SURVEY §8 configs run beside the C2 headline: a comma list of C1, C3, C4, C5, P "
                         "(the paper's shapes), F2 (solve to convergence), F4, SHARES, or ALL / NONE (overrides --rows)")
    ap.add_argument("--seed", type=int, default=SEED, help="generator seed of every synthetic input (18824)")
    ap.add_argument("--sweeps", type=int, default=SWEEPS, help="sweeps per step of the C2 headline (100)")
    ap.add_argument("--mode", choices=["random", "closed", "intvalued"], default=MODE,
                    help="C2 input: U[0,1) interior (BASELINE), the harmonic field (i-1) + 8192 (j-1) (a fixed "
                         "point, checked bit for bit after the timed region), or integers in [-8, 8]")
    ap.add_argument("--contract", action="store_true",
                    help="the MULADD rows as one fused multiply-add per element (R#6)")
    args = ap.parse_args()
    SEED, SWEEPS, MODE, CONTRACT = args.seed, args.sweeps, args.mode, args.contract
    if SWEEPS < 1:
        ap.error("--sweeps must be >= 1")
    if args.config is not None:
        groups = {"C1": "c1", "C3": "c3", "C4": "c4", "C5": "c5", "P": "paper", "F2": "f2", "F4": "f4",
                  "SHARES": "shares"}
        sel = [c.strip().upper() for c in args.config.split(",") if c.strip()]
        if sel in (["ALL"],):
            args.rows = ",".join(groups.values())
        elif sel in (["NONE"], ["C2"]):
            args.rows = "none"
        else:
            bad = [c for c in sel if c not in groups and c != "C2"]
            if bad:
                ap.error(f"--config: unknown {bad}; choose from C1..C5, P, F2, F4, SHARES, ALL, NONE")
            args.rows = ",".join(groups[c] for c in sel if c in groups) or "none"
    args.rows = [] if args.rows == "none" else args.rows.split(",")
    if args.impl == "reference":
        return run_reference(args)

    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    ctx = {"world": world, "rank": rank, "dist": None, "force_dist": args.dist}
    from paper_2409_18824_b200 import ftn
    if world > 1 or args.dist:
        import torch.distributed as dist
        if not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        ctx["dist"] = dist
        ctx["comm"] = ftn.Comm.from_torch_distributed(local)
    clocks = ClockSampler(local)
    clocks.start()
    ctx["clocks"] = clocks
    hbm_peak, peak_src = load_peaks()

    head = bench_jacobi2d(torch, ftn, args, ctx)
    try:
        rows = bench_rows(torch, ftn, args, ctx, hbm_peak) if args.rows else {}
    except Exception as e:  # a failing extra row must not cost the headline line (1 GPU: no peers to desync)
        if world > 1:
            raise
        print(f"bench rows failed: {e!r}", file=sys.stderr)
        rows = {"error": repr(e)[:300]}
    clk = clocks.stop()

    if rank == 0:
        cpu = None if args.no_cpu or world > 1 else cpu_oracle_jacobi()
        # achieved_gbs is per GPU already (one rank's slab bytes per launch / max-over-ranks time)
        frac = head["achieved_gbs"] / hbm_peak
        line = {
            "metric": metric(), "value": head["value"], "unit": "GLUPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
            "ms_per_step_min": head["ms_step_min"], "ms_per_step_median": head["ms_step_median"],
            "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(config(), parallelism=f"slab{world}" if world > 1 else "1 GPU",
                           global_grid=f"8192x{8192 * world + (2 if world > 1 else 0)}"),
            "e2e": head.get("e2e"),
            **({"check": head["check"]} if "check" in head else {}),
            "gpu_launches": head["launches"],
            "roofline": {"bound": "hbm",
                         "kernel": fused_kernel_name(head["plan"]["sweeps_per_launch"]),
                         "achieved": head["achieved_gbs"],
                         "peak": hbm_peak, "unit": "GB/s", "frac": frac, "peak_source": peak_src,
                         "traffic": traffic_from_profiles(),
                         "algorithmic_bytes_per_launch": head["per_launch_bytes"],
                         "launch_plan_per_step": head["plan"],
                         "note": ("16 B per interior point per launch (u read once, result written once); a fused "
                                  "launch performs T sweeps (temporal blocking), so GLUPS can exceed the "
                                  "single-sweep roofline 6556/16 = 410 GLUPS; time = all launches of the timed region")},
            "cpu_baseline": cpu,
            "clocks": clk,
            "hbm_ceilings_in_run": in_run_ceilings(rows, hbm_peak),
            "rows": rows,
        }
        print(json.dumps(line), flush=True)
    if ctx.get("comm") is not None:
        ctx["comm"].destroy()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
