#!/usr/bin/env python
"""bench.py — sBMDS hot path on B200 (BASELINE.json metric at config 4).

Default workload: BASELINE.json configs[3] (torus 1200x1500, n = 1,800,000, l = 50,000,
k = 32, fp32 D_ll 10 GB, m = 3, block 16, exactly 50 subspace iterations). A step is one
full sbmds_eigs solve (50 applies of -1/2 J S D S^T J + Cholesky-QR + Rayleigh-Ritz +
embedding) on inputs already resident in HBM; value = operator applies per second over
all ranks. Inputs (10 GB D) are far larger than the 126 MB L2, so no flush is needed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (N independent replicas, weak scaling)

Rank 0 prints ONE JSON line. --impl reference times the fp64 CPU oracle (the only
baseline that exists: the paper ships no code) on the same workload and unit.
"""
from __future__ import annotations

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

METRIC = "sBMDS operator applies/s & HBM GB/s vs peak; top-p MDS time at n=1.8M,l=50k"
UNIT = "applies/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--iters", type=int, default=50, help="subspace iterations per eigs step")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--mode", default="eigs", choices=["eigs", "apply"],
                    help="eigs: one step = one 50-iteration sbmds_eigs (the headline); apply: one step = "
                         "one standalone sbmds_apply of an n x b block (SURVEY §8(d) per-config lines)")
    ap.add_argument("--b", type=int, default=0, help="apply mode: block width (default: the config's block)")
    ap.add_argument("--k5", type=int, default=16, help="config 5: nonzeros per row of S (8, 16, 64)")
    ap.add_argument("--shard", action="store_true",
                    help="eigs mode under torchrun: one sharded solve over all ranks (rows of S and "
                         "tiles of D per rank, NCCL allreduces; strong scaling) instead of replicas")
    return ap.parse_args()


# ------------------------------------------------------------------------------ distributed
def dist_setup(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        backend = "nccl" if args.impl == "ours" else "gloo"
        if backend == "nccl":
            import torch
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, ws: int, device=None) -> float:
    """Max of a per-rank device time over all ranks (the slowest replica sets the pace)."""
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_throughput(ws: int, units_per_rank: float, seconds_max: float) -> float:
    """Whole-job value: the units all ranks processed / the max-over-ranks time."""
    return ws * units_per_rank / seconds_max


def load_problem(cfg: int, ws: int, rank: int, k5: int = 16):
    """Rank 0 generates (and caches) first; the other ranks then load the cache."""
    from gen import configs
    if rank == 0:
        p = configs.config(cfg, k5=k5)
        barrier(ws)
    else:
        barrier(ws)
        p = configs.config(cfg, k5=k5)
    return p


def nnz_per_row(p) -> float:
    return round(p.nnz / p.n, 3)


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    """NVML SM clock + throttle reasons sampled every 100 ms while active."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks",
               0x10: "sync_boost"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                fn = getattr(self.nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    self.nv.nvmlDeviceGetCurrentClocksThrottleReasons
                self.reasons |= int(fn(self.h))
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        if self.nv:
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml_unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(v for k, v in self.REASONS.items() if self.reasons & k),
                "samples": len(self.samples)}


# ------------------------------------------------------------------------------ our arm
def algorithmic_bytes(p, b):
    """Bytes one apply must move: full fp32 D once, S via
    CSR and CSC (8 B per nnz each), row/col pointers, X read + Y written."""
    return 4 * p.l * p.l + 16 * p.nnz + 4 * (p.n + 1) + 4 * (p.l + 1) + 8 * p.n * b


DSTREAM_KERNELS = {1: "k_dstream_ffma", 2: "k_dstream_tc (tcgen05 3xTF32, full D)",
                   3: "k_dstream_sym8 (tcgen05 kind::i8, 24-bit fixed point, symmetric half of D)",
                   4: "k_dstream_pair (tcgen05 2xFP16, symmetric half of D, CTA pairs)"}


def log(msg):
    if os.environ.get("SBMDS_BENCH_TRACE"):
        sys.stderr.write(f"[bench {time.strftime('%H:%M:%S')}] {msg}\n")
        sys.stderr.flush()


def run_ours(args, ws, rank, local):
    import torch
    from paper_1705_10887_b200 import from_problem, launch_count
    torch.cuda.set_device(local)
    p = load_problem(args.config, ws, rank, args.k5)
    if args.mode == "apply":
        return run_apply_mode(args, ws, rank, local, p)
    m, b, iters = p.m, p.block, args.iters
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"

    log("inputs ready")
    if args.shard:
        # one solve over all ranks: rank g holds rows split_rows(.)[g] and tile range g of D; the
        # NCCL id of the library's communicator travels over torch.distributed
        import torch.distributed as dist
        from paper_1705_10887_b200.sbmds import nccl_unique_id, shard_from_problem
        h = shard_from_problem(p, rank, ws)
        idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
        if ws > 1:
            dist.broadcast(idt, 0)
        h.attach_nccl(bytes(idt.cpu().numpy().tobytes()))
        args.no_e2e = True
    else:
        h = from_problem(p, device="cuda")
    log("handle created")
    st = torch.cuda.current_stream()
    V = torch.empty((h.n, m), device="cuda")
    Z = torch.empty((h.n, m), device="cuda")

    def step():
        return h.eigs(m, b, max_iters=iters, tol=0.0, seed=0, V=V, Z=Z)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    log("warmup done")
    barrier(ws)
    h.set_option("profile", 1 << 2)          # CUDA events around the D-stream kernel only
    h.set_option("profile_reset", 1)
    n0 = launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        barrier(ws)
        e0.record(st)
        infos = [step()[3] for _ in range(args.steps)]
        e1.record(st)
        torch.cuda.synchronize()
    log("timed region done")
    n_launch = launch_count() - n0
    ms = e0.elapsed_time(e1)
    ds_ns, ds_n = h.stat("dstream_ns"), h.stat("dstream_launches")
    ds_path, ds_bytes = h.stat("dstream_path"), h.stat("dstream_bytes")   # per launch, DESIGN.md §4
    h.set_option("profile", 0)
    ms_max = max_over_ranks(ms, ws, device="cuda")
    applies = sum(i["n_applies"] for i in infos)
    # replicas: every rank's solve counts; a sharded solve is one solve over all ranks
    value = job_throughput(1 if args.shard else ws, applies, ms_max / 1e3)
    ds_avg_s = ds_ns / max(ds_n, 1) / 1e9
    ds_gbs = ds_bytes / ds_avg_s / 1e9
    apply_gbs = algorithmic_bytes(p, b) * applies / (ms / 1e3) / 1e9
    eigs_s = ms / 1e3 / args.steps

    # parity spot check at full size: eigenvalues of the timed solves are deterministic
    lam, _, _, info = step()

    # the second-largest kernel family, outside the timed region: the tensor-core sparse step
    # (A5 + Grams + next A2), CUDA events around its launches during one more solve
    sparse = None
    if h.stat("sp8_state") == 1:
        # (events around every kernel family: with events only around this kernel its programmatic
        # early start would count the previous kernel's tail; per-family times per iteration ride along)
        h.set_option("profile", (1 << 10) - 1)
        h.set_option("profile_reset", 1)
        n8 = h.stat("gram8_launches")
        step()
        torch.cuda.synchronize()
        n8 = h.stat("gram8_launches") - n8
        sp_ns, sp_n = h.stat("csr_ns"), h.stat("csr_launches")
        fams = {"landmark reduce + R^-1 fold + Y1 digits": "csc", "D stream": "dstream",
                "D-partial reduce + t + Y2 digits": "dreduce", "sparse step": "csr", "Rayleigh-Ritz": "rr"}
        fam_ms = {k: round(h.stat(f + "_ns") / 1e6 / iters, 5) for k, f in fams.items()}
        h.set_option("profile", 0)
        slots = h.stat("sp8_slots")
        # bytes the step must move per launch: the S images once, Y written once (n x b fp32), the
        # T partials written (one fp32 row of b per 128-row dictionary entry) and the gathered Y2
        # digit rows (48 B per entry)
        sp_bytes = h.stat("sp8_bytes") + 4 * p.n * b + (4 * b + 48) * slots
        sp_s = sp_ns / max(sp_n, 1) / 1e9
        sparse = {"kernel": "k_sp8_step (tcgen05 kind::i8 on dense 128-row images of S)", "launches": int(sp_n),
                  "avg_launch_ms": sp_s * 1e3, "algorithmic_bytes_per_launch": int(sp_bytes),
                  "achieved_gbs": sp_bytes / sp_s / 1e9, "frac_of_hbm_peak": sp_bytes / sp_s / 1e9 / hbm_peak,
                  "int8_gram_launches": int(n8),
                  "family_ms_per_iteration": fam_ms}

    # ---- the public sbmds_apply on its own (north_star's target names "the
    # operator apply"), outside the timed region: CUDA events around 20 calls on resident X, Y
    standalone = None
    if not args.shard:
        from gen import configs
        Xa = torch.from_numpy(configs.x_block(p.n, b, seed=3)).cuda()
        Ya = torch.empty_like(Xa)
        for _ in range(3):
            h.apply(Xa, out=Ya)
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        ea.record(st)
        for _ in range(20):
            h.apply(Xa, out=Ya)
        eb.record(st)
        torch.cuda.synchronize()
        a_s = ea.elapsed_time(eb) / 1e3 / 20
        a_bytes = h.stat("dstream_bytes") + 16 * p.nnz + 4 * (p.n + 1) + 4 * (p.l + 1) + 8 * p.n * b
        standalone = {"call": "sbmds_apply (n x b block, device X and Y)", "b": b, "ms_per_apply": a_s * 1e3,
                      "applies_per_s": 1.0 / a_s, "algorithmic_bytes_per_apply": int(a_bytes),
                      "achieved_gbs": a_bytes / a_s / 1e9, "frac_of_hbm_peak": a_bytes / a_s / 1e9 / hbm_peak,
                      "bytes_basis": "D stream's bytes + S through CSR and CSC (16 B per nonzero) + pointers + X, Y",
                      "on_tensor_core_sparse_kernels": bool(h.stat("sp8_apply_launches") > 0)}
        del Xa, Ya

    # ---- end to end through the C ABI from pinned HOST buffers (create + eigs + D2H)
    e2e = None
    if not args.no_e2e:
        from paper_1705_10887_b200 import Sbmds
        rp = torch.from_numpy(np.ascontiguousarray(p.row_ptr, dtype=np.int64)).pin_memory()
        ci = torch.from_numpy(np.ascontiguousarray(p.col_idx)).pin_memory()
        vv = torch.from_numpy(p.val32()).pin_memory()
        Dh = torch.from_numpy(p.D).pin_memory()
        Vh = torch.empty((p.n, m)).pin_memory()
        Zh = torch.empty((p.n, m)).pin_memory()
        del h
        torch.cuda.empty_cache()
        times = []
        log("e2e start")
        for s in range(args.e2e_steps + 1):
            a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record(st)
            t_a = time.perf_counter()
            with Sbmds(p.n, p.l, rp, ci, vv, Dh) as hh:
                d_h2d = hh.stat("h2d_bytes")      # D bytes create moved (block upper triangle)
                t_b = time.perf_counter()
                hh.eigs(m, b, max_iters=iters, tol=0.0, seed=0, V=Vh, Z=Zh)
                t_c = time.perf_counter()
            z.record(st)
            torch.cuda.synchronize()
            log(f"e2e step {s}: create {t_b - t_a:.3f} s, eigs {t_c - t_b:.3f} s, "
                f"destroy {time.perf_counter() - t_c:.3f} s (host clocks)")
            if s > 0:                       # first one warms allocator / tensor maps
                times.append(a.elapsed_time(z) / 1e3)
            log(f"e2e step {s}: {a.elapsed_time(z) / 1e3:.3f} s")
        # median over the timed steps: create's host-link transfer of 5.5 GB occasionally runs
        # several times slower on the shared GPU hosts (measured 0.11-0.75 s for the same call)
        t_e2e = max_over_ranks(float(np.median(times)), ws, device="cuda")
        h2d = d_h2d + 8 * (p.n + 1) + 8 * p.nnz   # D (upper strips) + int64 row_ptr + int32 col + f32 val
        d2h = 8 * m + 2 * p.n * m * 4
        e2e = {"value": job_throughput(ws, iters, t_e2e), "unit": UNIT, "seconds_per_solve": t_e2e,
               "seconds_each_step": [round(x, 4) for x in times], "aggregate": "median of the steps",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "includes": "sbmds_create from pinned host CSR + D (H2D of S and of D's block upper "
                           "triangle, CSC and row-block builds) + sbmds_eigs (D pack + 50 iters) + V, Z, "
                           "eigenvalues to host + destroy"}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(p)

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong" if args.shard else "weak", "vs_baseline": None,
        "dtype": {3: "f32 (D Y1 as 24-bit fixed point on int8 tensor cores, exact int32 accumulate; DESIGN.md §4)",
                  4: "f32 (D Y1 as a 2xfp16 split, fp32 accumulate; DESIGN.md §4)"}.get(ds_path, "f32"),
        "data": "synthetic (seeded torus mesh stand-in for Dragon1800k; DESIGN.md §3)",
        "config": {"workload": f"config {args.config}: {p.name}", "n": p.n, "l": p.l, "nnz_per_row": nnz_per_row(p),
                   "nnz": p.nnz, "block": b, "m": m, "iters_per_step": iters,
                   "parallelism": f"sharded x{ws} (rows of S, tiles of D; NCCL)" if args.shard else f"replicas x{ws}",
                   "l2": "inputs (10 GB D) >> 126 MB L2, no flush"},
        "top_p_mds_seconds": eigs_s,
        "apply_full_d_equivalent_gbs": apply_gbs,   # SURVEY §8(d) full-D bytes per apply / apply time
        "eigenvalues": [float(x) for x in lam],
        "max_residual": info["max_residual"], "orth_error": info["orth_error"],
        "roofline": {"bound": "hbm", "achieved": ds_gbs, "peak": hbm_peak, "unit": "GB/s",
                     "frac": ds_gbs / hbm_peak, "traffic": load_traffic(ds_path),
                     "kernel": DSTREAM_KERNELS.get(ds_path, str(ds_path)), "launches": ds_n,
                     "avg_launch_ms": ds_avg_s * 1e3, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": ds_bytes,
                     "full_d_equivalent_gbs": 4 * p.l * p.l / ds_avg_s / 1e9},
        "gpu_launches": int(n_launch),
        "clocks": clk.summary(),
    }
    if sparse:
        out["sparse_step"] = sparse
    if standalone:
        out["standalone_apply"] = standalone
    if e2e:
        out["e2e"] = e2e
    if cpu:
        out["cpu_baseline"] = cpu
    return out


def run_apply_mode(args, ws, rank, local, p):
    """One step = one standalone sbmds_apply (the public call) of an n x b block on HBM-resident
    inputs: the per-config operator-apply lines of SURVEY §8(d) (configs 3, 4 and the config-5
    sweep). Roofline on the whole apply: the bytes the path it takes must move (its D stream's
    bytes + S via CSR and CSC + X, Y + pointers) over the apply time; the D stream alone as in the
    eigs mode."""
    import torch
    from gen import configs
    from paper_1705_10887_b200 import from_problem, launch_count
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    b = args.b or p.block or 16
    h = from_problem(p, device="cuda")
    X = torch.from_numpy(configs.x_block(p.n, b, seed=3)).cuda()
    Y = torch.empty_like(X)
    st = torch.cuda.current_stream()
    for _ in range(max(3, args.warmup)):
        h.apply(X, out=Y)
    torch.cuda.synchronize()
    barrier(ws)
    h.set_option("profile", 1 << 2)
    h.set_option("profile_reset", 1)
    n0 = launch_count()
    steps = max(args.steps, 20)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        barrier(ws)
        e0.record(st)
        for _ in range(steps):
            h.apply(X, out=Y)
        e1.record(st)
        torch.cuda.synchronize()
    n_launch = launch_count() - n0
    ms = e0.elapsed_time(e1)
    ds_ns, ds_n = h.stat("dstream_ns"), h.stat("dstream_launches")
    ds_path, ds_bytes = h.stat("dstream_path"), h.stat("dstream_bytes")
    h.set_option("profile", 0)
    sp8_path = h.stat("sp8_apply_launches") > 0
    sp8_t = h.stat("sp8_apply_t_launches") > 0
    ms_max = max_over_ranks(ms, ws, device="cuda")
    apply_s = ms / 1e3 / steps
    path_bytes = ds_bytes + 16 * p.nnz + 4 * (p.n + 1) + 4 * (p.l + 1) + 8 * p.n * b
    ds_s = ds_ns / max(ds_n, 1) / 1e9
    return {
        "metric": "sBMDS operator applies/s (standalone sbmds_apply)", "value": job_throughput(ws, steps, ms_max / 1e3),
        "unit": "applies/s", "n_gpus": ws, "steps": steps, "warmup": max(3, args.warmup),
        "ms_per_step": ms_max / steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"config {args.config}: {p.name}", "mode": "apply", "n": p.n, "l": p.l,
                   "nnz_per_row": nnz_per_row(p), "b": b, "parallelism": f"replicas x{ws}",
                   "l2": "no flush: S, D and X, Y exceed the 126 MB L2 at configs 3-5"},
        "roofline": {"bound": "hbm", "achieved": path_bytes / apply_s / 1e9, "peak": hbm_peak, "unit": "GB/s",
                     "frac": path_bytes / apply_s / 1e9 / hbm_peak, "traffic": None,
                     "kernel": "whole apply (" + DSTREAM_KERNELS.get(ds_path, str(ds_path)) + " + " +
                               ("k_sp8_step T-only / N-only on the digit images of S" if sp8_path else "CSC/CSR SpMMs") + ")",
                     "algorithmic_bytes_per_launch": int(path_bytes),
                     "bytes_basis": "D stream's bytes + S once through CSR and once through CSC (16 B per nonzero) + "
                                    "pointers + X, Y; the tensor-core sparse path reads its images (sparse_image_bytes, "
                                    "twice per apply) instead of CSR/CSC and is charged the same algorithmic bytes"},
        "sparse_path": {"a5_on_tensor_cores": bool(sp8_path), "a2_on_tensor_cores": bool(sp8_t),
                        "sparse_image_bytes": int(h.stat("sp8_bytes")) if sp8_path else 0,
                        "x_fallbacks": int(h.stat("x_fallbacks"))},
        "dstream": {"kernel": DSTREAM_KERNELS.get(ds_path, str(ds_path)), "avg_launch_ms": ds_s * 1e3,
                    "bytes_per_launch": ds_bytes, "gbs": ds_bytes / ds_s / 1e9, "frac": ds_bytes / ds_s / 1e9 / hbm_peak},
        "apply_full_d_equivalent_gbs": algorithmic_bytes(p, b) / apply_s / 1e9,
        "gpu_launches": int(n_launch), "clocks": clk.summary(),
    }


def load_traffic(path_id):
    """DRAM bytes per launch of the D-stream kernel from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "dstream_traffic.json")
    try:
        d = json.load(open(path))
        return d.get("by_path", {}).get(str(path_id), d.get("dram_bytes_per_launch") if path_id == 2 else None)
    except Exception:
        return None


# ------------------------------------------------------------------------------ oracle arms
def cpu_baseline(p, reps: int = 1):
    """The fp64 oracle (oracle/sbmds_oracle.apply, as it stands) on this host's cores."""
    from gen import configs
    from oracle import sbmds_oracle as O
    S = O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val32())
    X = configs.x_block(p.n, p.block, seed=1)
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        O.apply(S, p.D, X)
        t.append(time.perf_counter() - t0)
    sec = float(np.median(t))
    return {"value": 1.0 / sec, "unit": UNIT, "cores": len(os.sched_getaffinity(0)), "kind": "oracle",
            "sample": f"{reps} fp64 oracle apply (b={p.block}) of the full config-{4 if p.n == 1800000 else '?'} "
                      f"operator, median wall {sec:.2f} s"}


def run_reference(args, ws, rank):
    if rank != 0:
        return None
    from gen import configs
    from oracle import sbmds_oracle as O
    p = configs.config(args.config)
    S = O.csr(p.n, p.l, p.row_ptr, p.col_idx, p.val32())
    X = configs.x_block(p.n, p.block, seed=1)
    steps, warm = max(1, min(args.steps, 5)), min(args.warmup, 1)
    for _ in range(warm):
        O.apply(S, p.D, X)
    t0 = time.perf_counter()
    for _ in range(steps):
        O.apply(S, p.D, X)
    sec = (time.perf_counter() - t0) / steps
    v = 1.0 / sec
    cores = len(os.sched_getaffinity(0))
    sample = (f"fp64 oracle apply (b={p.block}) of config {args.config}, {steps} timed + {warm} warm-up "
              f"(capped at 5 + 1 to bound the run)")
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws,
            "steps": steps, "warmup": warm, "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"config {args.config}: {p.name}", "n": p.n, "l": p.l, "block": p.block},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    ws, rank, local = dist_setup(args)
    if args.impl == "reference":
        out = run_reference(args, ws, rank)
    else:
        out = run_ours(args, ws, rank, local)
    if rank == 0 and out is not None:
        print(json.dumps(out), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
