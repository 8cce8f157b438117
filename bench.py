"""Benchmark of the HiGP hot path on B200 (contract: see DESIGN.md §Measurement).

Default workload = BASELINE.json configs[1]: the standalone fused MatMul,
Gaussian Khat.Z and dKhat/dl.Z, n=65536, d=8, Z (n, 32), l=1 f=1 s=1e-2,
synthetic seeded inputs. One step = one fused pass producing both outputs.

    metric: kernel entries x RHS / s  (entries x RHS = n_rows * n_cols * k per output matrix)

    python bench.py [--gpus N --steps K --warmup W] [--precision fast|tf32|fp64] [--impl reference]

Multi-GPU (torchrun): each rank owns a contiguous row block of Khat and needs
the whole RHS block; the RHS is replicated (an all-gather per application in a
solver, not in this single-pass benchmark). Per-GPU work is n/N rows x n cols;
"scaling": "strong" (total work fixed).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="fast", choices=["fast", "tf32", "fp64", "bf16x3"])
    ap.add_argument("--n", type=int, default=65536)
    ap.add_argument("--k", type=int, default=32)
    ap.add_argument("--cpu-rows", type=int, default=8192,
                    help="rows in the bounded CPU-baseline sample (~4 s of 16-core work at cfg2)")
    ap.add_argument("--ref-rows", type=int, default=2048, help="rows per step of the --impl reference arm")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--skip-nlml", action="store_true")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "peer", "replicated"],
                    help="nccl (default): each rank owns its rows of Z and every step all-gathers Z over "
                         "NCCL before the row-block product, as a solver iteration does; peer: each rank "
                         "publishes its rows and the fused all-gather operator reads the others' inside the "
                         "kernel (kgp_engine_peer_*, DESIGN.md section 6); replicated: every rank holds all "
                         "of Z (no exchange timed). At N=1 there is nothing to exchange.")
    ap.add_argument("--skip-secondary", action="store_true",
                    help="only the headline line's keys (no fp64/bf16x3/tf32/cfg5/NLML legs)")
    return ap.parse_args()


# ------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: NVML every 5 ms when
    available (the timed regions are tens of ms), else nvidia-smi every 200 ms."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits
    REASONS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
               "hw_thermal_slowdown": 0x40}

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.nvml = None
        self.stop = threading.Event()

    def _nvml_loop(self, pynvml, h):
        while not self.stop.is_set():
            try:
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
                bits = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                flags = ["Active" if bits & b else "Not Active" for b in
                         (self.REASONS["hw_slowdown"], self.REASONS["hw_thermal_slowdown"],
                          self.REASONS["sw_thermal_slowdown"], self.REASONS["sw_power_cap"])]
                self.lines.append(",".join([str(self.gpu), str(sm), str(mx), "", ""] + flags))
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.nvml = pynvml
            self.thread = threading.Thread(target=self._nvml_loop, args=(pynvml, h), daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.nvml is not None:
            self.stop.set()
            self.thread.join(timeout=2)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------------- CPU baseline (oracle port)
def cpu_baseline(w, rows, steps=1):
    """The reference algorithm (C restatement of kmat.py:165-189 + numba panels, OpenMP on every
    host core) on a bounded row sample of the same workload; returns entries x RHS / s."""
    from oracle import kgp_oracle_c as oc

    oc.matmul("gaussian", w.x, w.l, w.f, w.s, w.z, row0=0, nrows=8, want_dl=True)  # warm
    best = float("inf")
    for _ in range(max(1, steps)):
        t0 = time.perf_counter()
        oc.matmul("gaussian", w.x, w.l, w.f, w.s, w.z, row0=0, nrows=rows, want_dl=True)
        best = min(best, time.perf_counter() - t0)
    units = 2.0 * rows * w.n * w.z.shape[1]
    return units / best, best, oc.max_threads()


def bench_config(args, w, world):
    """The workload description both arms print (the driver compares them)."""
    return {"workload": "cfg2 standalone fused MatMul (BASELINE.json configs[1])", "n": w.n, "d": w.d,
            "k": w.z.shape[1], "kernel": "gaussian", "l": w.l, "f": w.f, "s": w.s,
            "outputs": ["Khat.Z", "dKhat/dl.Z"], "precision": args.precision,
            "l2": "flushed (256 MB write) between timed iterations", "parallelism": f"rows{world}",
            "exchange": args.exchange}


def run_reference(args):
    """--impl reference: the reference's CPU algorithm (oracle port) on this box's host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2503_02259_b200 import workloads

    w = workloads.cfg2(n=args.n, k=args.k)
    for _ in range(max(0, args.warmup)):
        cpu_baseline(w, 64)
    vals = []
    times = []
    for _ in range(args.steps):
        v, t, cores = cpu_baseline(w, args.ref_rows)
        vals.append(v)
        times.append(t)
    value = float(np.median(vals))
    line = {
        "impl": "reference", "metric": "kernel entries x RHS / s (fused Khat.Z + dKhat/dl.Z)",
        "value": value, "unit": "entries*RHS/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": float(np.median(times)) * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, cfg2 shapes)",
        "config": bench_config(args, w, args.gpus),
        "cpu_baseline": {"value": value, "unit": "entries*RHS/s", "cores": cores, "kind": "port",
                         "sample": f"{args.ref_rows} of {args.n} rows per step, both outputs, fp64; "
                                   "oracle/kgp_oracle.c (C restatement of kmat.py:165-189)"},
        "e2e": {"value": value, "unit": "entries*RHS/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ------------------------------------------------------------------------- GPU arm
def measured_tf32_peak(torch):
    """cuBLAS TF32 GEMM (8192^3), best of 5 -- the tensor-pipe denominator for tf32 MMA work."""
    a = torch.randn(8192, 8192, device="cuda", dtype=torch.float32)
    b = torch.randn(8192, 8192, device="cuda", dtype=torch.float32)
    old = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    for _ in range(2):
        a @ b
    best = float("inf")
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        a @ b
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    torch.backends.cuda.matmul.allow_tf32 = old
    del a, b
    return 2.0 * 8192 ** 3 / best / 1e12


def profiled_traffic(precision: str, n: int, k: int):
    """DRAM bytes per launch of the main kernel (dram__bytes_read.sum + dram__bytes_write.sum)
    from the committed `ncu --set full` capture of this exact workload, or None."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "kmm_tc_traffic.json")
    try:
        with open(path) as fh:
            rec = json.load(fh)
    except (OSError, ValueError):
        return None
    key = f"{precision}_n{n}_k{k}"
    return rec.get(key, {}).get("bytes_per_launch")


def fp64_slots(d: int, k: int, nout: int) -> int:
    """FP64 instruction slots per kernel entry of the Gaussian fp64 operator as shipped: 3d for the
    distance (subtract, multiply, add per coordinate: the reference's rounding order takes no FMA),
    13 for the kernel value (argument scale, clamp, exp_neg64t's 11), 2 more for dkappa/dl, and one
    FMA per right-hand side and output. The FP64 pipe issues one instruction per lane slot whether
    it is an FMA or not, so the roofline is counted in slots and reported as 2 flops per slot
    against the DFMA micro-benchmark (exp timed at the software-exp rate)."""
    return 3 * d + 13 + (2 if nout == 2 else 0) + k * nout


FP64_SLOTS_NOTE = ("per entry 3d (distance) + 13 (kernel value, exp_neg64t) + 2 (dkappa/dl, two outputs) + k per "
                   "output FP64 instruction slots, 2 flops per slot against the DFMA rate")


def nlml_metric(cpu: bool):
    """Secondary metric: NLML+gradient evaluations/s at BASELINE configs[0] (n=4096, Gaussian,
    16 probes, rank 256) with its fixed recipe (PCG 50 iterations, 20 Lanczos steps), fp64.

    Credited number: the engine in ON_THE_FLY mode -- every product is the repo's fused fp64
    operator (kmm_f64_kernel), Khat never stored, the north star's path. Secondary ("dense"):
    the reference's own default at n <= 20000 (auto -> DENSE, kmat.py:93-94), where Khat is
    materialised once per eval and the 17-column products are a cuBLAS DGEMM. Each eval includes
    the H2D copy of y and the probes; the preconditioner build is timed separately (the
    reference's 1.41 s likewise excludes its 0.19 s build).

    Roofline (FP64 pipe): the recipe's operator passes from its fixed iteration counts -- w:
    50 x 1 column, probes: 20 x 16 columns, the fused derivative pass: 17 columns x 2 outputs --
    each costing per kernel entry fp64_slots(d, k, outputs) FP64 instruction slots (every entry of
    every pass counted as the reference streams it), over the eval time, against the measured
    DFMA rate."""
    import torch

    from paper_2503_02259_b200 import gp, precond, workloads
    from paper_2503_02259_b200.kmat import EngineMode, Hyperparams, KernelEngine
    from paper_2503_02259_b200.kernels import KernelType

    w = workloads.cfg1()
    probes = gp.ProbeSet.generate(w.n, w.k_z, w.probe_seed)
    torch.linalg.cholesky(torch.eye(8, dtype=torch.float64, device="cuda"))  # one-time cuSOLVER init
    torch.linalg.solve_triangular(torch.eye(8, dtype=torch.float64, device="cuda"),
                                  torch.eye(8, dtype=torch.float64, device="cuda"), upper=False)

    def run(mode, reps=10, precision="fp64"):
        eng = KernelEngine(KernelType.GAUSSIAN, w.x, Hyperparams(w.l, w.f, w.s), mode=mode, precision=precision)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pre = precond.build(eng, w.rank)
        torch.cuda.synchronize()
        t_first = time.perf_counter() - t0  # includes lazy module loading of every kernel it uses
        tb = []
        for _ in range(5):  # steady state (training rebuilds it every step): median of 5
            t0 = time.perf_counter()
            pre = precond.build(eng, w.rank)
            torch.cuda.synchronize()
            tb.append(time.perf_counter() - t0)
        t_build = float(np.median(tb))

        def ev():
            return gp.nlml_grad_iterative(eng, w.y, pre, probes, tol=0.0, max_iter=50, probe_tol=0.0,
                                          probe_max_iter=20)

        for _ in range(2):
            ev()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            lg = ev()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / reps, t_build, t_first, lg

    t_eval, t_build, t_first, lg = run(EngineMode.ON_THE_FLY)
    t_dense, _, _, lg_dense = run(EngineMode.DENSE)
    t_fast, _, _, lg_fast = run(EngineMode.ON_THE_FLY, precision="fast")
    n, d = w.n, w.d
    passes = [(50, 1, 1), (20, 16, 1), (1, 17, 2)]  # (iterations, columns, outputs)
    flops = sum(it * n * n * 2 * fp64_slots(d, k, nout) for it, k, nout in passes)
    achieved = flops / t_eval / 1e12
    out = {"workload": "cfg1 fixed recipe (BASELINE.json configs[0]): n=4096 d=3 Gaussian, 16 probes, "
                       "rank 256, PCG 50 + SLQ 20, fp64 operator, ON_THE_FLY (fused kernel, Khat never stored)",
           "evals_per_s": 1.0 / t_eval, "ms_per_eval": t_eval * 1e3, "precond_build_ms": t_build * 1e3,
           "precond_build_first_call_ms": t_first * 1e3, "precond_build_note": "median of 5 rebuilds (torch "
           "linalg / allocator spikes of up to ~0.9 s are seen on single calls)", "loss": lg.loss,
           "timer": "wall clock around synchronous calls (each eval ends in a D2H read)",
           "roofline": {"bound": "fp64", "achieved": achieved, "peak": FP64_DFMA_TFLOPS, "unit": "TFLOP/s",
                        "frac": achieved / FP64_DFMA_TFLOPS,
                        "algorithmic": "operator passes of the fixed recipe (50 x 1 + 20 x 16 columns, one "
                                       "17-column two-output derivative pass), " + FP64_SLOTS_NOTE +
                                       "; PCG vector work and SLQ not counted"},
           "dense": {"workload": "same recipe, DENSE mode (the reference's default at n <= 20000): Khat "
                                 "materialised by the repo's panel kernel, 17-column products by cuBLAS DGEMM",
                     "evals_per_s": 1.0 / t_dense, "ms_per_eval": t_dense * 1e3, "loss": lg_dense.loss},
           "fast_mode": {"workload": "same recipe, ON_THE_FLY with the 3xTF32 fused tcgen05 operator (the north "
                                     "star's tensor-core NLML mode, <= 1e-3: tests/test_gpu_parity.py "
                                     "test_cfg1_fast_mode_within_tf32_bar)",
                         "evals_per_s": 1.0 / t_fast, "ms_per_eval": t_fast * 1e3, "loss": lg_fast.loss,
                         "loss_rel_diff_vs_fp64": abs(lg_fast.loss - lg.loss) / abs(lg.loss),
                         "loss_note": "the fixed recipe stops the solves unconverged (PCG 50, probes 20 "
                                      "iterations, SLQ 20 steps), so the two precisions end on different "
                                      "partial CG trajectories; converged (tol 1e-10) the same evaluation is "
                                      "within 1e-3 of the reference in every component (the cited test)"}}
    if cpu:
        from oracle import kgp_oracle as orc
        from oracle import kgp_oracle_c as oc

        ny = orc.Nystrom("gaussian", w.x, w.l, w.f, w.s, w.rank)
        best = float("inf")
        for _ in range(2):
            t0 = time.perf_counter()
            ref = orc.nlml_grad("gaussian", w.x, w.y, w.l, w.f, w.s, probes.vectors, ny, tol=0.0, max_iter=50,
                                probe_tol=0.0, dense=True, probe_max_iter=20, panels="c")
            best = min(best, time.perf_counter() - t0)
        out["cpu_baseline"] = {"evals_per_s": 1.0 / best, "kind": "port", "cores": oc.max_threads(),
                               "sample": "one full eval (best of 2), the reference's default DENSE path: Khat and "
                                         "the two derivative matrices by OpenMP C panels (oracle/kgp_oracle.c, "
                                         "numba-prange equivalent), products by numpy BLAS; on the 8-core build host it "
                                         "takes 0.96x kernelgp's own time for the same eval (0.403 vs 0.419 s, same "
                                         "loss; tools/cpu_nlml_baseline.py)"}
        out["loss_rel_diff_vs_cpu"] = abs(lg.loss - ref[0]) / abs(ref[0])
    return out


def nlml_cfg3_metric(n: int = 262144, reps: int = 1):
    """Secondary: NLML+gradient evaluations/s on configs[2] at its full n = 262144
    (Matern-3/2, d=4, 32 probes, rank 1024, tol = probe_tol = 1e-6 -- probe_tol defaults to tol
    in the reference's gp.py as here -- fast operator) with the AFN preconditioner and the
    preconditioned-probe ESTIMATOR EXTENSION: probes are drawn from N(0, M), so this line is
    not the reference's same-probe number (parity of the reference estimator on this generator
    is tested at reduced n, tests/test_gpu_parity.py). The reference's own estimator does not
    converge its unpreconditioned probes
    within 2000 iterations here (103 s on the device). One warm-up eval,
    then `reps` timed ones (~4.6 s each)."""
    import torch

    from paper_2503_02259_b200 import gp, precond, workloads
    from paper_2503_02259_b200.kmat import Hyperparams, KernelEngine
    from paper_2503_02259_b200.kernels import KernelType

    w = workloads.cfg3(n=n)
    e = KernelEngine(KernelType.MATERN32, w.x, Hyperparams(w.l, w.f, w.s), precision="fast")
    probes = gp.ProbeSet.generate(n, w.k_z, 0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pre = precond.build_afn(e, w.rank, 32)
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0

    def ev():
        return gp.nlml_grad_iterative(e, w.y, pre, probes, tol=1e-6, max_iter=2000, probe_tol=1e-6,
                                      preconditioned_probes=True)

    ev()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        lg = ev()
    torch.cuda.synchronize()
    t_eval = (time.perf_counter() - t0) / reps
    return {"workload": f"EXTENSION (not the reference estimator): configs[2] generator at n={n}, Matern-3/2 "
                        "d=4, 32 probes drawn from N(0, M_AFN), AFN rank 1024, tol = probe_tol = 1e-6, "
                        "fast operator, preconditioned-probe estimator",
            "reps": reps,
            "evals_per_s": 1.0 / t_eval, "ms_per_eval": t_eval * 1e3, "precond_build_ms": t_build * 1e3,
            "loss": lg.loss, "converged": lg.converged,
            "timer": "wall clock around synchronous calls"}


# tcgen05 kind::tf32 issue rate at the contraction's shape (M=128, N=32, K=8, A in TMEM),
# tools/micro/mma_n.cu on this pool (profiles/r01_micro_tensor_fp64.txt)
TC_TF32_N32_TFLOPS = 1056.9
# FP64 pipe: DFMA-only micro-benchmark on this pool (tools/micro/fp64_mix.cu,
# profiles/r01_micro_tensor_fp64.txt); MEASURED_PEAKS.json has no FP64 figure
FP64_DFMA_TFLOPS = 36.07
DTYPES = {"fast": "f32 tile + 3xtf32 mma", "tf32": "f32 tile + tf32 mma", "fp64": "f64",
          "bf16x3": "f32 tile + bf16x3 mma (A0B0 + A0B1 + A1B0)"}
# tensor products per output of each precision (hi.hi + hi.lo + lo.hi; hi.hi; A0B0 + A0B1 + A1B0)
SPLITS = {"fast": 3, "tf32": 1, "bf16x3": 3}


def measured_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def tc_roofline(precision, entries, k, kernel_t, measure_cublas):
    """Tensor roofline of the fused operator: ALGORITHMIC tensor flops = entries x 2 outputs x
    products x 2k, over the kernel's own launch time, against MEASURED_PEAKS.json's dense bf16
    burst figure (/2 for tf32 MMAs, which issue at half the bf16 rate; x1 for the bf16x3 mode's
    kind::f16 MMAs). Alternatives: the sustained bf16 figure, a cuBLAS TF32 GEMM measured in this
    run, and the tcgen05 N=32 issue rate from the micro-benchmark."""
    import torch

    flops = 2 * SPLITS[precision] * 2.0 * entries * k
    achieved = flops / kernel_t / 1e12
    mp = measured_peaks()
    bf16 = float(mp.get("bf16_tflops", 0.0)) or None
    div = 1.0 if precision == "bf16x3" else 2.0
    peak = bf16 / div if bf16 else None
    alts = []
    if mp.get("bf16_tflops_sustained"):
        ps = float(mp["bf16_tflops_sustained"]) / div
        alts.append({"source": "MEASURED_PEAKS.json bf16_tflops_sustained" + (" / 2" if div == 2 else ""),
                     "peak": ps, "frac": achieved / ps})
    if measure_cublas and precision != "bf16x3":
        pc = measured_tf32_peak(torch)
        alts.append({"source": "cuBLAS TF32 GEMM 8192^3 measured in this run", "peak": pc, "frac": achieved / pc})
    if precision != "bf16x3":
        alts.append({"source": "tcgen05 kind::tf32 M=128 N=32 issue rate (tools/micro/mma_n.cu, "
                               "profiles/r01_micro_tensor_fp64.txt)",
                     "peak": TC_TF32_N32_TFLOPS, "frac": achieved / TC_TF32_N32_TFLOPS})
    if peak is None:  # no driver-written peaks: the profiling recipe's fallback is the cuBLAS figure
        peak = next((x["peak"] for x in alts if x["source"].startswith("cuBLAS")), None)
    return {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak if peak else None,
            "peak_source": ("MEASURED_PEAKS.json bf16_tflops (burst; the kernel is timed alone)"
                            + (" / 2 (tf32 MMAs issue at half the bf16 rate)" if div == 2 else "")),
            "peak_alternatives": alts,
            "algorithmic": f"2 outputs x {SPLITS[precision]} products x 2k flops per kernel entry"}


def mode_metric(w, ref_k, ref_l, precision, steps: int = 10):
    """Secondary: the same cfg2 step in another tensor-core precision ("tf32": 1xTF32, the north
    star's "TF32 mode", operator bar 1e-3; "bf16x3": split-bf16 A0B0 + A0B1 + A1B0), with its
    error against the 3xTF32 outputs of the main run and its own roofline."""
    import torch

    from paper_2503_02259_b200 import KernelEngine, KernelType, _lib
    from paper_2503_02259_b200.kmat import Hyperparams

    n, k = w.n, w.z.shape[1]
    e = KernelEngine(KernelType.GAUSSIAN, w.x, Hyperparams(w.l, w.f, w.s), precision=precision)
    zd = torch.from_numpy(w.z).cuda()
    ok, ol = torch.empty_like(ref_k), torch.empty_like(ref_l)
    st = torch.cuda.current_stream()

    def step():
        _lib.call("kgp_engine_matmul", e.handle, k, zd.data_ptr(), zd.stride(0), zd.stride(1), ok.data_ptr(),
                  ol.data_ptr(), None, ok.stride(0), ok.stride(1), st.cuda_stream)

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    _lib.call("kgp_engine_set_timing", e.handle, 1)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for s_ev, e_ev in ev:
        flush.zero_()
        s_ev.record(st)
        step()
        e_ev.record(st)
    torch.cuda.synchronize()
    kern_ms, kern_n = _lib.kernel_time(e.handle)
    _lib.call("kgp_engine_set_timing", e.handle, 0)
    t = float(np.mean([a.elapsed_time(b) / 1e3 for a, b in ev]))
    err_k = float((ok - ref_k).abs().max() / ref_k.abs().max())
    err_l = float((ol - ref_l).abs().max() / ref_l.abs().max())
    e.close()
    kt = kern_ms / 1e3 / kern_n if kern_n else t
    roof = tc_roofline(precision, n * n, k, kt, False)
    roof["kernel_ms"] = kt * 1e3
    notes = {"tf32": "1xTF32 contraction; not the NLML mode (its loss/gradient errors reach 1e-1, DESIGN.md 4)",
             "bf16x3": "two round-to-nearest bf16 terms per operand, 3 kind::f16 products; operator error ~5e-6 "
                       "(tests/test_gpu_parity.py), d > 4 only"}
    return {"value": 2.0 * n * n * k / t, "unit": "entries*RHS/s", "ms_per_step": t * 1e3,
            "max_rel_diff_vs_fast": {"Khat.Z": err_k, "dKhat/dl.Z": err_l}, "roofline": roof,
            "note": notes[precision]}


def fp64_mode_metric(w, steps: int = 5):
    """Secondary: the cfg2 step with the fp64 operator (the parity precision), and its
    roofline on the FP64 pipe: fp64_slots(d, k, 2) instruction slots per kernel entry against the
    measured DFMA rate."""
    import torch

    from paper_2503_02259_b200 import KernelEngine, KernelType, _lib
    from paper_2503_02259_b200.kmat import EngineMode, Hyperparams

    n, k, d = w.n, w.z.shape[1], w.d
    e = KernelEngine(KernelType.GAUSSIAN, w.x, Hyperparams(w.l, w.f, w.s), mode=EngineMode.ON_THE_FLY,
                     precision="fp64")
    zd = torch.from_numpy(w.z).cuda()
    ok = torch.empty((n, k), dtype=torch.float64, device="cuda")
    ol = torch.empty_like(ok)
    st = torch.cuda.current_stream()

    def step():
        _lib.call("kgp_engine_matmul", e.handle, k, zd.data_ptr(), zd.stride(0), zd.stride(1), ok.data_ptr(),
                  ol.data_ptr(), None, ok.stride(0), ok.stride(1), st.cuda_stream)

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for s_ev, e_ev in ev:
        s_ev.record(st)
        step()
        e_ev.record(st)
    torch.cuda.synchronize()
    t = float(np.mean([a.elapsed_time(b) / 1e3 for a, b in ev]))
    e.close()
    per_entry = 2 * fp64_slots(d, k, 2)
    achieved = per_entry * n * n / t / 1e12
    return {"value": 2.0 * n * n * k / t, "unit": "entries*RHS/s", "ms_per_step": t * 1e3,
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": FP64_DFMA_TFLOPS, "unit": "TFLOP/s",
                         "frac": achieved / FP64_DFMA_TFLOPS,
                         "peak_source": "DFMA micro-benchmark on this pool (profiles/r01_micro_tensor_fp64.txt); "
                                        "MEASURED_PEAKS.json has no FP64 figure",
                         "algorithmic": f"{per_entry} DFMA-equivalent flops per kernel entry: " + FP64_SLOTS_NOTE}}


def cfg5_operator_metric(world, rank, local, dist, steps: int = 3):
    """Secondary (every N): the configs[4]-size operator that a cfg5 PCG iteration applies --
    Matern-5/2, n = 1048576, d = 2, Khat.[y, Z] with 64 RHS, fast precision -- row-sharded over
    the N ranks, each step all-gathering the RHS block over NCCL (N > 1) before the row-block
    product (the north star's >= 85 % scaling target is stated for n >= 1M). Device-timed, max
    over ranks; value = whole-job entries x RHS / s."""
    import torch

    from paper_2503_02259_b200 import KernelEngine, KernelType, _lib, workloads
    from paper_2503_02259_b200 import dist as kdist
    from paper_2503_02259_b200.kmat import Hyperparams

    w = workloads.cfg5(m_test=1)
    n, k = w.n, 64
    r0, r1 = kdist.row_range(n, world, rank)
    e = KernelEngine(KernelType.MATERN52, w.x, Hyperparams(w.l, w.f, w.s), precision="fast")
    if world > 1:
        _lib.call("kgp_engine_set_rows", e.handle, r0, r1 - r0)
    zfull = torch.from_numpy(np.random.default_rng(5).standard_normal((n, k))).cuda()
    zloc = zfull[r0:r1].clone()
    if world > 1:
        zfull = torch.empty_like(zfull)
    out = torch.empty((r1 - r0, k), dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream()

    def step():
        if world > 1:
            dist.all_gather_into_tensor(zfull, zloc)
        _lib.call("kgp_engine_matmul", e.handle, k, zfull.data_ptr(), zfull.stride(0), zfull.stride(1),
                  out.data_ptr(), None, None, out.stride(0), out.stride(1), st.cuda_stream)

    step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for s_ev, e_ev in ev:
        s_ev.record(st)
        step()
        e_ev.record(st)
    torch.cuda.synchronize()
    t = float(np.mean([a.elapsed_time(b) / 1e3 for a, b in ev]))
    if world > 1:
        tt = torch.tensor([t], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    e.close()
    return {"workload": "configs[4] operator: Matern-5/2 n=1048576 d=2, Khat.[y,Z] 64 RHS, fast, rows sharded "
                        "over the ranks" + (", NCCL all-gather of the RHS block in every step" if world > 1 else ""),
            "value": 1.0 * n * n * k / t, "unit": "entries*RHS/s", "ms_per_step": t * 1e3, "steps": steps,
            "n_gpus": world, "scaling": "strong"}


def run_gpu(args):
    import torch
    import torch.distributed as dist

    from paper_2503_02259_b200 import KernelEngine, KernelType, _lib, workloads
    from paper_2503_02259_b200.kmat import Hyperparams

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    w = workloads.cfg2(n=args.n, k=args.k)
    n, k = w.n, w.z.shape[1]
    from paper_2503_02259_b200 import dist as kdist

    peer = args.exchange == "peer"
    r0, r1 = kdist.row_range(n, world, rank, 32 if peer else 1)
    hp = Hyperparams(w.l, w.f, w.s)
    eng = KernelEngine(KernelType.GAUSSIAN, w.x, hp, precision=args.precision)
    if world > 1 or peer:
        _lib.call("kgp_engine_set_rows", eng.handle, r0, r1 - r0)
    rows = r1 - r0
    zd = torch.from_numpy(w.z).cuda()
    out_k = torch.empty((rows, k), dtype=torch.float64, device="cuda")
    out_l = torch.empty_like(out_k)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # 256 MB > 126 MB L2
    tiles = None
    if peer:
        starts = [kdist.row_range(n, world, q, 32)[0] for q in range(world)] + [n]
        if world == 1:  # the fused path on one GPU: the rank reads its own published tiles
            import ctypes

            nb, ptr = ctypes.c_int64(), ctypes.c_void_p()
            _lib.call("kgp_engine_peer_buffer_bytes", eng.handle, k, rows, ctypes.byref(nb))
            _lib.call("kgp_peer_alloc", nb.value, ctypes.byref(ptr), None)
            tiles = kdist.PeerTiles(eng.handle, 1, 0, starts, k, bases=[ptr.value])
            tiles._own = ptr.value
        else:
            tiles = kdist.PeerTiles(eng.handle, world, rank, starts, k, comm=kdist.Comm(n, align=32))
    zloc = zd[r0:r1]
    epoch = [0]
    gather = args.exchange == "nccl" and world > 1
    if gather:
        # the rank owns only its rows of Z; every step gathers the whole block (equal row
        # blocks: all_gather_into_tensor concatenates them in rank order), as a PCG iteration
        # does before its row-block product (dist.py)
        assert n % world == 0, "--exchange nccl needs n divisible by the world size"
        zloc = zd[r0:r1].clone()
        zd = torch.empty_like(zd)

    def step():
        if peer:  # publish own rows of Z, then the operator pulls every rank's tiles
            epoch[0] += 1
            _lib.call("kgp_engine_peer_publish", eng.handle, k, zloc.data_ptr(), zloc.stride(0), zloc.stride(1),
                      epoch[0], stream.cuda_stream)
            _lib.call("kgp_engine_peer_matmul", eng.handle, k, epoch[0], out_k.data_ptr(), out_l.data_ptr(), None,
                      out_k.stride(0), out_k.stride(1), stream.cuda_stream)
            return
        if gather:
            dist.all_gather_into_tensor(zd, zloc)
        _lib.call("kgp_engine_matmul", eng.handle, k, zd.data_ptr(), zd.stride(0), zd.stride(1),
                  out_k.data_ptr(), out_l.data_ptr(), None, out_k.stride(0), out_k.stride(1), stream.cuda_stream)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    # the dominant kernel is bracketed by CUDA events inside libkgp, on the stream it launches on
    _lib.call("kgp_engine_set_timing", eng.handle, 1)
    launches0 = _lib.launch_count()
    with ClockSampler(local) as clk:
        for s_ev, e_ev in ev:
            flush.zero_()  # L2 flush between timed iterations (outside the event pair)
            s_ev.record(stream)
            step()
            e_ev.record(stream)
        torch.cuda.synchronize()
    launches = _lib.launch_count() - launches0
    kern_ms, kern_n = _lib.kernel_time(eng.handle)
    _lib.call("kgp_engine_set_timing", eng.handle, 0)
    times = [s.elapsed_time(e) / 1e3 for s, e in ev]
    t_step = float(np.mean(times))
    if world > 1:
        t = torch.tensor([t_step], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_step = float(t.item())
    units = 2.0 * n * n * k  # both outputs, whole job
    value = units / t_step

    # ---- e2e: the C-ABI host-buffer entry (kgp_engine_matmul_host): H2D of Z and D2H of both
    # outputs inside the timed region (pinned host memory; the output transfer is pipelined
    # behind the computation in row chunks by the library)
    zh = torch.from_numpy(w.z).pin_memory()
    ok_h = torch.empty((rows, k), dtype=torch.float64).pin_memory()
    ol_h = torch.empty_like(ok_h).pin_memory()

    def e2e_step():
        _lib.call("kgp_engine_matmul_host", eng.handle, k, zh.data_ptr(), ok_h.data_ptr(), ol_h.data_ptr(), None,
                  stream.cuda_stream)

    for _ in range(3):
        e2e_step()
    torch.cuda.synchronize()
    ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for s_ev, e_ev in ev2:
        flush.zero_()
        s_ev.record(stream)
        e2e_step()
        e_ev.record(stream)
    torch.cuda.synchronize()
    t_e2e = float(np.mean([s.elapsed_time(e) / 1e3 for s, e in ev2]))
    if world > 1:
        t = torch.tensor([t_e2e], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_e2e = float(t.item())

    # ---- roofline of the dominant kernel (kmm_tc_kernel): average duration of its launches
    # inside the timed region (events recorded by libkgp around each launch)
    kernel_t = kern_ms / 1e3 / kern_n if kern_n else t_step
    roof = None
    if args.precision != "fp64":
        roof = tc_roofline(args.precision, rows * n, k, kernel_t, rank == 0)
        roof.update({"traffic": profiled_traffic(args.precision, n, k), "kernel_ms": kernel_t * 1e3,
                     "kernel_launches_timed": kern_n,
                     "kernel_share_of_step": kernel_t * max(kern_n, 1) / args.steps / t_step})
    # ---- secondary legs: cfg5-size operator on every rank (collective when N > 1), the rest
    # on rank 0 at N = 1
    extra = {}
    if not args.skip_secondary:
        extra["cfg5_operator"] = cfg5_operator_metric(world, rank, local, dist if world > 1 else None)
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            v, t, cores = cpu_baseline(w, args.cpu_rows)
            cpu = {"value": v, "unit": "entries*RHS/s", "cores": cores, "kind": "port",
                   "sample": f"{args.cpu_rows} of {n} rows, both outputs, fp64, best of 1 "
                             "(oracle/kgp_oracle.c: C restatement of kmat.py:165-189 + numba panels)"}
        line = {
            "metric": "kernel entries x RHS / s (fused Khat.Z + dKhat/dl.Z)",
            "value": value, "unit": "entries*RHS/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": t_step * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": DTYPES[args.precision],
            "data": "synthetic (seeded numpy default_rng, BASELINE configs[1] shapes and distributions)",
            "config": bench_config(args, w, world),
            "e2e": {"value": units / t_e2e, "unit": "entries*RHS/s", "h2d_bytes_per_step": int(zh.numel() * 8),
                    "d2h_bytes_per_step": int(2 * ok_h.numel() * 8), "ms_per_step": t_e2e * 1e3},
            "gpu_launches": launches,
            "roofline": roof,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
        }
        line.update(extra)
        if world == 1 and not args.skip_secondary:
            if args.precision == "fast":
                line["fp64_mode"] = fp64_mode_metric(w)
                line["bf16x3_mode"] = mode_metric(w, out_k, out_l, "bf16x3")
                line["tf32_mode"] = mode_metric(w, out_k, out_l, "tf32")
            if not args.skip_nlml:
                line["nlml"] = nlml_metric(cpu=not args.no_cpu_baseline)
                line["nlml_cfg3"] = nlml_cfg3_metric()
        print(json.dumps(line))
    if tiles is not None:
        tiles.close()  # synchronises and barriers before unmapping (dist.PeerTiles.close)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    run_gpu(args)


if __name__ == "__main__":
    main()
