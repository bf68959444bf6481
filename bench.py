#!/usr/bin/env python
"""Benchmark: rank-1 SVD updates/s (fp64, n = 4096) on BASELINE.json config C3, plus
the FMM Cauchy-apply fraction of the FP64 (DMMA) roofline.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one svd1_update (Alg 6.1) of the C3 stream
(m = n = 4096, sigma_i = 10^(-6 i/n), a, b ~ N(0,1)); the K timed steps are updates
1..K of that stream (indices wrap at 16), applied in place to device-resident
factors.  N > 1: one process per GPU (torchrun; `--gpus N` without torchrun relaunches
itself under torch.distributed.run), rows of U and V sharded across ranks, the STEP-1
projections all-reduced over NCCL and every eigen-update's spectral phase sliced across
the ranks and all-gathered inside libsvd1; time = max over ranks.
`--impl reference` times the CPU oracle (oracle/, the base contract's reference arm
for this tier) on whole updates of the same workload (one whole C3 update per step,
about 8 s each on a 16-core host).
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "rank-1 SVD updates/s (fp64, n=4096) and FMM Cauchy-apply % of FP64 roofline"
UNIT = "updates/s"
CFG_ID = 3
WORKLOADS = {
    1: "C1: m=n=64 fp64, A i.i.d. N(0,1), U,S,V from an SVD of A, update a,b ~ N(0,1) (repeated)",
    2: "C2: m=n=1024 fp64, A i.i.d. N(0,1), update a,b ~ N(0,1)/sqrt(n) (repeated)",
    3: ("C3: m=n=4096 fp64, A = Q1 diag(sigma) Q2^T, sigma_i = 10^(-6 i/n) (graded), "
        "16-update stream a,b ~ N(0,1), eps=1e-10 (p=16)"),
    4: "C4: m=2048, n=8192 fp64, A i.i.d. N(0,1), 64-update stream a,b ~ N(0,1)*1e-2",
    5: ("C5: m=n=16384 fp64, A = Q1 diag(sigma) Q2^T, sigma ~ U[1,100] with 5% bitwise "
        "duplicates, 8-update stream a,b ~ N(0,1)"),
}
WORKLOAD = WORKLOADS[3]
FP64_PEAK_TFLOPS = 37.17  # measured DMMA m8n8k4 sustained on this pool's B200 (profiles/fp64_peak_r01.jsonl)
HBM_PEAK_GBS = 6553.0


def _measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """NVML polling thread: SM clock and clock-event reasons during the timed region."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index):
        self.samples, self.reasons, self.ok = [], set(), False
        # polling period (s; SVD1_BENCH_CLOCK_MS overrides: 2 and 10 ms gave the same C3
        # values over 6 runs each, so the sampler does not perturb the timed region)
        self.interval = float(os.environ.get("SVD1_BENCH_CLOCK_MS", "2")) / 1e3
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.interval)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def cpu_info():
    """Host description for the CPU numbers: logical CPUs and model."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def oracle_update_times(inp, steps, threads=None):
    """The CPU oracle (oracle/, as it stands) running WHOLE C3 updates of the stream in
    order (each on the previous step's output): Alg 6.1 with the literal STEP-1 products,
    bisection over every root, Loewner, X and the explicit O(n^3) products on ALL rows of
    U and V (no sampling, nothing extrapolated); sign rule by probes (pinned equal to the
    explicit rule).  threads: oracle threads and BLAS threads (None = all host cores).
    Returns the per-step times (s)."""
    import oracle as O
    import oracle.svd1_oracle as OM
    U, s, V = inp["U"], inp["sigma"], inp["V"]
    if not isinstance(U, np.ndarray):
        U, s, V = U.cpu().numpy(), s.cpu().numpy(), V.cpu().numpy()
    from contextlib import nullcontext
    try:
        from threadpoolctl import threadpool_limits
    except Exception:  # pragma: no cover
        threadpool_limits = None
    old = OM.THREADS
    t = []
    cm = threadpool_limits(limits=threads) if (threads and threadpool_limits) else nullcontext()
    try:
        if threads:
            OM.THREADS = threads
        with cm:
            for k in range(steps):
                a, b = inp["ab"][k % len(inp["ab"])]
                t0 = time.perf_counter()
                r = O.svd_update(U, s, V, a, b, sign_rule="probe")
                t.append(time.perf_counter() - t0)
                U, s, V = r["U"], r["sigma"], r["V"]
    finally:
        OM.THREADS = old
    return t


def run_reference(args, rank, world):
    """The reference arm for this tier: the CPU oracle on the same workload and metric
    (C3 updates/s), each step one whole C3 update of the stream (all rows, full explicit
    products), on all host cores; rank 0 alone (the others exit without work)."""
    if rank != 0:
        return
    from synth import config_inputs
    inp = config_inputs(CFG_ID)
    oracle_update_times(inp, args.warmup)
    t0 = time.perf_counter()
    t = oracle_update_times(inp, args.steps)
    wall = time.perf_counter() - t0
    total = sum(t)
    val = args.steps / total
    import oracle.svd1_oracle as OM
    sample = ("per step: one whole C3 update of the 16-update stream (m = n = 4096) by the oracle: literal "
              "STEP-1 products, bisection over all 4096 roots of each of the 4 eigen-updates, Loewner, X, explicit "
              "products on all 4096 rows of U and V; nothing sampled or extrapolated")
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, BASELINE.json C3 recipe)",
            "config": {"workload": WORKLOAD, "m": 4096, "n": 4096, "eps": 1e-10},
            "timed_wall_s": wall,
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": OM.THREADS, "kind": "oracle", "sample": sample,
                             **cpu_info()},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=16)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline oracle timing")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--full-v", action="store_true",
                    help="keep the full n x n right factor for m < n configs (default: thin V, "
                         "SVD1_THIN_V, DESIGN.md §4.10)")
    ap.add_argument("--fused", action="store_true",
                    help="fused per-side pass (SVD1_FUSED_SIDE, SURVEY 8(f) #1): both applies of a side "
                         "row chunk by row chunk, L2-resident")
    ap.add_argument("--sequential", action="store_true",
                    help="time the per-update API (svd1_update) instead of svd1_update_batch")
    ap.add_argument("--no-seq", action="store_true",
                    help="skip the per-update API reference leg (profiling the stream alone)")
    ap.add_argument("--config", type=int, default=CFG_ID, choices=[1, 2, 3, 4, 5],
                    help="BASELINE.json config (default C3, the headline metric's workload)")
    args = ap.parse_args()
    if os.environ.get("SVD1_BENCH_FUSED"):  # (experiments: select the fused pass through the environment)
        args.fused = True
    global WORKLOAD, METRIC
    if args.config != CFG_ID:
        WORKLOAD = WORKLOADS[args.config]
        METRIC = f"rank-1 SVD updates/s (fp64, config C{args.config})"
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if args.gpus != world:
        if "WORLD_SIZE" not in os.environ and args.gpus > 1:
            # one process per GPU: relaunch this command under torch.distributed.run
            import socket
            import subprocess
            sk = socket.socket()
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
            sk.close()
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
                   "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
            sys.exit(subprocess.call(cmd))
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}: run one process per GPU"}),
              flush=True)
        sys.exit(2)

    import torch
    import torch.distributed as dist
    import paper_1707_08369_b200 as P
    from synth import config_inputs

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    inp = config_inputs(args.config, device=dev)
    cfg = inp["cfg"]
    m, n = cfg["m"], cfg["n"]
    ab = [(torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)) for a, b in inp["ab"]]
    U0, s0, V0 = inp["U"], inp["sigma"], inp["V"]
    # row shards (paper_1707_08369_b200.parallel: NCCL all-reduce of the projections)
    from paper_1707_08369_b200.parallel import ShardedUpdater
    stream = torch.cuda.current_stream()
    thin = m < n and not args.full_v
    upd = ShardedUpdater(m, n, rank, world, eps=cfg["eps"], stream=stream,
                         flags=(P.THIN_V if thin else 0) | (P.FUSED_SIDE if args.fused else 0))
    u0, u1, v0, v1 = upd.u_lo, upd.u_hi, upd.v_lo, upd.v_hi
    U = U0[u0:u1].clone()
    if thin:  # V[:, :m] plus one workspace column (SVD1_THIN_V)
        V = torch.zeros((v1 - v0, m + 1), dtype=torch.float64, device=dev)
        V[:, :m] = V0[v0:v1, :m]
    else:
        V = V0[v0:v1].clone()
    sig = s0.clone()
    Upr, Vpr, spr = U.clone(), V.clone(), sig.clone()

    def step(t, a=None, b=None):
        a_t, b_t = ab[t % len(ab)] if a is None else (a, b)
        return upd.update(U, sig, V, a_t, b_t)

    # the stream of updates goes through svd1_update_batch (pipelined: update t+1's
    # spectral phase overlaps update t's applies); row-sharded: the K
    # projection vectors of a chunk are all-reduced once, then svd1_update_batch_projected
    # (C1/C2 are launch-bound, where the per-update API is the faster of the two)
    batch = not args.sequential and m * n > 1024 * 1024
    A_all = torch.stack([a for a, _ in ab])
    B_all = torch.stack([b for _, b in ab])

    def run(t0, K, A_src=None, B_src=None):
        """updates t0 .. t0+K-1 of the stream; returns their reports"""
        if not batch:
            return [step(t) for t in range(t0, t0 + K)]
        out = []
        t = t0
        while t < t0 + K:
            kc = min(28, t0 + K - t)
            idx = [(t + q) % len(ab) for q in range(kc)]
            if A_src is None:
                Ab, Bb = A_all[idx], B_all[idx]
            else:
                Ab, Bb = A_src[[q - t0 for q in range(t, t + kc)]], B_src[[q - t0 for q in range(t, t + kc)]]
            out += upd.update_batch(U, sig, V, Ab, Bb)
            t += kc
        return out

    def restore():
        U.copy_(Upr)
        V.copy_(Vpr)
        sig.copy_(spr)

    def barrier():
        if world > 1:
            dist.barrier()

    # warm-up: W steps, and at least the timed stream's length (its later updates build deeper
    # trees than the first W: their first-time host / device costs stay out of the timed region)
    # (twice: the first stream of a process pays one-off host costs -- thread start, first
    # touch of the host-side plan buffers -- measured as a 5-7 % slower first run)
    for _ in range(2):
        run(0, max(args.warmup, args.steps))
        restore()
    torch.cuda.synchronize()
    reps = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    import gc
    gc.collect()
    gc.disable()  # no Python collector pause inside the timed region
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        e0.record(stream)
        reps = run(0, args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
    gc.enable()
    barrier()
    ms = e0.elapsed_time(e1)
    if world > 1:
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    value = args.steps / (ms / 1e3)
    seq = None
    if batch and not args.no_seq:  # the per-update API on the same stream, for reference (not the headline)
        restore()
        for t in range(max(args.warmup, args.steps)):  # its own buffers warm too
            step(t)
        restore()
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        seqreps = [step(t) for t in range(args.steps)]
        g1.record(stream)
        torch.cuda.synchronize()
        sms = g0.elapsed_time(g1)
        sreps = seqreps
        s_ap = sum(r["t_ms"][5] for r in sreps)
        s_fl = sum(sum(r["apply_flops"]) for r in sreps)
        seq = {"api": "svd1_update (one call per update)", "value": args.steps / (sms / 1e3),
               "ms_per_step": sms / args.steps,
               "apply_achieved_tflops": s_fl / (s_ap / 1e3) / 1e12 if s_ap > 0 else None}

    # roofline of the dominant kernel (the FMM Cauchy apply), from live CUDA events
    ap_ms = sum(r["t_ms"][5] for r in reps)  # apply phase (U and V sides concurrent)
    ap_fl = sum(sum(r["apply_flops"]) for r in reps)
    ap_fx = sum(sum(r["apply_flops_exec"]) for r in reps)
    sp_ms = sum(sum(r["spectral_ms"]) for r in reps)
    n_apply = sum(sum(1 for x in r["apply_flops"] if x > 0) for r in reps)
    # dominant kernel: the FMM Cauchy apply (its GEMM passes carry every algorithmic
    # flop).  The U- and V-side applies run concurrently on two streams (and may overlap
    # the other side's last spectral step), so per-kernel durations overlap; the
    # achieved rate is the applies' algorithmic flops over the apply-phase window (first
    # apply start -> last apply end, CUDA events on the launching streams): conservative.
    achieved, kern_ms, kern_fl = (ap_fl / (ap_ms / 1e3) / 1e12 if ap_ms > 0 else 0.0), ap_ms, ap_fl
    achieved_windows = achieved
    span_ms = sum(r["t_ms"][6] for r in reps)  # stream: first apply start -> last apply end
    if batch and span_ms > 0:
        # in the stream the per-update windows overlap one another; the applies' busy
        # time is the span of the whole stream's applies (both apply streams busy
        # throughout it: tools/diag_batch.py measures 96-97 %)
        achieved, kern_ms = ap_fl / (span_ms / 1e3) / 1e12, span_ms
    launches = sum(r["kernel_launches"] for r in reps)
    traffic, traffic_src = None, None
    try:  # DRAM bytes per apply from the committed ncu capture of this workload
        with open(os.path.join(ROOT, "profiles", "ncu_traffic_r02.json")) as f:
            tj = json.load(f)
        if args.config == CFG_ID:
            traffic, traffic_src = tj["traffic_bytes_per_apply"], "profiles/ncu_traffic_r02.json: " + tj["label"]
    except Exception:
        pass
    roof = {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic, "traffic_source": traffic_src,
            "algorithmic_bytes_per_apply": 16.0 * (m * m + n * n) / 2.0,
            "kernel": "FMM Cauchy apply (fmm_gemm_kernel passes P2M, M2M bands, M2L, L2L bands, "
                      "L2P+P2P; operator build; Householder/passthrough), 4 applies per update",
            "flops_per_apply": kern_fl / max(n_apply, 1), "ms_per_apply": kern_ms / max(n_apply, 1),
            "apply_phase_ms_per_update": ap_ms / args.steps,
            "flops_exec_per_apply": ap_fx / max(n_apply, 1),
            "frac_executed": (ap_fx / ((kern_ms if kern_ms > 0 else 1.0) / 1e3) / 1e12) / FP64_PEAK_TFLOPS,
            "flops_note": "achieved counts the algorithmic flops of SURVEY §8(d) (level-by-level "
                          "P2M/M2M/M2L/L2L/L2P/P2P from the plan, plus the one-sided P2L/M2P terms that "
                          "replace near-field products: about 11 % fewer flops than the symmetric lists at "
                          "C3, so frac reads lower for a faster apply); the plan executes "
                          "flops_exec_per_apply (coarse levels in bands, DESIGN.md §4.4)",
            "timing": ("CUDA events on the launching streams around the apply phase of every update in "
                       "the timed region; svd1_update_batch: achieved = algorithmic apply flops over the "
                       "span from the stream's first apply start to its last apply end (achieved_windows: "
                       "over the sum of the per-update windows, which overlap one another); "
                       "the timed region (both sides' applies; window includes any overlap with the "
                       "other side's last spectral step)"),
            "apply_share_of_step": ap_ms / ms if ms else None,
            "achieved_windows": achieved_windows if batch else None,
            "apply_span_ms": span_ms if batch else None,
            "achieved_isolated": (seq or {}).get("apply_achieved_tflops"),
            "frac_isolated": ((seq or {}).get("apply_achieved_tflops") or 0.0) / FP64_PEAK_TFLOPS or None,
            "isolated_note": ("the same applies timed in the per-update API run (sequential_api) of the "
                              "same stream: there the next update's spectral kernels do not share the GPU "
                              "with them") if batch else None,
            "spectral_share_of_step": sp_ms / ms if ms else None,
            "peak_source": "measured fp64 DMMA sustained (profiles/fp64_peak_r01.jsonl); "
                           "MEASURED_PEAKS.json has no fp64 entry"}

    # end-to-end: a, b from pinned host memory each step, sigma read back each step
    e2e = None
    if not args.no_e2e:
        a_h = [x.cpu().pin_memory() for x, _ in ab]
        b_h = [y.cpu().pin_memory() for _, y in ab]
        a_d, b_d = torch.empty(m, dtype=torch.float64, device=dev), torch.empty(n, dtype=torch.float64, device=dev)
        s_h = torch.empty(m, dtype=torch.float64).pin_memory()
        if batch:
            A_h = torch.stack([a_h[t % len(ab)] for t in range(args.steps)]).pin_memory()
            B_h = torch.stack([b_h[t % len(ab)] for t in range(args.steps)]).pin_memory()
            A_d, B_d = torch.empty_like(A_h, device=dev), torch.empty_like(B_h, device=dev)

        def e2e_once():
            restore()
            torch.cuda.synchronize()
            barrier()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record(stream)
            if batch:  # every step's a, b copied from pinned host memory; sigma read back
                A_d.copy_(A_h, non_blocking=True)
                B_d.copy_(B_h, non_blocking=True)
                run(0, args.steps, A_d, B_d)
                s_h.copy_(sig, non_blocking=True)
            else:
                for t in range(args.steps):
                    a_d.copy_(a_h[t % len(ab)], non_blocking=True)
                    b_d.copy_(b_h[t % len(ab)], non_blocking=True)
                    step(t, a_d, b_d)
                    s_h.copy_(sig, non_blocking=True)
            f1.record(stream)
            torch.cuda.synchronize()
            barrier()
            ems = f0.elapsed_time(f1)
            if world > 1:
                tt = torch.tensor([ems], device=dev, dtype=torch.float64)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                ems = float(tt.item())
            return args.steps / (ems / 1e3)
        # three repetitions of the whole end-to-end stream (each: every step's copies inside
        # the timed region); the median is reported, all three listed.  One untimed pass first:
        # the per-update leg just before uses other buffers, and the first repetition after it
        # was sometimes 2-3x slow (one-off host/driver costs)
        e2e_once()
        reps_e2e = [e2e_once() for _ in range(3)]
        e2e = {"value": statistics.median(reps_e2e), "unit": UNIT, "h2d_bytes_per_step": 8 * (m + n),
               "d2h_bytes_per_step": (8 * m * -(-args.steps // 28)) / args.steps if batch else 8 * m,
               "repetitions": reps_e2e,
               "note": ("median of 3 repetitions of the timed stream; factors stay resident (streaming update); "
                        "every step's a, b copied from pinned host memory inside the timed region, "
                        "svd1_update_batch over the stream (chunks of <= 28), sigma read back after it" if batch else
                        "median of 3 repetitions; factors stay resident (streaming update); a, b copied from "
                        "pinned host memory and sigma read back every step through the public API")}

    # correctness check of the timed stream (outside the timed region): residual and
    # orthogonality against the explicitly accumulated A_hat (verification only)
    check = None
    if not args.no_check and world == 1:
        restore()
        A = (U0 * s0[None, :]) @ V0[:, :m].T
        run(0, args.steps)
        for t in range(args.steps):
            a_t, b_t = ab[t % len(ab)]
            A = A + torch.outer(a_t, b_t)
        res = float(torch.linalg.norm(A @ V[:, :m] - U * sig[None, :], dim=0).max() / sig[0])
        I = torch.eye(m, dtype=torch.float64, device=dev)
        Vc = V[:, :m] if thin else V
        In = torch.eye(Vc.shape[1], dtype=torch.float64, device=dev)
        orth = max(float((U.T @ U - I).abs().max()), float((Vc.T @ Vc - In).abs().max()))
        check = {"residual": res, "orthogonality": orth, "updates": args.steps,
                 "n_active_last": reps[-1]["n_active"], "max_secular_iter": max(max(r["max_iter"]) for r in reps),
                 "fmm_levels": reps[-1]["fmm_levels"], "fmm_max_near": reps[-1]["fmm_max_near"],
                 "mean_secular_evals": sum(sum(r["mean_iter"]) for r in reps) / (4 * len(reps))}
        if m * n <= 4096 * 4096:
            # sigma against the singular values of the accumulated A_hat (cuSOLVER, a library
            # reference for verification; the oracle parity is in tests/): Gram-normalised
            # error (reading D2), strict relative error over all sigma and over sigma >= 0.1 sigma_1
            sv = torch.linalg.svdvals(A)
            kk = min(m, n)
            ref, got = sv[:kk], sig[:kk]
            rel = (got - ref).abs() / ref.clamp_min(1e-300)
            top = ref >= 0.1 * ref[0]
            # strict relative error in units of its rounding sensitivity eps (sigma_1/sigma_i)^2 / 2
            # (a Gram eigenvalue perturbed by eps sigma_1^2)
            sens = (2.0 ** -52) * (ref[0] / ref.clamp_min(1e-300)) ** 2 / 2.0
            rs = rel / sens
            check["sigma_vs_svdvals"] = {
                "gram": float((got * got - ref * ref).abs().max() / (ref[0] * ref[0])),
                "max_rel": float(rel.max()), "max_rel_top": float(rel[top].max()),
                "rel_sens": float(rs.max()), "rel_sens_at": float(ref[int(rs.argmax())] / ref[0]),
                "note": ("reference: torch.linalg.svdvals of the explicitly accumulated A_hat (fp64), after all "
                         "the timed updates; sigma^2 are Gram eigenvalues (D2), so the error of a small sigma_i "
                         "scales with (sigma_1 / sigma_i)^2, and the FMM tolerance eps bounds the factors; rel_sens = "
                         "max_i rel_i / (eps (sigma_1/sigma_i)^2 / 2), the strict error in units of one rounding of "
                         "the Gram eigenvalue, accumulated over the whole stream of updates (the per-update parity "
                         "against the oracle is in tests/, profiles/parity_r02.jsonl)")}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and args.config == CFG_ID:
        from synth import config_inputs as ci
        import oracle.svd1_oracle as OM
        cin = ci(CFG_ID)
        t_all = oracle_update_times(cin, 2)          # two whole updates, all host cores
        t_one = oracle_update_times(cin, 1, threads=1)  # one whole update, one core
        cpu = {"value": len(t_all) / sum(t_all), "unit": UNIT, "cores": OM.THREADS, "kind": "oracle",
               "sample": ("updates 0-1 of the C3 stream, each a whole update by the oracle (literal STEP-1 "
                          "products, bisection over all roots, Loewner, explicit products on all 4096 rows of U "
                          "and V; numpy fp64, oracle and BLAS threads on every host core); nothing sampled"),
               "seconds_per_update": t_all, "one_core": {"value": 1.0 / t_one[0], "unit": UNIT, "cores": 1,
                                                          "seconds_per_update": t_one[0]},
               **cpu_info()}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded, BASELINE.json C3 recipe)",
                "config": {"workload": WORKLOAD, "m": m, "n": n, "eps": cfg["eps"], "p": reps[-1]["p"],
                           "updates_in_stream": cfg["updates"],
                           "warmup_updates": 2 * max(args.warmup, args.steps),
                           "l2": (f"inputs larger than L2 (U + V = {8 * (m * m + n * n) / 2**20:.0f} MiB > 126 MB)"
                                  if 8 * (m * m + n * n) > 126e6 else
                                  f"inputs fit in L2 ({8 * (m * m + n * n) / 2**20:.1f} MiB); no flush"),
                           "parallelism": f"row-sharded x{world}" if world > 1 else "1 GPU",
                           "api": "svd1_update_batch (pipelined stream)" if batch else "svd1_update",
                           "fused_side": bool(args.fused),
                           "thin_v": thin},
                "sequential_api": seq,
                "clocks": clk.summary(), "e2e": e2e, "gpu_launches": launches, "roofline": roof,
                "allocations_in_timed_region": sum(r.get("allocations", 0) for r in reps),
                "cpu_baseline": cpu, "check": check,
                "spectral_ms_per_step": sp_ms / args.steps, "apply_ms_per_step": ap_ms / args.steps,
                "host_phase_ms": [sum(r["t_ms"][i] for r in reps) / args.steps for i in range(5)]}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
