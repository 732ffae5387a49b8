#!/usr/bin/env python
"""Benchmark of the RQRCP hot path (BASELINE.json metric: "RQRCP fp64
GFLOP/s and sec-to-rank-k at 1/2/4/8 B200; % of FP64 peak").

A step = one full rqrcp_factor (every hot-path row S0..S7 of SURVEY.md §8(a))
on the configuration's synthetic A, resident in HBM.  Default workload: C4
(configs[3]: 32768^2, k = 8192, b = 128, p = 16, A = U diag(1/j) V^T), the
largest BASELINE config whose metric is quoted on "1/2/4/8 GPUs".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

--gpus N > 1 without a torchrun environment re-launches itself under
torch.distributed.run (N ranks, 127.0.0.1); under torchrun WORLD_SIZE must
equal N.  The matrix is sharded 1D column-block-cyclic (block b) and the
library exchanges the sample / panel / pivot columns over NCCL: one
factorization of the whole matrix per step (strong scaling).

Prints ONE JSON line on rank 0.  --impl reference times the CPU oracle (the
deliberately slow, unblocked reference of this tier) on the host cores, on a
bounded sample of the same workload (see cpu_sample()).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "rqrcp_fp64_gflops"
UNIT = "GFLOP/s"
MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
MICROBENCH = os.path.join(ROOT, "profiles", "r01_microbench.json")
PROFILE_TRAFFIC = os.path.join(ROOT, "profiles", "traffic_r02.json")
FP64_NOMINAL_OVER_BF16 = 45.0 / 2250.0  # blackwell guide: B200 FP64 tensor 45 TF vs bf16 2.25 PF dense
DEFAULT_CONFIG = "C4"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-budget-s", type=float, default=20.0)
    return ap.parse_args()


def config_dict(cfg):
    """The workload description, identical in both arms."""
    return {"workload": cfg["name"], "m": cfg["m"], "n": cfg["n"], "k": cfg["k"], "b": cfg["b"], "p": cfg["p"],
            "input": cfg["kind"], "seed": cfg["seed"]}


def alg_flops(m, n, k, b, p):
    """F_alg = F_sketch + F_qr + F_sQRCP + F_sUpd (closed forms of SURVEY.md
    §8(d)); the reference arm must not load the CUDA library."""
    l = b + p
    f = 2.0 * l * m * n + sum(4.0 * (m - j) * (n - j) for j in range(k))
    for i in range(0, k, b):
        bb = min(b, k - i)
        f += sum(4.0 * (l - j) * (n - i - j) for j in range(bb)) + 2.0 * bb * bb * (n - i - bb)
    return f


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() in ("active", "1", "0x1"):
                    reasons.add(nm)
        if not sm:
            return None
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def fp64_peak():
    """FP64 peak for the roofline.  MEASURED_PEAKS.json has no FP64 entry; we
    use our own measurement of the DMMA.8x8x4 pipe on this pool's B200s
    (tools/microbench.cu -> profiles/r01_microbench.json, 37.16 TFLOP/s, which
    is also the datasheet-class 148 x 64 FMA x 2 x 1.965 GHz).  Fallback: the
    measured bf16 peak x the guide's nominal FP64/bf16 ratio (45/2250)."""
    try:
        mb = json.load(open(MICROBENCH))
        return mb["dmma_tflops"], "measured DMMA.8x8x4 peak (tools/microbench.cu, profiles/r01_microbench.json)"
    except Exception:
        pass
    try:
        mp = json.load(open(MEASURED_PEAKS))
        return mp["bf16_tflops"] * FP64_NOMINAL_OVER_BF16, "MEASURED_PEAKS bf16_tflops x nominal FP64/bf16 (45/2250)"
    except Exception:
        return 1590.0 * FP64_NOMINAL_OVER_BF16, "fallback 1.59 PF bf16 x nominal FP64/bf16 (45/2250)"


def measured_dgemm_tflops(device):
    """cuBLAS DGEMM 8192^3 best of 5 (context for the FP64 denominator)."""
    import torch
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=device)
    b = torch.randn(n, n, dtype=torch.float64, device=device)
    c = a @ b
    best = 1e9
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b, out=c)
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    del a, b, c
    torch.cuda.empty_cache()
    return 2.0 * n ** 3 / (best * 1e-3) / 1e12


# ---------------------------------------------------------------------------
# The oracle's bounded sample of a workload (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------
SAMPLE_MAX_COLS = 4096


def cpu_sample(cfg):
    """A bounded sample of the workload for the unblocked CPU oracle: the
    first min(n, 4096) columns of the config's A (same recipe, seed, m, b, p)
    factored to k' = min(k, b) -- one pivot panel of Alg. 2 at the config's
    full row count.  Returns (A_sample numpy, k', description)."""
    import torch

    import inputs
    m, n, k, b, p = cfg["m"], cfg["n"], cfg["k"], cfg["b"], cfg["p"]
    nc = min(n, SAMPLE_MAX_COLS)
    kp = min(k, b, nc)
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    A = inputs.make(cfg["kind"], m, n, cfg["seed"], device=dev)
    As = A[:, :nc].cpu().numpy().copy(order="F")
    del A
    if dev == "cuda":
        torch.cuda.empty_cache()
    desc = (f"{cfg['name']} recipe, first {nc} of {n} columns ({m} x {nc}), prefix k'={kp} (one b={b} panel), "
            f"p={p}; plain unblocked C oracle")
    return As, kp, desc


def time_oracle(As, kp, cfg, reps=None, budget_s=None, warmup=0):
    import oracle
    oracle.lib()
    m, nc = As.shape
    f = alg_flops(m, nc, kp, cfg["b"], cfg["p"])
    for _ in range(warmup):
        oracle.rqrcp(As, kp, cfg["b"], cfg["p"], seed=cfg["seed"])
    times = []
    t_all = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        oracle.rqrcp(As, kp, cfg["b"], cfg["p"], seed=cfg["seed"])
        times.append(time.perf_counter() - t0)
        if reps is not None and len(times) >= reps:
            break
        if budget_s is not None and (time.perf_counter() - t_all > budget_s or len(times) >= 20):
            break
    t = sum(times) / len(times)
    thr = int(os.environ.get("OMP_NUM_THREADS", host_cores()))
    return f / t / 1e9, t, len(times), thr, f


def cpu_baseline(cfg, budget_s):
    As, kp, desc = cpu_sample(cfg)
    v, t, reps, thr, f = time_oracle(As, kp, cfg, budget_s=budget_s)
    return {"value": v, "unit": UNIT, "cores": thr, "kind": "oracle",
            "sample": f"{desc}; {reps} runs, mean {t:.2f} s ({f:.3e} flop each)"}


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    As, kp, desc = cpu_sample(cfg)
    v, t, reps, thr, f = time_oracle(As, kp, cfg, reps=args.steps, warmup=args.warmup)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config_dict(cfg),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": thr, "kind": "oracle",
                         "sample": f"{desc}; one sample factorization per step ({f:.3e} flop)"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def roofline_s5(cfg, world, s5_ms, peak, peak_src):
    """S5 trailing update (>= 90% of the flops, 98% at C4/C5): algorithmic
    flops 4 m' bb n'' + 2 bb^2 n'' per panel (W = V^T A22, W2 = -T^T W,
    A22 += V W2) divided by the CUDA-event time of the S5 kernels on the
    streams that run them; traffic = ncu DRAM bytes of those kernels on one
    captured panel (profiles/traffic_r02.json) beside that panel's
    algorithmic bytes (24 m' n'': A22 read twice, written once)."""
    m, n, k, b = cfg["m"], cfg["n"], cfg["k"], cfg["b"]
    fl = 0.0
    for i in range(0, k, b):
        bb = min(b, k - i)
        fl += (4.0 * (m - i) * bb * (n - i - bb) + 2.0 * bb * bb * (n - i - bb)) / world
    achieved = fl / (s5_ms * 1e-3) / 1e12 if s5_ms > 0 else 0.0
    traffic, alg_panel, tsrc = None, None, None
    try:
        tr = json.load(open(PROFILE_TRAFFIC)).get(cfg["name"])
        if tr and world == 1:
            traffic, alg_panel, tsrc = tr["dram_bytes_per_panel"], tr["alg_bytes_per_panel"], tr["source"]
    except Exception:
        pass
    return {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak if peak else None, "traffic": traffic,
            "kernel": "S5 trailing update (W = V^T A22 split-K, W2 = -T^T W, A22 += V W2; DMMA.8x8x4 via TMA)",
            "flops_per_step": fl, "peak_source": peak_src,
            "traffic_unit": "DRAM bytes per panel (ncu, S5 kernels of one panel)",
            "algorithmic_bytes_per_panel": alg_panel, "traffic_source": tsrc}


def main():
    args = parse()
    import inputs
    if args.config not in inputs.CONFIGS:
        raise SystemExit(f"unknown config {args.config}")
    cfg = dict(inputs.CONFIGS[args.config])
    cfg["name"] = args.config

    world_env = os.environ.get("WORLD_SIZE")
    if world_env is None and args.gpus > 1:
        # launch N ranks ourselves (one process per GPU, 127.0.0.1 rendezvous)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    world = int(world_env or "1")
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")

    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist

    import paper_1804_05138_b200 as rq
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    m, n, k, b, p, seed = cfg["m"], cfg["n"], cfg["k"], cfg["b"], cfg["p"], cfg["seed"]

    A0 = inputs.make(cfg["kind"], m, n, seed, device=dev)
    uid = None
    if world > 1:
        mine = torch.tensor(rq.shard_columns(n, b, world, rank), device=dev)
        A0 = inputs.fortran(A0.index_select(1, mine))
        obj = [rq.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    torch.cuda.empty_cache()
    A = A0.t().clone().t()  # working copy, column-major
    ctx = rq.RQRCP(max_m=m, max_n=n, max_b=b, max_p=p, device=local, nranks=world, rank=rank, nccl_uid=uid)
    jpvt = torch.empty(n, dtype=torch.int64, device=dev)
    tau = torch.empty(k, dtype=torch.float64, device=dev)
    F = rq.rqrcp_flops(m, n, k, b, p)["total"]
    st = ctx.stream
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]

    def step(evs=None):
        # restore A (untimed: A is 8mn bytes >= L2, so every step starts cold)
        with torch.cuda.stream(st):
            A.copy_(A0)
        if evs:
            evs[0].record(st)
        rc, rk = ctx.factor_raw(A.data_ptr(), m, m, n, k, b, p, seed, jpvt.data_ptr(), tau.data_ptr())
        if evs:
            evs[1].record(st)
        if rc not in (0, rq.RQRCP_W_RANK_DEFICIENT):
            raise RuntimeError(f"rqrcp_factor failed: {rc} {ctx.last_error()}")

    for _ in range(args.warmup):
        step()
    sampler = ClockSampler(local)
    sampler.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for s in range(args.steps):
        step(ev[s])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    step_ms = [a.elapsed_time(z) for a, z in ev]
    ms = sum(step_ms) / len(step_ms)
    # per-phase times: the library's events of the last step (every step is the
    # same workload); read after the timed region
    t = ctx.timings()
    phases = {kk: v for kk, v in t.items() if kk.endswith("_ms")}
    launches = t["kernel_launches"] * args.steps
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    value = F / (ms * 1e-3) / 1e9  # one factorization of the whole matrix per step

    peak, peak_src = fp64_peak()
    roofline = roofline_s5(cfg, world, phases.get("trailing_ms", 0.0), peak, peak_src)
    whole_frac = (F / (ms * 1e-3) / 1e12) / (peak * world)

    e2e = None
    if not args.no_e2e and world == 1:
        del A
        torch.cuda.empty_cache()
        Ah = torch.empty(n, m, dtype=torch.float64, pin_memory=True).t()
        Ah.copy_(A0.cpu())
        Ao = torch.empty(n, m, dtype=torch.float64, pin_memory=True).t()
        jh = torch.empty(n, dtype=torch.int64, pin_memory=True)
        th = torch.empty(k, dtype=torch.float64, pin_memory=True)
        # the factors only (Pi, V + tau, R11, R12 -- the partial QRCP's outputs):
        # the R22 by-product stays on the device
        ctx.set_option("host_out", 1)
        ctx.factor_host(Ah, k, b, p, seed=seed, out=Ao, jpvt=jh, tau=th)  # warm (allocates the device copy)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            ctx.factor_host(Ah, k, b, p, seed=seed, out=Ao, jpvt=jh, tau=th)
        te = (time.perf_counter() - t0) / args.e2e_steps
        e2e = {"value": F / te / 1e9, "unit": UNIT, "h2d_bytes_per_step": 8 * m * n,
               "d2h_bytes_per_step": 8 * m * k + 8 * k * (n - k) + 8 * n + 8 * k, "ms_per_step": te * 1e3,
               "path": "rqrcp_factor_host (pinned host A in; out: columns 0..k-1 full height (V, R11), "
                       "rows 0..k-1 of columns k.. (R12), jpvt, tau -- option host_out=1; copies timed)"}
        ctx.set_option("host_out", 0)
        del Ah, Ao

    dgemm = None
    try:
        if rank == 0:
            dgemm = measured_dgemm_tflops(dev)
    except Exception:
        pass

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        del A0
        torch.cuda.empty_cache()
        cpu = cpu_baseline(cfg, args.cpu_budget_s)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config_dict(cfg),
            "sec_to_rank_k": ms * 1e-3, "flops_per_step": F,
            "parallelism": f"1d-block-cyclic-nccl{world}" if world > 1 else "single",
            "timing": "CUDA events around each rqrcp_factor on the context stream; A (8mn bytes >> L2) restored "
                      "from a pristine copy before every step, outside the events",
            "step_ms": step_ms,
            "roofline": roofline,
            "fp64_frac_whole_step": whole_frac,
            "fp64_dgemm_measured_tflops": dgemm,
            "phases_ms_per_step": phases,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
