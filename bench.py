#!/usr/bin/env python
"""Benchmark of the RQRCP hot path (BASELINE.json metric: "RQRCP fp64
GFLOP/s and sec-to-rank-k at 1/2/4/8 B200; % of FP64 peak").

A step = one full rqrcp_factor (all hot-path rows S0..S7 of SURVEY.md §8(a))
on the configuration's synthetic A, resident in HBM.  Default workload:
configs[1] = C2 (4096^2, k=512, b=64, p=10, A iid N(0,1)).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

Prints ONE JSON line on rank 0.  --impl reference times the CPU oracle (the
deliberately slow, unblocked reference of this tier) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "rqrcp_fp64_gflops"
UNIT = "GFLOP/s"
MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FP64_NOMINAL_OVER_BF16 = 45.0 / 2250.0  # blackwell guide: B200 FP64 tensor 45 TF vs bf16 2.25 PF dense
PROFILE_TRAFFIC = os.path.join(ROOT, "profiles", "traffic_r01.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-budget-s", type=float, default=20.0)
    return ap.parse_args()


def flops_of(cfg):
    import paper_1804_05138_b200 as rq
    return rq.rqrcp_flops(cfg["m"], cfg["n"], cfg["k"], cfg["b"], cfg["p"])


def alg_flops_host(cfg):
    """F_alg from the closed forms; used by the reference arm
    (which must not load the CUDA library)."""
    m, n, k, b, p = cfg["m"], cfg["n"], cfg["k"], cfg["b"], cfg["p"]
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


MICROBENCH = os.path.join(ROOT, "profiles", "r01_microbench.json")


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


def cpu_baseline(cfg, budget_s):
    """The oracle as it stands on this host's cores: full factorizations of the
    same workload, repeated until ~budget_s (at least one)."""
    import inputs
    import oracle
    A = inputs.make(cfg["kind"], cfg["m"], cfg["n"], cfg["seed"]).numpy()
    f = alg_flops_host(cfg)
    oracle.lib()
    times = []
    t_all = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        oracle.rqrcp(A, cfg["k"], cfg["b"], cfg["p"], seed=cfg["seed"])
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_all > budget_s or len(times) >= 20:
            break
    t = sum(times) / len(times)
    thr = int(os.environ.get("OMP_NUM_THREADS", host_cores()))
    return {"value": f / t / 1e9, "unit": UNIT, "cores": thr, "kind": "oracle",
            "sample": f"{len(times)} full {cfg['name']} factorizations ({cfg['m']}x{cfg['n']}, k={cfg['k']}), "
                      f"mean {t:.2f} s each"}


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import inputs
    import oracle
    A = inputs.make(cfg["kind"], cfg["m"], cfg["n"], cfg["seed"]).numpy()
    oracle.lib()
    for _ in range(args.warmup):
        oracle.rqrcp(A, cfg["k"], cfg["b"], cfg["p"], seed=cfg["seed"])
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.rqrcp(A, cfg["k"], cfg["b"], cfg["p"], seed=cfg["seed"])
    dt = (time.perf_counter() - t0) / args.steps
    f = alg_flops_host(cfg)
    v = f / dt / 1e9
    thr = int(os.environ.get("OMP_NUM_THREADS", host_cores()))
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["name"], "m": cfg["m"], "n": cfg["n"], "k": cfg["k"], "b": cfg["b"],
                   "p": cfg["p"], "input": cfg["kind"], "sec_to_rank_k": dt},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": thr, "kind": "oracle",
                         "sample": f"full {cfg['name']} factorization per step (plain unblocked C oracle)"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    args = parse()
    import inputs
    cfg = dict(inputs.CONFIGS[args.config])
    cfg["name"] = args.config
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist

    import paper_1804_05138_b200 as rq
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    m, n, k, b, p, seed = cfg["m"], cfg["n"], cfg["k"], cfg["b"], cfg["p"], cfg["seed"]

    # one factorization of the config matrix per step; with N GPUs it is
    # sharded 1D column-block-cyclic (block b) and the library exchanges the
    # sample / panel / swapped columns over NCCL (strong scaling)
    A0 = inputs.make(cfg["kind"], m, n, seed, device=dev)
    uid = None
    if world > 1:
        mine = torch.tensor(rq.shard_columns(n, b, world, rank), device=dev)
        A0 = inputs.fortran(A0.index_select(1, mine))
        obj = [rq.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    n_loc = A0.shape[1]
    A = A0.t().clone().t()  # working copy, column-major
    ctx = rq.RQRCP(max_m=m, max_n=n, max_b=b, max_p=p, device=local, nranks=world, rank=rank, nccl_uid=uid)
    jpvt = torch.empty(n, dtype=torch.int64, device=dev)
    tau = torch.empty(k, dtype=torch.float64, device=dev)
    fl = flops_of(cfg)
    F = fl["total"]

    def step():
        A.copy_(A0)
        rc, rk = ctx.factor_raw(A.data_ptr(), m, m, n, k, b, p, seed, jpvt.data_ptr(), tau.data_ptr())
        if rc not in (0, rq.RQRCP_W_RANK_DEFICIENT):
            raise RuntimeError(f"rqrcp_factor failed: {rc}")

    for _ in range(args.warmup):
        step()
    sampler = ClockSampler(local)
    sampler.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    phases = {}
    launches = 0
    e0.record(ctx.stream)
    for _ in range(args.steps):
        step()
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    # per-phase times: the library's events of the last step (every step is the
    # same workload); read after the timed region, outside it
    t = ctx.timings()
    for kk, v in t.items():
        if kk.endswith("_ms"):
            phases[kk] = v * args.steps
    launches = (t["kernel_launches"] + 1) * args.steps  # + the restore copy
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    value = F / (ms * 1e-3) / 1e9  # one factorization of the whole matrix per step

    # dominant kernel roofline: the trailing update (FP64 DMMA contraction)
    tr_ms = phases.get("trailing_ms", 0.0) / args.steps
    tr_flops = 0.0
    for i in range(0, k, b):
        bb = min(b, k - i)
        mp, npp = m - i, n - i - bb
        bbpad = (bb + 7) // 8 * 8
        tr_flops += (4.0 * mp * bb * npp + 2.0 * bb * bb * npp) / world  # this rank's share
    peak, peak_src = fp64_peak()
    achieved = tr_flops / (tr_ms * 1e-3) / 1e12 if tr_ms > 0 else 0.0
    traffic = None
    try:  # ncu dram__bytes_read + dram__bytes_write of the S5 kernels per panel (profiles/traffic_r01.json)
        traffic = json.load(open(PROFILE_TRAFFIC)).get(args.config, {}).get("dram_bytes_per_panel_trailing")
    except Exception:
        pass
    # algorithmic S5 bytes per panel (unfused: A22 read twice, written once)
    alg_bytes = 0.0
    for i in range(0, k, b):
        bb = min(b, k - i)
        alg_bytes += 24.0 * (m - i) * (n - i - bb) / world
    alg_bytes /= max(1, (k + b - 1) // b)
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak if peak else None, "traffic": traffic,
                "kernel": "S5 trailing update (W = V^T A22, W2 = -T^T W, A22 += V W2; DMMA.8x8x4)",
                "peak_source": peak_src, "traffic_unit": "DRAM bytes per panel (ncu, S5 kernels)",
                "algorithmic_bytes_per_panel": alg_bytes}
    whole_frac = (F / (ms * 1e-3) / 1e12) / peak

    e2e = None
    if not args.no_e2e and world == 1:
        Ah = torch.empty(n, m, dtype=torch.float64, pin_memory=True).t()
        Ah.copy_(A0.cpu())
        Ao = torch.empty(n, m, dtype=torch.float64, pin_memory=True).t()
        jh = torch.empty(n, dtype=torch.int64, pin_memory=True)
        th = torch.empty(k, dtype=torch.float64, pin_memory=True)
        import ctypes
        L = rq.lib()
        rk = ctypes.c_int64()
        L.rqrcp_factor_host(ctx._h, Ah.data_ptr(), m, m, n, k, b, p, seed, Ao.data_ptr(), jh.data_ptr(),
                            th.data_ptr(), ctypes.byref(rk))
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            rc = L.rqrcp_factor_host(ctx._h, Ah.data_ptr(), m, m, n, k, b, p, seed, Ao.data_ptr(), jh.data_ptr(),
                                     th.data_ptr(), ctypes.byref(rk))
            assert rc in (0, rq.RQRCP_W_RANK_DEFICIENT), rc
        te = (time.perf_counter() - t0) / args.e2e_steps
        e2e = {"value": F / te / 1e9, "unit": UNIT, "h2d_bytes_per_step": 8 * m * n,
               "d2h_bytes_per_step": 8 * m * n + 8 * n + 8 * k, "ms_per_step": te * 1e3}

    dgemm = None
    try:
        dgemm = measured_dgemm_tflops(dev)
    except Exception:
        pass

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, args.cpu_budget_s)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["name"], "m": m, "n": n, "k": k, "b": b, "p": p, "input": cfg["kind"],
                       "sec_to_rank_k": ms * 1e-3, "flops_per_step": F,
                       "l2": "A (8mn bytes) restored from a pristine copy every step, inputs >= L2",
                       "parallelism": f"1d-block-cyclic-nccl{world}" if world > 1 else "single"},
            "roofline": roofline,
            "fp64_frac_whole_step": whole_frac,
            "fp64_dgemm_measured_tflops": dgemm,
            "phases_ms_per_step": {kk: v / args.steps for kk, v in phases.items()},
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
