#!/usr/bin/env python
"""GFORS hot-path benchmark (BASELINE.json metric) on B200.

One "step" = one Alg. 1 sampling block over the whole hot path: k_int PDHG
iterations (dual + primal kernels), the trigger indicators, k_r rounds of [Philox sampling of
k_b candidates per rank + feasibility + objective + argmin/incumbent], CheckHalt/UpdatePenalty.
The timed region is one gfors_run of exactly K blocks (halting disabled, fixed max_iters), i.e.
one CUDA-graph launch whose WHILE node runs the K blocks on the device.

value  = sampled candidates evaluated per second, whole job (all ranks), device time (CUDA events,
         max over ranks).  pdhg_iters_per_s is the same clock over the replicated PDHG trajectory.
e2e    = the same metric through the public C-ABI calls from HOST (pinned) buffers: load (H2D of the
         instance) + preprocess + run + best_incumbent (D2H), timed end to end.
Workload: BASELINE config 5 by default (set cover n=5e6, m=1e6, ~5e7 nonzeros), synthetic, seeded.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--precision 32|64] [--k-b 128]
    python bench.py --impl reference ...   (the CPU oracle as the reference arm)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PDHG iters/s and sampled candidates evaluated/s; time-to-incumbent at 1/2/4/8 B200"
# measured random-gather ceilings (x1e9 gathers/s) on B200, profiles/gather_bench.cu ->
# profiles/r02_gather_microbench.txt: 4-byte elements from a 20 MB vector (x-bar of the PDHG dual,
# cp.async 2048-chunk recipe) and 16-byte elements from an 80 MB vector (the k_b = 128 sample batch
# read by the feasibility kernel, cp.async 1024-chunk recipe)
GATHER_CEILING_G = 253.9
GATHER16_CEILING_G = 211.6
L2_READ_GBS = 15580.0  # streaming read of a 48 MB L2-resident buffer (same microbenchmark)
UNIT = "candidates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--precision", type=int, default=32, choices=(32, 64))
    ap.add_argument("--k-b", type=int, default=128)
    ap.add_argument("--k-int", type=int, default=10)
    ap.add_argument("--impl", default="gfors", choices=("gfors", "reference"))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-row-shard", action="store_true", help="N > 1: replicate the PDHG dual instead of row-sharding it")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-tti", action="store_true", help="skip the time-to-incumbent solves of configs 1-4")
    ap.add_argument("--profile-blocks", type=int, default=0, help="eager blocks replayed with per-kernel events (0 = --steps)")
    ap.add_argument("--no-f1", action="store_true", help="skip the dense-Q max-cut leg (next row f1, config 6)")
    ap.add_argument("--f1-steps", type=int, default=50)
    ap.add_argument("--no-f2", action="store_true", help="skip the TU-reformulation facility-location leg (next row f2, config 7)")
    ap.add_argument("--f2-iters", type=int, default=3000)
    ap.add_argument("--no-f3", action="store_true", help="skip the customised-sampler 3D-assignment leg (next row f3, config 8)")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the PDHG-only and sampling-only legs (the ncu launch list of the step uses this)")
    ap.add_argument("--f3-iters", type=int, default=2000)
    return ap.parse_args()


# ------------------------------------------------------------------------------------------------
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), "measured (MEASURED_PEAKS.json hbm_gbs)", d
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)", {}


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region (B200_PROFILING.md recipe).

    NVML in a background thread every 10 ms (the device is found by UUID, so CUDA_VISIBLE_DEVICES
    remapping cannot point it at another GPU); only samples inside [region_begin, region_end] count.
    Falls back to `nvidia-smi -lms 100` when NVML is unavailable."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.thread = None
        self.samples = []  # (perf_counter, sm_mhz, max_mhz, reasons)
        self.t0 = self.t1 = None

    def _nvml_handle(self):
        import pynvml
        import torch
        pynvml.nvmlInit()
        try:
            uuid = str(torch.cuda.get_device_properties(self.idx).uuid)
            return pynvml, pynvml.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.idx)

    def start(self):
        import threading
        try:
            nv, h = self._nvml_handle()
            bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                    nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
            mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self.stop_flag = threading.Event()

            def loop():
                while not self.stop_flag.is_set():
                    sm = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((time.perf_counter(), sm, mx,
                                         [nm for nm, b in zip(self.NAMES, bits) if r & b]))
                    time.sleep(0.01)
            self.thread = threading.Thread(target=loop, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.thread = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def region_begin(self):
        self.t0 = time.perf_counter()

    def region_end(self):
        self.t1 = time.perf_counter()

    def stop(self):
        if self.thread is not None:
            self.stop_flag.set()
            self.thread.join(timeout=5)
            inside = [s for s in self.samples
                      if (self.t0 is None or s[0] >= self.t0) and (self.t1 is None or s[0] <= self.t1)]
            sm = [s[1] for s in inside]
            reasons = sorted({nm for s in inside for nm in s[3]})
            return {"sm_mhz": statistics.median(sm) if sm else None,
                    "sm_max_mhz": self.samples[0][2] if self.samples else None,
                    "reasons": reasons, "samples": len(sm), "source": "nvml, 10 ms, timed region only"}
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], None, set()
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0])); mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(self.NAMES, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi -lms 100"}


def algorithmic_bytes(inst_meta, fb):
    """Algorithmic HBM bytes per launch of the two PDHG kernels.
    fb = bytes per iterate element.  Indices int32, pointers int64, SIGN matrices carry no values;
    every vector is counted once (gathers assumed cache hits); g and r-hat are fp64."""
    n, m, nnz = inst_meta["n"], inst_meta["m"], inst_meta["nnz"]
    val = inst_meta["val_bytes"]
    dual = nnz * (4 + val) + 8 * (m + 1) + n * fb + m * (fb + fb + fb + 8 + 8 + 1)
    primal = nnz * (4 + val) + 8 * (n + 1) + m * fb + n * (fb + fb + fb + fb)
    return {"pdhg_dual": dual, "pdhg_primal": primal}


def make_instance(cfg, seed):
    from gen import instances as G
    return G.make_config(cfg, seed)


def inst_meta(inst):
    vals = inst["k_val"]
    sign_rows = True
    ptr = inst["k_rowptr"]
    # +-1 single-sign rows -> SIGN storage (no value bytes)
    if not np.all(np.abs(vals) == 1.0):
        sign_rows = False
    else:
        first = np.repeat(vals[ptr[:-1]][np.diff(ptr) > 0], np.diff(ptr)[np.diff(ptr) > 0])
        sign_rows = bool(np.all(vals == first))
    i8 = np.all(vals == np.round(vals)) and np.all(np.abs(vals) <= 127)
    return {"n": int(inst["n"]), "m": int(inst["m"]), "nnz": int(ptr[-1]),
            "qnnz": int(inst["q_rowptr"][-1]) if inst.get("q_rowptr") is not None else 0,
            "val_bytes": 0 if sign_rows else (1 if i8 else 8)}


# ------------------------------------------------------------------------------------------------
def _oracle_one_block(o, k_int, k_b, seed):
    """One real Alg. 1 block of the oracle as it stands (orc_run: k_int PDHG iterations, sampling of k_b
    candidates, EvalBest, indicators, CheckHalt); returns its wall time."""
    from oracle import oracle as O
    prm = O.params(k_int=k_int, k_b=k_b, max_iters=k_int, tol_primal=-1.0, tol_dual=-1.0, tol_binary=-1.0,
                   stall_rel=-1.0, seed=seed)
    t0 = time.perf_counter()
    o.run(prm)
    return time.perf_counter() - t0


def oracle_baseline(inst, k_int, seed=20251030, max_procs=32):
    """cpu_baseline: the CPU oracle as it stands on the FULL instance, one real Alg. 1 block with
    k_b = 64 candidates (the bounded sample: 64 instead of 128 candidates per block; Preprocess
    bounded to 5 power iterations, excluded from the time as in PAPER L193).
    1 core: one process.  All host cores: the same block in os.cpu_count() forked processes at
    once (copy-on-write instance, each its own candidates: weak scaling over cores), candidates/s =
    procs * 64 / wall."""
    from oracle import oracle as O
    o = O.Oracle(inst)
    o.preprocess(max_iter=5)
    t1 = _oracle_one_block(o, k_int, 64, seed)
    procs = max(1, min(os.cpu_count() or 1, max_procs))
    all_cores = None
    if procs > 1 and hasattr(os, "fork"):
        t0 = time.perf_counter()
        pids = []
        for p in range(procs):
            pid = os.fork()
            if pid == 0:
                try:
                    _oracle_one_block(o, k_int, 64, seed + p)
                finally:
                    os._exit(0)
            pids.append(pid)
        ok = all(os.waitpid(pid, 0)[1] == 0 for pid in pids)
        wall = time.perf_counter() - t0
        if ok:
            all_cores = {"value": procs * 64 / wall, "cores": procs, "wall_s": wall}
    try:
        model = [l.split(":", 1)[1].strip() for l in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines()
                 if l.startswith("Model name")][0]
    except Exception:
        model = None
    return {"t_block": t1, "value": 64 / t1, "all_cores": all_cores, "cpu_model": model,
            "sample": (f"oracle (1 thread, as it stands) Alg. 1 on the full config instance: one block of {k_int} PDHG "
                       f"iterations + sampling and EvalBest of 64 candidates (k_b = 64 instead of 128) + indicators + "
                       f"CheckHalt; Preprocess bounded to 5 power iterations and not timed")}


def scaled_instance(cfg, seed, f):
    """The same generator recipe at a fraction f of the size (used to bound the oracle's time)."""
    from gen import instances as G
    if cfg == 5:
        return G.set_cover(max(50, int(1_000_000 * f)), max(100, int(5_000_000 * f)), 2, 98, seed, f"config5_x{f:.4g}")
    if cfg == 3:
        return G.multi_knapsack(max(100, int(100_000 * f)), 50, 0.5, seed, f"config3_x{f:.4g}")
    if cfg == 4:
        a = max(4, int(400 * f ** 0.5)); b = max(5, int(500 * f ** 0.5))
        return G.assignment_bqp(a, b, 4, seed, f"config4_x{f:.4g}")
    if cfg == 2:
        return G.max_independent_set(max(50, int(10_000 * f)), 1e-3 / max(f, 1e-3), seed, name=f"config2_x{f:.4g}")
    return G.make_config(cfg, seed)


def oracle_small_configs(seed):
    """the oracle as it stands (1 thread) on configs 1-4 — s per PDHG iteration
    (sampling off; 1000 iterations each) and s per candidate (sampling + EvalBest of 128 candidates around
    the final iterate)."""
    from oracle import oracle as O
    out = {}
    for cfg, iters in ((1, 1000), (2, 1000), (3, 1000), (4, 1000)):
        inst_c = make_instance(cfg, seed)
        o = O.Oracle(inst_c)
        o.preprocess(max_iter=50)
        o.state_init()
        tau = 0.99 ** 0.5
        t0 = time.perf_counter()
        for _ in range(iters):
            o.step(1e-3, tau, tau)
        t_it = (time.perf_counter() - t0) / iters
        x, _, _ = o.get_state()
        t0 = time.perf_counter()
        bits = O.sample(np.clip(x, 0.0, 1.0), 20251030, 0, 0, 2)
        o.eval(bits)
        t_c = (time.perf_counter() - t0) / 128
        out[f"config{cfg}"] = {"s_per_iteration": t_it, "iterations_timed": iters, "s_per_candidate": t_c,
                               "candidates_timed": 128}
    return out


def run_reference(args):
    """Reference arm: the CPU oracle as it stands, on the host cores, same metric/unit/config.
    Each step runs one real oracle Alg. 1 block (k_int PDHG iterations + k_r*k_b candidates) on a
    fraction f of the workload (same generator recipe), sized so the whole run ends in ~3 minutes;
    the per-step time is scaled by 1/f to the full workload (cost is linear in the instance size)."""
    from oracle import oracle as O
    rank, world, _ = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        if rank != 0:
            dist.barrier()
            dist.destroy_process_group()
            return
    k_b_total = args.k_b * args.gpus
    nsteps = args.steps + args.warmup
    budget = 150.0
    full_block_est = {5: 100.0, 4: 1.0, 3: 15.0, 2: 0.3, 1: 0.001}.get(args.config, 10.0) * k_b_total / 128.0
    f = min(1.0, (budget / nsteps) / full_block_est)
    inst = scaled_instance(args.config, args.seed, f) if f < 1.0 else make_instance(args.config, args.seed)
    o = O.Oracle(inst)
    o.preprocess(max_iter=50)
    prm = O.params(k_int=args.k_int, k_b=k_b_total, max_iters=args.k_int, tol_primal=-1.0, tol_dual=-1.0,
                   tol_binary=-1.0, stall_rel=-1.0)
    times, raw = [], []
    for st in range(nsteps):
        t0 = time.perf_counter()
        o.run(prm)
        dt = time.perf_counter() - t0
        if st >= args.warmup:
            times.append(dt / f)
            raw.append(dt)
    t = statistics.median(times)
    value = k_b_total / t
    full = inst_meta(make_instance(args.config, args.seed)) if f < 1.0 else inst_meta(inst)
    sample = (f"oracle (1 thread) Alg. 1 blocks on the config{args.config} recipe at size fraction f={f:.4g} "
              f"(n={inst['n']}, m={inst['m']}, nnz={int(inst['k_rowptr'][-1])}); per-step time scaled by 1/f")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "pdhg_iters_per_s": args.k_int / t,
            "extrapolation": {"size_fraction": f, "ms_per_step_measured": statistics.median(raw) * 1e3,
                              "note": "each step is one real oracle block on the size-f instance of the same recipe; "
                                      "ms_per_step = measured / f (cost linear in the instance size)"},
            "config": {"workload": f"config{args.config}", "n": full["n"], "m": full["m"], "nnz": full["nnz"],
                       "k_int": args.k_int, "k_b_per_rank": args.k_b, "seed": args.seed},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


# ------------------------------------------------------------------------------------------------
def run_f1_maxcut(args, gf, stream, local):
    """Next row f1: the dense-Q path on the paper's largest max-cut size (config 6,
    n = 20480, density 0.5).  Same step definition and clock as the headline line
    (one Alg. 1 block per step, one graph launch for all timed blocks, CUDA events); rooflines of
    its two kernels: the dense int8 GEMV (HBM: n^2 bytes of Q per launch) and the tcgen05 int8
    objective (tensor: 2 * 128^2 * k_b ops per upper-triangle tile; HBM: its Q tile bytes)."""
    import torch
    t_gen = time.perf_counter()
    inst = make_instance(6, args.seed)
    t_gen = time.perf_counter() - t_gen
    n = int(inst["n"])
    s = gf.Solver(local, stream=stream.cuda_stream)
    t0 = time.perf_counter()
    s.load(inst)
    sc = s.preprocess(precision=args.precision)
    torch.cuda.synchronize()
    t_load = time.perf_counter() - t0
    common = dict(k_int=args.k_int, k_b=args.k_b, tol_primal=-1.0, tol_dual=-1.0, tol_binary=-1.0,
                  stall_rel=-1.0, time_limit_s=1e9, trace_cap=16)
    s.run(max_iters=max(3, args.warmup) * args.k_int, **common)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    K = args.f1_steps
    e0.record(stream)
    info = s.run(max_iters=K * args.k_int, **common)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    z, _, inc = s.best_incumbent(want_x=False)
    prof = s.profile_blocks(min(K, 20), **common)
    act = s.profile_active()
    nb = min(K, 20)
    peak_hbm, peak_src, peaks = measured_peaks()
    fb = 8 if args.precision == 64 else 4
    # GEMV: k_int primal products + 1 trigger product per block (each = dense + final launch); with
    # fp32 iterates and k_int > 1 the next block's first primal reuses the trigger's product
    # (option qx_reuse, on by default), so k_int products are computed per block
    qx_ms, qx_launches = act.get("pdhg_qx", (0.0, 0))
    reuse = args.precision == 32 and args.k_int > 1
    gemv_per_block = args.k_int if reuse else args.k_int + 1
    gemv_ms = qx_ms / (nb * gemv_per_block)
    gemv_bytes = n * n + 2 * n * fb + 8 * n
    # objective tensor kernel: the upper block triangle of Q (T(T+1)/2 tiles of 128 x 128)
    T = (n + 127) // 128
    tiles = T * (T + 1) // 2
    tc_ms, _ = act.get("obj_tc", (0.0, 0))
    tc_ms /= nb
    tc_ops = 2.0 * tiles * 128 * 128 * args.k_b
    tc_bytes = tiles * 128 * 128 + (n * args.k_b)  # Q tiles + unpacked samples (first touch)
    i8_peak = peaks.get("bf16_tflops", 1628.4) * 2.0  # int8 dense = 2x bf16 (guide's nominal ratio)
    value = K * args.k_b / (ms * 1e-3)
    s.close()
    return {
        "workload": "config6", "desc": "max cut QP n=20480, density 0.5, w ~ U{-8..10} (dense int8 Q)",
        "n": n, "qnnz": int(inst["q_rowptr"][-1]), "value": value, "unit": UNIT, "steps": K,
        "ms_per_step": ms / K, "pdhg_iters_per_s": K * args.k_int / (ms * 1e-3),
        "z_best": z if inc["has_incumbent"] else None, "obj_scale": sc["obj_scale"],
        "gen_s": t_gen, "load_preprocess_s": t_load, "kernel_ms_per_step": prof,
        "roofline_gemv": {"bound": "hbm", "kernel": "k_qx_tma_fix+k_qx_final" if args.precision == 32 else "k_qx_tma+k_qx_final", "achieved": gemv_bytes / (gemv_ms * 1e-3) / 1e9,
                          "peak": peak_hbm, "unit": "GB/s", "frac": gemv_bytes / (gemv_ms * 1e-3) / 1e9 / peak_hbm,
                          "algorithmic_bytes_per_launch": gemv_bytes, "avg_launch_ms": gemv_ms, "peak_source": peak_src},
        "roofline_obj_tc": {"bound": "hbm" if tc_bytes / (peak_hbm * 1e9) > tc_ops / (i8_peak * 1e12) else "tensor",
                            "kernel": "k_unpack_samples+k_obj_dense_tc", "avg_launch_ms": tc_ms,
                            "achieved_tops": tc_ops / (tc_ms * 1e-3) / 1e12, "peak_tops_int8": i8_peak,
                            "tensor_frac": tc_ops / (tc_ms * 1e-3) / 1e12 / i8_peak,
                            "achieved_gbs": tc_bytes / (tc_ms * 1e-3) / 1e9, "hbm_frac": tc_bytes / (tc_ms * 1e-3) / 1e9 / peak_hbm,
                            "ops_per_launch": tc_ops, "bytes_per_launch": tc_bytes,
                            "peak_note": "int8 peak = MEASURED_PEAKS bf16 burst x 2 (nominal int8/bf16 ratio)"},
    }


def run_f1_dense_k(args, gf, stream, local):
    """Next row f1, dense-K half ("int8 MMA for MKP's K.X"): config 3 (MKP n = 1e5, m = 50,
    density 0.5).  Per Alg. 1 block (eager replay with per-launch CUDA events, 20 blocks from x0): the
    feasibility class with the integer rows on tensor cores (split-K tcgen05 kind::i8, exact int32)
    against the CUDA-core integer path (option dense_k = 0), and the tensor kernel's roofline: ops
    2 * ceil128(m) * k_b * ceil128(n) per launch; bytes = the int8 rows + the unpacked samples."""
    inst = make_instance(3, args.seed)
    n, m = int(inst["n"]), int(inst["m"])
    out = {"workload": "config3", "desc": "multi-dimensional knapsack n=1e5, m=50, density 0.5"}
    peak_hbm, _, peaks = measured_peaks()
    i8_peak = peaks.get("bf16_tflops", 1628.4) * 2.0
    for dk in (1, 0):
        s = gf.Solver(local, stream=stream.cuda_stream, options={"dense_k": dk})
        s.load(inst)
        s.preprocess(precision=args.precision)
        common = dict(k_int=args.k_int, k_b=args.k_b, tol_primal=-1.0, tol_dual=-1.0, tol_binary=-1.0, stall_rel=-1.0)
        prof = s.profile_blocks(20, **common)
        act = s.profile_active()
        out["tensor_core" if dk else "cuda_core"] = {"feas_ms_per_block": prof.get("feas"), "unpack_ms_per_block": prof.get("obj_tc"),
                                                     "block_ms": sum(prof.values())}
        s.close()
    tc_ms = out["tensor_core"]["feas_ms_per_block"]
    ld = (n + 127) // 128 * 128
    ops = 2.0 * 128 * args.k_b * ld
    byts = 128 * ld + args.k_b * ld
    out["roofline_feas_tc"] = {"kernel": "k_obj_dense_tc<FEAS>+k_feas_dense_final (feas class per round)",
                               "ops_per_launch": ops, "bytes_per_launch": byts, "ms": tc_ms,
                               "tensor_frac": ops / (tc_ms * 1e-3) / 1e12 / i8_peak,
                               "hbm_frac": byts / (tc_ms * 1e-3) / 1e9 / peak_hbm,
                               "note": "k_b = 128 leaves the MMA N-starved and the split-K K-ranges short (5 K-blocks per CTA): "
                                       "latency-bound; the win is against the per-(nonzero, lane) integer path"}
    out["speedup_feas"] = out["cuda_core"]["feas_ms_per_block"] / tc_ms if tc_ms else None
    return out


def run_f2_facility(args, gf, stream, local):
    """Next row f2: TUReformulate (PAPER §2.4.1) on the paper's facility-location
    workload at (nf, nc) = (512, 2048) (config 7), three forms, same Alg. 1 run
    (fixed iteration budget, halting disabled): "tu" = all-equality slack form with every row
    eliminated (general, unit-triangular B_JI: sparse exact elimination; reading R24 rev.),
    "tu_gub" = inequality form with the customer rows eliminated (B_JI = identity; round-1 reading),
    "no_tu" = inequality form as is.  Objective reached, time to incumbent (device %globaltimer,
    Preprocess excluded as in PAPER L193), candidates/s, and the host time of the reformulation
    itself (the paper's 'Avg. TU Time' column)."""
    from gen import instances as G
    out = {"workload": "config7", "desc": "facility location nf=512, nc=2048 (n = 1,049,088; m = 1,050,624)",
           "note": "fixed iteration budget, halting disabled; 'small' = (nf, nc) = (16, 64), fp64, 30000 iterations"}
    for key, nf, nc, iters, prec in (("", 512, 2048, args.f2_iters, args.precision), ("small_", 16, 64, 30000, 64)):
        _f2_forms(out, key, nf, nc, iters, prec, args, gf, stream, local, G)
    return out


def _f2_forms(out, key, nf, nc, iters, prec, args, gf, stream, local, G):
    import torch
    fl = G.facility_location(nf, nc, args.seed)
    out[key + "n"], out[key + "m"] = int(fl["n"]), int(fl["m"])
    for form in ("tu", "tu_gub", "no_tu"):
        inst = G.facility_location_slack(nf, nc, args.seed) if form == "tu" else fl
        s = gf.Solver(local, stream=stream.cuda_stream)
        s.load(inst)
        t_tu = None
        if form != "no_tu":
            t0 = time.perf_counter()
            s.tu_reformulate(inst["tu_rows"], inst["tu_cols"])
            t_tu = time.perf_counter() - t0
        s.preprocess(precision=prec)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        info = s.run(max_iters=iters, k_int=args.k_int, k_b=args.k_b, tol_primal=-1.0, tol_dual=-1.0,
                     tol_binary=-1.0, stall_rel=-1.0)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        z, x, meta = s.best_incumbent()
        feasible = None
        if meta["has_incumbent"]:
            # the lifted incumbent against the ORIGINAL inequality rows (host check, exact integers)
            x = x[: fl["n"]]
            K_rows = np.repeat(np.arange(fl["m"]), np.diff(fl["k_rowptr"]))
            ax = np.bincount(K_rows, weights=fl["k_val"] * x[fl["k_col"]], minlength=fl["m"])
            ok = np.where(fl["sense"] == 0, ax == fl["r"], np.where(fl["sense"] == 1, ax >= fl["r"], ax <= fl["r"]))
            feasible = bool(ok.all()) and float(fl["c"] @ x) == z
        out[key + form] = {
            "reduced_n": s.n, "reduced_m": s.m, "tu_seconds": t_tu, "iters": info["iters"],
            "halt_reason": info["halt_reason"], "z_best": z if meta["has_incumbent"] else None,
            "time_to_incumbent_s": meta["found_time_s"] if meta["has_incumbent"] else None,
            "loop_ms": ms, "candidates_per_s": info["candidates"] / (ms * 1e-3),
            "pdhg_iters_per_s": info["iters"] / (ms * 1e-3), "incumbent_feasible_for_original": feasible}
        s.close()


def run_f3_assign3d(args, gf, stream, local):
    """Next row f3: the customised RandSampleStep of Alg. 4 on 3D
    assignment n = 64 (config 8; 262,144 binaries, 192 equality rows) against the default Bernoulli
    sampler, same iteration budget (halting disabled): objective reached, time to incumbent,
    candidates/s and the sampler's share of the step (CUDA events of an eager replay)."""
    import torch
    inst = make_instance(8, args.seed)
    n3 = int(inst["a3_n"])
    out = {"workload": "config8", "desc": "3D assignment n=64 (n^3 = 262,144 binaries)", "a3_n": n3,
           "gamma": 4.0, "L": 2 * n3}
    # custom = Alg. 4 sampler; default = Bernoulli sampler; relax_repair = Bernoulli sampler on the
    # monotone relaxation + repair (next row f4)
    for name, sampler, relax in (("custom", 1, 0), ("default", 0, 0), ("relax_repair", 0, 1)):
        s = gf.Solver(local, stream=stream.cuda_stream)
        s.load(inst)
        s.preprocess(precision=args.precision)
        kw = dict(k_int=args.k_int, k_b=args.k_b, tol_primal=-1.0, tol_dual=-1.0, tol_binary=-1.0, stall_rel=-1.0,
                  sampler=sampler, a3_n=n3, relax=relax, repair=relax)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        info = s.run(max_iters=args.f3_iters, **kw)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        z, _, meta = s.best_incumbent(want_x=False)
        prof = s.profile_blocks(20, **kw)
        out[name] = {
            "iters": info["iters"], "z_best": z if meta["has_incumbent"] else None,
            "time_to_incumbent_s": meta["found_time_s"] if meta["has_incumbent"] else None,
            "found_iter": meta["found_iter"], "loop_ms": ms, "candidates_per_s": info["candidates"] / (ms * 1e-3),
            "pdhg_iters_per_s": info["iters"] / (ms * 1e-3), "sample_ms_per_block": prof.get("sample"),
            "block_ms_eager": sum(prof.values())}
        s.close()
    return out


def run_gpu(args):
    import torch
    rank, world, local = dist_env()
    if world != args.gpus:
        args.gpus = world
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2510_27117_b200 as gf

    inst = make_instance(args.config, args.seed)
    meta = inst_meta(inst)
    stream = torch.cuda.current_stream()
    def fresh_nccl_id():
        """a new ncclUniqueId made on rank 0 and broadcast (one per communicator: ids are not reused)"""
        import torch.distributed as dist
        buf = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            buf.copy_(torch.frombuffer(bytearray(gf.nccl_unique_id()), dtype=torch.uint8).cuda())
        dist.broadcast(buf, 0)
        return bytes(buf.cpu().numpy().tobytes())

    nccl_id = None
    if world > 1:
        # in-loop incumbent exchange (one 32-byte record per rank per sampling round, ncclAllGather
        # captured in the loop graph): id made on rank 0, broadcast through torch.distributed
        import torch.distributed as dist
        buf = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            buf.copy_(torch.frombuffer(bytearray(gf.nccl_unique_id()), dtype=torch.uint8).cuda())
        dist.broadcast(buf, 0)
        nccl_id = bytes(buf.cpu().numpy().tobytes())
    s = gf.Solver(local, stream=stream.cuda_stream, rank=rank, world=world, nccl_id=nccl_id)
    # device-resident inputs (value leg): torch tensors on cuda
    dev = {k: (torch.from_numpy(np.ascontiguousarray(v)).cuda() if isinstance(v, np.ndarray) else v)
           for k, v in inst.items()}
    s.load(dev)
    torch.cuda.synchronize()
    sc = s.preprocess(precision=args.precision)
    fb = 8 if args.precision == 64 else 4
    common = dict(k_int=args.k_int, k_b=args.k_b, tol_primal=-1.0, tol_dual=-1.0, tol_binary=-1.0,
                  stall_rel=-1.0, time_limit_s=1e9, trace_cap=16)
    if world > 1 and not args.no_row_shard:
        common["row_shard"] = 1  # row-sharded dual over the ranks (f4): y all-gathered each iteration
    # warm-up (also instantiates the CUDA graph)
    s.run(max_iters=args.warmup * args.k_int, **common)
    torch.cuda.synchronize()

    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(local)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    clk.start()
    time.sleep(0.3)
    clk.region_begin()
    e0.record(stream)
    info = s.run(max_iters=args.steps * args.k_int, **common)
    e1.record(stream)
    torch.cuda.synchronize()
    clk.region_end()
    clocks = clk.stop()
    ms = e0.elapsed_time(e1)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    t_s = ms * 1e-3
    cand = info["candidates"] * world if world > 1 else info["candidates"]
    value = args.steps * args.k_b * world / t_s
    iters_s = args.steps * args.k_int / t_s
    z, _, inc = s.best_incumbent(want_x=False)

    # phases of the trajectory (the per-block cost falls as the iterate sparsifies and the
    # push modes engage, so the headline depends on K): blocks 1..K from x0 is what --steps K times
    # (the headline); the steady window 181..200 is t(200 blocks) - t(180 blocks), same clock
    phases = None
    if rank == 0 and world == 1:
        def run_ms(blocks):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            s.run(max_iters=blocks * args.k_int, **common)
            b.record(stream)
            torch.cuda.synchronize()
            return a.elapsed_time(b)
        t200, t180 = run_ms(200), run_ms(180)
        phases = {"blocks_1_to_K": {"K": args.steps, "candidates_per_s": value, "ms_per_block": ms / args.steps},
                  "blocks_181_to_200": {"candidates_per_s": 20 * args.k_b / ((t200 - t180) * 1e-3),
                                        "ms_per_block": (t200 - t180) / 20,
                                        "how": "t(200 blocks from x0) - t(180 blocks from x0), CUDA events"},
                  "blocks_1_to_200": {"candidates_per_s": 200 * args.k_b / (t200 * 1e-3), "ms_per_block": t200 / 200}}

    # PDHG alone (sampling off): Alg. 2 steps through the step hook (same kernels, eager launches),
    # fixed rho = rho_min, from x0 (dense phase: iterations 1-100) and after 1000 steps (1001-1100)
    pdhg_only = None
    if rank == 0 and world == 1 and not args.no_extras:
        x0 = np.full(meta["n"], 0.5)
        s.set_state(x0, x0, np.zeros(meta["m"]))
        tau = 0.99 ** 0.5
        def steps_ms(k):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            s.step(k, 1e-3, tau, tau)
            b.record(stream)
            torch.cuda.synchronize()
            return a.elapsed_time(b)
        d = steps_ms(100)
        s.step(900, 1e-3, tau, tau)
        l = steps_ms(100)
        pdhg_only = {"iters_1_100_per_s": 100 / (d * 1e-3), "iters_1001_1100_per_s": 100 / (l * 1e-3),
                     "how": "gfors_step hook (eager launches, rho = 1e-3 fixed, no sampling), CUDA events"}
        # graph replay: one block of k_int = 1000 iterations (the loop graph, rho schedule,
        # trigger pass once, one sampling round of 64 candidates), from x0, median of 3 runs
        gms = []
        for _ in range(4):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            s.run(max_iters=1000, k_int=1000, k_b=64, tol_primal=-1.0, tol_dual=-1.0, tol_binary=-1.0, stall_rel=-1.0)
            b.record(stream)
            torch.cuda.synchronize()
            gms.append(a.elapsed_time(b))
        pdhg_only["graph_iters_1_1000_per_s"] = 1000 / (statistics.median(gms[1:]) * 1e-3)
        pdhg_only["graph_how"] = "one gfors_run of 1000 iterations with k_int = 1000 (one trigger pass and one 64-candidate round), from x0, median of 3 after one warm-up, CUDA events"

    # sampling-only candidates/s: RandSampleStep + EvalBest + argmin at fixed p, no
    # PDHG, per p-distribution (x_k of the blocks 1-K trajectory, U(0,1), 90/10 exact/uniform mix)
    # and per k_b; device time over 10 rounds (gfors_sample_eval_timed)
    sampling_only = None
    if rank == 0 and world == 1 and not args.no_extras:
        from gen import instances as G
        pv = G.p_vectors(meta["n"], 5)
        x_now = None
        try:
            s.run(max_iters=args.steps * args.k_int, **common)
            x_now = s.get_state()[0]
        except Exception:
            x_now = None
        if x_now is not None:
            pv["traj"] = np.clip(x_now, 0.0, 1.0)
        sampling_only = {"how": "10 rounds of sample + evaluate + argmin at fixed p after one warm-up round, CUDA events (gfors_sample_eval_timed)",
                         "traj": f"x_k after {args.steps} blocks from x0"}
        for name in ("traj", "unif", "mix"):
            if name not in pv:
                continue
            row = {}
            for kb in (64, 128, 512, 1024, 4096):
                s.sample_eval_timed(pv[name], 20251030, kb // 64, 1)  # warm-up: first launches load the kernels
                ms_r = s.sample_eval_timed(pv[name], 20251030, kb // 64, 10)
                row[str(kb)] = 10 * kb / (ms_r * 1e-3)
            sampling_only[name] = row

    # time-to-incumbent on the headline workload: the default (Alg. 3) sampler finds no feasible set
    # cover within the run; with the cover completion of the samples (R27) every lane is feasible
    cover = None
    if rank == 0 and world == 1 and args.config == 5:
        e2 = torch.cuda.Event(enable_timing=True)
        e3 = torch.cuda.Event(enable_timing=True)
        e2.record(stream)
        ic = s.run(max_iters=1000, **dict(common, complete=1, trace_cap=1000))
        e3.record(stream)
        torch.cuda.synchronize()
        zc, _, mc = s.best_incumbent(want_x=False)
        cover = {"note": "same instance, RandSampleStep + cover completion (DESIGN R27), 100 blocks, halting off",
                 "z_best": zc if mc["has_incumbent"] else None,
                 "time_to_best_incumbent_s": mc["found_time_s"] if mc["has_incumbent"] else None,
                 "found_iter": mc["found_iter"], "candidates_per_s": ic["candidates"] / (e2.elapsed_time(e3) * 1e-3)}
        tr = s.trace()
        fin = tr[np.isfinite(tr[:, 6])] if len(tr) else tr
        cover["first_incumbent_iter"] = int(fin[0, 0]) if len(fin) else None
        cover["first_incumbent_z"] = float(fin[0, 6]) if len(fin) else None

    # per-kernel device times (CUDA events around every launch of an eager replay of the same blocks)
    prof = s.profile_blocks(args.profile_blocks or args.steps, **common)
    step_ms = sum(prof.values())
    byt = algorithmic_bytes(meta, fb)
    act = s.profile_active()  # class -> (active ms over all profiled blocks, launches that did work)
    # roofline kernel: the gather-mode PDHG kernel with the most active time; its average over the
    # launches that ran the dense product (mode-switched launches that exited early are excluded)
    dom = max(("pdhg_primal", "pdhg_dual"), key=lambda k: act.get(k, (0.0, 0))[0])
    if act.get(dom, (0.0, 0))[1] > 0:
        per_launch_ms = act[dom][0] / act[dom][1]
    else:
        per_launch_ms = prof[dom] / args.k_int
    peak, peak_src, peaks = measured_peaks()
    achieved = byt[dom] / (per_launch_ms * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        tj = json.load(open(tpath))
        traffic = tj.get(f"config{args.config}_fp{args.precision}", {}).get(dom)

    # EvalBest + RandSampleStep per round (k_b candidates): algorithmic bytes with the batch X materialised
    # (DESIGN §6): sampler reads p (n fb) and writes X (n W 8); feasibility streams the indices of the
    # count rows (4 nnz + 4 m) and reads X once (gathers assumed cache hits); the objective reads X and
    # the coefficient planes (n NB/8, NB = 7 for c in [1, 100]).  The binding limits are the 16-byte
    # random gathers of the feasibility kernel (one per nonzero) and the sampler's Philox ALU work.
    W = args.k_b // 64
    ev_ms = {k: prof.get(k, 0.0) for k in ("sample", "feas", "obj")}
    ev_total = sum(ev_ms.values())
    ev_bytes = meta["n"] * fb + meta["n"] * W * 8 + (4 * meta["nnz"] + 4 * meta["m"] + meta["n"] * W * 8) \
        + (meta["n"] * W * 8 + meta["n"] * 7 // 8)
    evaluator = None
    if ev_total > 0:
        feas_g = meta["nnz"] * max(1, W // 2) / (ev_ms["feas"] * 1e-3) / 1e9 if ev_ms["feas"] else None
        evaluator = {"kernels": "k_sample_thr+k_sample, k_feas_skip+k_feas_rb, k_obj_bits+k_obj_final",
                     "ms_per_round": ev_total, "ms_by_class": ev_ms, "algorithmic_bytes_per_round": ev_bytes,
                     "achieved": ev_bytes / (ev_total * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": ev_bytes / (ev_total * 1e-3) / 1e9 / peak,
                     "feas_gather": {"gathers_per_round": meta["nnz"] * max(1, W // 2), "bytes_per_gather": 16 if W % 2 == 0 else 8,
                                     "achieved_G_per_s": feas_g, "ceiling_G_per_s": GATHER16_CEILING_G,
                                     "frac": feas_g / GATHER16_CEILING_G if feas_g else None},
                     "window": f"blocks 1..{args.profile_blocks or args.steps} from x0 (eager replay with per-launch events)"}

    # the streaming column pass of the push-mode primal (k_primal_push), the largest non-gather kernel
    # of the steady state: bytes if every column is streamed (stationary columns are skipped, so
    # this bounds its algorithmic bytes from above) and the DRAM bytes of its ncu capture
    col = None
    if act.get("pdhg_primal_col", (0.0, 0))[1] > 0:
        col_ms = act["pdhg_primal_col"][0] / act["pdhg_primal_col"][1]
        sbytes = meta["n"] * (5 * fb + 8 + 1)
        dram = None
        if os.path.exists(tpath):
            dram = json.load(open(tpath)).get(f"config{args.config}_fp{args.precision}", {}).get("pdhg_primal_col")
        col = {"kernel": "k_primal_push", "avg_active_launch_ms": col_ms, "stream_bytes_per_launch": sbytes,
               "stream_GBs": sbytes / (col_ms * 1e-3) / 1e9, "stream_frac": sbytes / (col_ms * 1e-3) / 1e9 / peak,
               "dram_bytes_per_launch_ncu": dram,
               "dram_GBs": (dram / (col_ms * 1e-3) / 1e9) if dram else None,
               "dram_frac": (dram / (col_ms * 1e-3) / 1e9 / peak) if dram else None}

    # the device-resident solver is done: release its memory before the e2e leg allocates its own
    s.close()
    torch.cuda.synchronize()

    # e2e through the public API from pinned host buffers
    e2e = None
    if not args.no_e2e and rank == 0 or (world > 1 and not args.no_e2e):
        host = {}
        h2d = 0
        for k, v in inst.items():
            if isinstance(v, np.ndarray):
                tv = torch.from_numpy(np.ascontiguousarray(v)).pin_memory()
                host[k] = tv.numpy()
                h2d += v.nbytes
            else:
                host[k] = v
        reps = []
        for _rep in range(3):  # three independent call chains; the median one is reported (host-side load varies)
            s2 = gf.Solver(local, stream=stream.cuda_stream, rank=rank, world=world,
                           nccl_id=fresh_nccl_id() if world > 1 else None)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            s2.load(host)
            ta = time.perf_counter()
            s2.preprocess(precision=args.precision)
            tb = time.perf_counter()
            s2.run(max_iters=args.steps * args.k_int, **common)
            tc = time.perf_counter()
            z2, x2, _ = s2.best_incumbent()
            torch.cuda.synchronize()
            te = time.perf_counter() - t0
            s2.close()
            reps.append((te, {"load_s": ta - t0, "preprocess_s": tb - ta, "run_s": tc - tb, "best_incumbent_s": t0 + te - tc}))
        te, e2e_split = sorted(reps, key=lambda r: r[0])[1]
        e2e = {"value": args.steps * args.k_b * world / te, "unit": UNIT, "h2d_bytes_per_step": h2d / args.steps,
               "d2h_bytes_per_step": (meta["n"] + 64) / args.steps,
               "note": "one gfors_load+preprocess+run(K blocks)+best_incumbent call chain from pinned host memory, "
                       "a fresh solver each time; instance bytes amortised over the K steps; median of 3 chains",
               "seconds": te, "split_s": e2e_split, "chains_s": [r[0] for r in reps]}

    # time-to-incumbent (BASELINE metric, third part): full solves of the small configs with the
    # default halting rule, %globaltimer stamp of the last improvement (Preprocess excluded)
    tti = None
    if rank == 0 and world == 1 and not args.no_tti:
        tti = {}
        for cfg in (1, 2, 3, 4):
            inst_c = make_instance(cfg, args.seed)
            sc_ = gf.Solver(local, stream=stream.cuda_stream)
            sc_.load(inst_c)
            sc_.preprocess(precision=args.precision)
            info_c = sc_.run(max_iters=20000, k_b=args.k_b)
            zc, _, mc = sc_.best_incumbent(want_x=False)
            tti[f"config{cfg}"] = {"z_best": zc if mc["has_incumbent"] else None,
                                   "time_to_incumbent_s": mc["found_time_s"] if mc["has_incumbent"] else None,
                                   "found_iter": mc["found_iter"], "iters": info_c["iters"],
                                   "halt_reason": info_c["halt_reason"], "loop_s": info_c["elapsed_s"]}
            sc_.close()
        # config 5 (the workload) under the same SPEC halting rule: its incumbent comes from Alg. 1's final
        # round(x_k) once the penalised PDHG has converged (found_round = -1)
        sc_ = gf.Solver(local, stream=stream.cuda_stream)
        sc_.load(inst)
        sc_.preprocess(precision=args.precision)
        info_c = sc_.run(max_iters=200000, k_b=args.k_b)
        zc, _, mc = sc_.best_incumbent(want_x=False)
        tti["config5"] = {"z_best": zc if mc["has_incumbent"] else None,
                          "time_to_incumbent_s": mc["found_time_s"] if mc["has_incumbent"] else None,
                          "found_iter": mc["found_iter"], "found_round": mc["found_round"], "iters": info_c["iters"],
                          "halt_reason": info_c["halt_reason"], "loop_s": info_c["elapsed_s"]}
        sc_.close()

    # configs 2-4: their per-iteration working sets fit in the 126 MB L2, so the PDHG
    # step is judged against the measured L2 read bandwidth as well as HBM; iterations 1-100 from x0,
    # sampling off (step hook), algorithmic bytes as for config 5
    small_l2 = None
    if rank == 0 and world == 1 and not args.no_tti:
        small_l2 = {"l2_read_GBs": L2_READ_GBS, "hbm_GBs": peak}
        for cfg in (2, 3, 4):
            inst_c = make_instance(cfg, args.seed)
            meta_c = inst_meta(inst_c)
            sc_ = gf.Solver(local, stream=stream.cuda_stream)
            sc_.load(inst_c)
            sc_.preprocess(precision=args.precision)
            x0 = np.full(meta_c["n"], 0.5)
            sc_.set_state(x0, x0, np.zeros(meta_c["m"]))
            sc_.step(10, 1e-3, 0.99 ** 0.5, 0.99 ** 0.5)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            sc_.step(100, 1e-3, 0.99 ** 0.5, 0.99 ** 0.5)
            b.record(stream)
            torch.cuda.synchronize()
            it_ms = a.elapsed_time(b) / 100
            by = algorithmic_bytes(meta_c, fb)
            qb = 12 * meta_c["qnnz"] + meta_c["n"] * fb if meta_c["qnnz"] else 0
            tot = by["pdhg_dual"] + by["pdhg_primal"] + qb
            small_l2[f"config{cfg}"] = {"ms_per_iteration": it_ms, "iters_per_s": 1e3 / it_ms,
                                        "algorithmic_bytes_per_iteration": tot,
                                        "achieved_GBs": tot / (it_ms * 1e-3) / 1e9,
                                        "l2_frac": tot / (it_ms * 1e-3) / 1e9 / L2_READ_GBS,
                                        "hbm_frac": tot / (it_ms * 1e-3) / 1e9 / peak}
            sc_.close()

    f1 = None
    if rank == 0 and world == 1 and not args.no_f1 and args.config != 6:
        f1 = run_f1_maxcut(args, gf, stream, local)
    f1k = None
    if rank == 0 and world == 1 and not args.no_f1:
        f1k = run_f1_dense_k(args, gf, stream, local)
    f2 = None
    if rank == 0 and world == 1 and not args.no_f2:
        f2 = run_f2_facility(args, gf, stream, local)
    f3 = None
    if rank == 0 and world == 1 and not args.no_f3:
        f3 = run_f3_assign3d(args, gf, stream, local)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ob = oracle_baseline(inst, args.k_int)
        cpu = {"value": ob["value"], "unit": UNIT, "cores": 1, "kind": "oracle", "sample": ob["sample"],
               "ms_per_block": ob["t_block"] * 1e3, "all_host_cores": ob["all_cores"], "cpu_model": ob["cpu_model"],
               "host_cpu_count": os.cpu_count(), "small_configs": oracle_small_configs(args.seed)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32" if args.precision == 32 else "f64", "data": "synthetic",
            "pdhg_iters_per_s": iters_s,
            # time-to-incumbent / z of config 5 solved under the SPEC halting rule (the timed run above
            # disables halting and stops after K blocks, before any incumbent)
            "time_to_incumbent_s": (tti or {}).get("config5", {}).get("time_to_incumbent_s"),
            "z_best": (tti or {}).get("config5", {}).get("z_best"),
            "time_to_incumbent_how": "config 5 solved with the SPEC halting defaults (time_to_incumbent_small_configs.config5); "
                                     "the timed K-block run itself ends before the first incumbent",
            "config": {"workload": f"config{args.config}", "desc": "set cover n=5e6 cols, m=1e6 rows, row degree U{2..98}"
                       if args.config == 5 else f"BASELINE config {args.config}",
                       "n": meta["n"], "m": meta["m"], "nnz": meta["nnz"], "k_int": args.k_int, "k_r": 1,
                       "k_b_per_rank": args.k_b, "precision": f"fp{args.precision} iterates, fp64 accumulation, exact int64 evaluation",
                       "parallelism": (f"sample-sharded x{world} (NCCL record all-gather per round), "
                                       + ("dual row-sharded (y all-gather per iteration), rest of PDHG replicated"
                                          if world > 1 and not args.no_row_shard else "PDHG replicated")), "l2": "inputs larger than L2 (K stream ~0.5 GB/iter)",
                       "seed": args.seed, "obj_scale": sc["obj_scale"], "k_scale": sc["k_scale"]},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": byt[dom], "avg_launch_ms": per_launch_ms,
                         # the binding limit of a random sparse product on B200: one L1TEX wavefront per
                         # gathered element; ceiling measured by scratch/gather_bench.cu (profiles/)
                         "gather": {"gathers_per_launch": meta["nnz"], "achieved_G_per_s": meta["nnz"] / (per_launch_ms * 1e-3) / 1e9,
                                    "ceiling_G_per_s": GATHER_CEILING_G, "frac": meta["nnz"] / (per_launch_ms * 1e-3) / 1e9 / GATHER_CEILING_G}},
            "roofline_push_primal_column_pass": col,
            "roofline_evaluator": evaluator,
            "sampling_only_candidates_per_s": sampling_only,
            "pdhg_l2_rooflines_configs_2_4": small_l2,
            "phases": phases,
            "pdhg_only": pdhg_only,
            "kernel_ms_per_step": prof, "kernel_share": {k: v / step_ms for k, v in prof.items()} if step_ms else {},
            "kernel_active": {k: {"active_launches": v[1], "avg_active_ms": (v[0] / v[1]) if v[1] else None}
                              for k, v in act.items()},
            "clocks": clocks,
            "gpu_launches": int(info["launches"]),
            "e2e": e2e,
            "cpu_baseline": cpu,
            "time_to_incumbent_small_configs": tti,
            "config5_with_cover_completion": cover,
            "next_rows": {"f1_dense_q_maxcut": f1, "f1_dense_k_mkp": f1k, "f2_tu_facility": f2,
                          "f3_assign3d_custom_sampler": f3},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
