#!/usr/bin/env python
"""Benchmark: DovetailSort of BASELINE.json's headline configuration on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2|c1|c3-zipf1.0|c4-exp1e-5|...] [--n N]

Default workload (BASELINE.json configs[1], "C2"): 10^9 records of uint32
key + uint32 value, keys i.i.d. uniform on [0, 10^9) from a seeded torch
generator, values = original index.  A step = one full stable sort of that
batch, device-resident when the timed region starts (the per-step restore
of the unsorted input is outside the CUDA-event bracket).  Inputs (8 GB)
exceed the 126 MB L2, so no flush is needed between steps.

--impl reference times the reference algorithm's CPU implementation on the
host cores (the C++ oracle restatement, oracle/; the reference itself is
Python and cannot travel to the GPU box) on a bounded sample of the same
workload.  Prints one JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gkeys/s sorted (32/64-bit key-value) at 1/2/4/8 B200; % of HBM roofline"
UNIT = "Gkeys/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------
CONFIGS = {
    "c1": dict(desc="C1 keys-only u32 uniform [0,2^32), n=1e6", n=10**6, kb=4, vb=0, dist="u32full"),
    "c2": dict(desc="C2 u32 key + u32 value, keys uniform [0,1e9), values = index, n=1e9",
               n=10**9, kb=4, vb=4, dist="uniform1e9"),
    "c3-zipf0.6": dict(desc="C3 Zipf s=0.6 ranks over 1..1e9 mapped by a seeded permutation",
                       n=10**9, kb=4, vb=4, dist="zipf", s=0.6, D_ref=2.9997e9),
    "c3-zipf1.0": dict(desc="C3 Zipf s=1.0", n=10**9, kb=4, vb=4, dist="zipf", s=1.0, D_ref=2.3637e9),
    "c3-zipf1.2": dict(desc="C3 Zipf s=1.2", n=10**9, kb=4, vb=4, dist="zipf", s=1.2, D_ref=1.4729e9),
    "c3-zipf1.5": dict(desc="C3 Zipf s=1.5", n=10**9, kb=4, vb=4, dist="zipf", s=1.5, D_ref=1.1554e9),
    "c4-exp1e-5": dict(desc="C4 u64/u64 keys floor(Exp(rate 1e-5))", n=10**9, kb=8, vb=8,
                       dist="exp", rate=1e-5, D_ref=3.5897e9),
    "c4-exp1e-7": dict(desc="C4 u64/u64 keys floor(Exp(rate 1e-7))", n=10**9, kb=8, vb=8,
                       dist="exp", rate=1e-7, D_ref=2.9198e9),
    "c4-bexp": dict(desc="C4 u64/u64 keys w >> Geometric(0.5)", n=10**9, kb=8, vb=8, dist="bexp", D_ref=2.1875e9),
    # graph transpose: n is the TOTAL edge count, split over the ranks
    # (strong scaling); key = dst, value = src, both uint32
    "c5": dict(desc="C5 R-MAT 2^28 vertices, 2^32 edges (a,b,c,d)=(.57,.19,.19,.05), (dst, src) sorted "
                    "stably by dst, CSR offsets after", n=2**32, kb=4, vb=4, dist="rmat", scale=28,
               strong=True),
}


def gen_device(cfg, n, seed, device, gbase=0):
    """Seeded synthetic keys on the GPU (see gen.py for the distributions)."""
    from paper_2401_00710_b200 import gen

    return gen.generate_device(cfg, n, seed, device, gbase)


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    """SM clocks and throttle reasons sampled DURING the timed region: NVML
    every 1 ms from a thread (a region of a few ms still gets samples), else
    nvidia-smi every 20 ms."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu_index: int):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        ids = [x.strip() for x in vis.split(",") if x.strip()]
        self.idx = int(ids[gpu_index]) if gpu_index < len(ids) and ids[gpu_index].isdigit() else gpu_index
        self.proc = None
        self.nvml = None
        self.lines = []
        self.samples = []  # (sm_mhz, max_mhz, reasons bitmask)
        self.stop_ev = threading.Event()

    def start(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.idx)
            self.nvml = (pynvml, h)
            self.bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                         "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                         "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                         "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _poll(self):
        nv, h = self.nvml
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self.stop_ev.is_set():
            try:
                self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), mx,
                                     nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
            except Exception:
                pass
            time.sleep(0.001)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def wait_first(self, timeout_s: float = 5.0):
        """Block until the sampler has produced its first sample (nvidia-smi's
        start-up can outlast a short timed region); keep only later samples."""
        t0 = time.time()
        while (self.proc is not None and not self.lines) or (self.nvml is not None and not self.samples):
            if time.time() - t0 > timeout_s:
                break
            time.sleep(0.001)
        self.lines.clear()
        self.samples.clear()

    def stop(self):
        if self.nvml is not None:
            self.stop_ev.set()
            self.t.join(timeout=2)
            sm = [x[0] for x in self.samples]
            reasons = sorted(nm for nm, bit in self.bits.items() if any(x[2] & bit for x in self.samples))
            return {"sm_mhz": float(np.median(sm)) if sm else None,
                    "sm_max_mhz": float(self.samples[0][1]) if self.samples else None,
                    "reasons": reasons, "samples": len(sm), "source": "nvml, 1 ms"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampler unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(self.NAMES, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi, 20 ms"}


# ---------------------------------------------------------------------------
# reference arm / CPU baseline: the oracle restatement on host cores
# ---------------------------------------------------------------------------
def cpu_sample_sort(cfgd, n, seed, threads=0):
    from oracle import oracle as ora

    keys, vals = gen_host(cfgd, n, seed)
    t0 = time.perf_counter()
    ora.sort_inplace(keys, vals, "dt", threads=threads)
    dt = time.perf_counter() - t0
    return dt, keys, vals


def gen_host(cfgd, n, seed):
    rng = np.random.default_rng(seed)
    d = cfgd["dist"]
    if d == "uniform1e9":
        k = rng.integers(0, 10**9, size=n, dtype=np.uint32)
    elif d == "u32full":
        k = rng.integers(0, 2**32, size=n, dtype=np.uint32)
    elif d == "exp":
        k = np.floor(rng.exponential(1.0 / cfgd["rate"], size=n)).astype(np.uint64)
    elif d == "bexp":
        w = rng.integers(0, 2**64 - 1, size=n, dtype=np.uint64, endpoint=True)
        g = np.minimum(rng.geometric(0.5, size=n) - 1, 63).astype(np.uint64)
        k = w >> g
    elif d == "zipf":
        from paper_2401_00710_b200 import gen

        k = gen.zipf_keys_host(cfgd["s"], n, 10**9, seed)
    elif d == "rmat":
        import torch

        from paper_2401_00710_b200 import gen

        if torch.cuda.is_available():  # same edges as the numpy twin, generated fast
            dk, dv = gen.rmat_edges(n, cfgd.get("scale", 28), seed)
            return dk.cpu().numpy().view(np.uint32), dv.cpu().numpy().view(np.uint32)
        return gen.rmat_edges_host(n, cfgd.get("scale", 28), seed)
    else:
        raise ValueError(d)
    vdt = {0: None, 4: np.uint32, 8: np.uint64}[cfgd["vb"]]
    v = None if vdt is None else np.arange(n, dtype=vdt)
    return k, v


def cpu_bounded_sample(cfgd, seed, budget_s=12.0, n0=10**7, nmax=None):
    """Sort growing samples until one run takes >= budget/2 seconds."""
    nmax = nmax or cfgd["n"]
    n = min(n0, nmax)
    dt = 0.0
    while True:
        dt, _, _ = cpu_sample_sort(cfgd, n, seed)
        if dt >= budget_s / 2 or n >= nmax:
            break
        n = min(nmax, n * 4 if dt < budget_s / 8 else n * 2)
    return n, dt


def run_reference(args, cfgd, rank, world):
    if rank != 0:
        return
    from oracle import oracle as ora

    cores = ora.max_threads()
    n, _ = cpu_bounded_sample(cfgd, seed=1, budget_s=8.0)
    times = []
    for _ in range(args.warmup):
        cpu_sample_sort(cfgd, n, 1)
    for _ in range(args.steps):
        dt, _, _ = cpu_sample_sort(cfgd, n, 1)
        times.append(dt)
    ms = 1e3 * float(np.mean(times))
    value = n / (ms / 1e3) / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u32" if cfgd["kb"] == 4 else "u64", "data": "synthetic",
        "config": {"workload": args.config, "desc": cfgd["desc"], "sample_records": n},
        "cpu_baseline": {"value": round(value, 6), "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{n} records of the {args.config} workload, oracle dt_sort "
                                   f"(C++ restatement of the reference, OpenMP {cores} threads)"},
        "e2e": {"value": round(value, 6), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args, cfgd, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2401_00710_b200 import RecordArray, SortConfig, dt_sort
    from paper_2401_00710_b200.dtsort import sort_device

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    n = args.n or cfgd["n"]
    strong = bool(cfgd.get("strong"))
    if strong:  # n = total over the ranks; one global input (seed 0, global edge index)
        n //= world
    kb, vb = cfgd["kb"], cfgd["vb"]
    cfg = SortConfig(seed=0)
    src_k, src_v = gen_device(cfgd, n, 0 if strong else 1000 + rank, dev, gbase=rank * n)
    k = torch.empty_like(src_k)
    v = None if src_v is None else torch.empty_like(src_v)
    from paper_2401_00710_b200 import _lib
    from paper_2401_00710_b200.dtsort import split_n

    # (inputs of >= 2^32 records are split inside sort_device, which sizes its
    # own per-part workspaces)
    ws = None
    if n < split_n():
        ws = torch.empty(int(_lib.lib().dts_workspace_bytes(n, kb, vb)), dtype=torch.uint8, device=dev)
    multi = world > 1 or args.force_dist
    if multi:
        from paper_2401_00710_b200.distributed import CudaOps, dist_sort

        ops = CudaOps(cfg)

    def restore():
        k.copy_(src_k)
        if v is not None:
            v.copy_(src_v)

    def one_sort(profile=False, ordered=False):
        if multi:
            rk, rv, st = dist_sort(k, v, ops=ops)
            return None, st
        return sort_device(k, v, cfg, 0, profile=profile, workspace=ws, report=True, stream_ordered=ordered), None

    for _ in range(args.warmup):
        restore()
        one_sort()
    torch.cuda.synchronize()
    # correctness certificate on the last warm-up output (paper_2401_00710_b200/
    # certify.py): values = index -> the O(n) stable-sort certificate; C5
    # (values = src) and keys-only C1 -> sorted keys + the permutation-invariant
    # pair checksum of the input
    cert = None
    if not multi:
        from paper_2401_00710_b200 import certify

        if v is not None and cfgd["dist"] != "rmat":
            err = certify.stable_sort_certificate(src_k, k, v)
            cert = "stable-sort certificate (sorted, permutation, stable, key[i] == in[val[i]])"
        else:
            err = None if certify.keys_sorted(k) else "keys not sorted"
            if err is None and certify.pair_checksum(k, v) != certify.pair_checksum(src_k, src_v):
                err = "output records are not a permutation of the input records"
            cert = "sorted keys + permutation-invariant (key, value) checksum"
        if err is not None:
            raise SystemExit(f"certificate failed on the last warm-up output: {err}")
    clocks = Clocks(local_rank)
    if multi:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    clocks.wait_first()
    total_ms = 0.0
    reps = []
    dstats = []
    stream = torch.cuda.current_stream(dev)
    if multi:
        ops.launches = 0
    for _ in range(args.steps):
        restore()
        torch.cuda.synchronize()
        if multi:
            dist.barrier()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        rep, st = one_sort(ordered=True)  # (stream-ordered: no host return path in the step)
        b.record(stream)
        b.synchronize()
        total_ms += a.elapsed_time(b)
        reps.append(rep)
        dstats.append(st)
    torch.cuda.synchronize()
    if multi:
        dist.barrier()
    clk = clocks.stop()
    # per-kernel CUDA-event times (roofline, step shares): separate profiled
    # steps after the timed region (the profiled run drains the stream at its
    # end, which is not part of the timed step)
    if not multi:
        timed_launches = int(sum(r.gpu_launches for r in reps))
        reps, prof_ms = [], 0.0
        for _ in range(min(args.steps, 3)):
            restore()
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            reps.append(one_sort(profile=True)[0])
            b.record(stream)
            b.synchronize()
            prof_ms += a.elapsed_time(b)
    ms_local = total_ms / args.steps
    if multi:
        t = torch.tensor([ms_local], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    else:
        ms = ms_local
    n_total = n * world
    value = n_total / (ms / 1e3) / 1e9

    # roofline of the dominant kernel (k_scatter), CUDA events inside the
    # library on the launching stream, summed over the profiled steps
    peak, peak_kind = peaks()
    roof = None
    launches = int(ops.launches) if multi else None
    if multi:
        # SURVEY.md §8(d), G GPUs: per rank B_HBM = beta * (n_in (partition
        # pass) + D_local), B_NVL = bytes sent to other ranks; T_roof = max over
        # ranks of B_HBM / HBM peak + B_NVL / 900 GB/s (NVLink 5 per direction)
        beta = kb + 2 * (kb + vb)
        sts = [s for s in dstats if s is not None]
        b_hbm = beta * (sum(s.n_local_in for s in sts) + sum(s.local_distributed for s in sts)) / max(len(sts), 1)
        b_nvl = sum(s.bytes_sent_remote for s in sts) / max(len(sts), 1)
        x_ms = sum(s.exchange_ms for s in sts) / max(len(sts), 1)
        t = torch.tensor([b_hbm / (peak * 1e9) + b_nvl / 900e9, b_hbm, b_nvl, x_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_roof, hbm_max, nvl_max, xmax = [float(x) for x in t.tolist()]
        roof = {"bound": "hbm+nvlink", "achieved": round(n_total / (ms / 1e3) / 1e9, 4), "unit": "Gkeys/s",
                "frac": round(t_roof * 1e3 / ms, 4), "peak_hbm_GBps": peak, "peak_nvlink_GBps": 900.0,
                "peak_kind": peak_kind, "traffic": None,
                "B_hbm_GB_max_rank": round(hbm_max / 1e9, 3), "B_nvlink_GB_max_rank": round(nvl_max / 1e9, 3),
                "T_roof_ms": round(t_roof * 1e3, 3),
                "exchange_ms_max_rank": round(xmax, 3),
                "exchange_GBps": round(nvl_max / (xmax / 1e3) / 1e9, 1) if xmax > 0 else None}
    if not multi and reps and reps[0] is not None:
        sc_ms = sum(r.kernel_ms["scatter"] for r in reps)
        sc_launch = sum(r.kernel_launches["scatter"] for r in reps)
        sc_rec = sum(r.kernel_records["scatter"] for r in reps)
        bytes_alg = sc_rec * 2 * (kb + vb)  # read + write of every record
        per_launch_ms = sc_ms / max(sc_launch, 1)
        per_launch_bytes = bytes_alg / max(sc_launch, 1)
        achieved = per_launch_bytes / (per_launch_ms / 1e3) / 1e9
        launches = timed_launches
        shares = {c: round(sum(r.kernel_ms[c] for r in reps) / prof_ms, 4) for c in reps[0].kernel_ms}
        # ncu dram bytes of the scatter per record (profiles/traffic.json, one
        # --set full capture) x records per launch of this run
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
                bpr = json.load(f).get("dram_bytes_per_record")
            if bpr:
                traffic = int(bpr * sc_rec / max(sc_launch, 1))
        except Exception:
            pass
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "kernel": "k_scatter_wc (write-combining scatter)", "peak_kind": peak_kind,
                "algorithmic_bytes_per_launch": int(per_launch_bytes),
                "ms_per_launch": round(per_launch_ms, 4),
                "step_share": shares}
        # D of the reference's own distribution structure on THIS input:
        # profiles/D_exact.json (tools/d_exact.py: the oracle's
        # records_distributed on bench.py's exact rank-0 input); else the
        # SURVEY.md §8d table value scaled to --n
        D_ref, D_src = None, None
        try:
            with open(os.path.join(ROOT, "profiles", "D_exact.json")) as f:
                dx = json.load(f).get(args.config)
            if dx and int(dx["n"]) == n:
                D_ref, D_src = int(dx["D"]), "exact (oracle on this input, profiles/D_exact.json)"
        except Exception:
            pass
        if D_ref is None:
            D_ref = 3 * n if args.config == "c2" else (
                int(cfgd["D_ref"] * n / CONFIGS[args.config]["n"]) if "D_ref" in cfgd else None)
            D_src = "SURVEY.md §8d table" if D_ref is not None else None
        D_ours = reps[0].records_distributed
        beta = kb + 2 * (kb + vb)
        pipe = {"beta_bytes": beta, "D_ours": D_ours, "D_reference": D_ref, "D_reference_source": D_src,
                "B_alg_GB": round(beta * (D_ref or D_ours) / 1e9, 3),
                "achieved_GBps": round(beta * (D_ref or D_ours) / (ms / 1e3) / 1e9, 1),
                "frac_of_peak": round(beta * (D_ref or D_ours) / (ms / 1e3) / 1e9 / peak, 4)}
    else:
        pipe = None

    # end to end through the public API with pinned host buffers
    e2e = None
    if not multi and not args.no_e2e:
        hk = torch.empty(n, dtype=src_k.dtype, pin_memory=True)
        hv = None if src_v is None else torch.empty(n, dtype=src_v.dtype, pin_memory=True)
        ku = hk.view(torch.uint32 if kb == 4 else torch.uint64)
        vu = None if hv is None else hv.view(torch.uint32 if vb == 4 else torch.uint64)
        e_steps = max(1, min(args.steps, args.e2e_steps))
        e_ms = 0.0
        for i in range(e_steps + 1):
            hk.copy_(src_k)  # the unsorted input, back in pinned host memory (outside the timing)
            if hv is not None:
                hv.copy_(src_v)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dt_sort(RecordArray(ku, vu), cfg)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            if i > 0:
                e_ms += (t1 - t0) * 1e3
        e_ms /= e_steps
        e2e = {"value": round(n / (e_ms / 1e3) / 1e9, 4), "unit": UNIT,
               "h2d_bytes_per_step": n * (kb + vb), "d2h_bytes_per_step": n * (kb + vb),
               "ms_per_step": round(e_ms, 2), "steps": e_steps,
               "path": "dt_sort(RecordArray(pinned host tensors)) -> H2D, dts_sort, D2H"}
    elif multi and not args.no_e2e:
        # every rank: pinned host slice -> device, dist_sort, result -> pinned
        # host; max over ranks of the wall time between barriers.  One pinned
        # buffer per column holds the input and then the result (a rank
        # receives ~n records; 1/8 slack): 8 ranks x 10^9 u32/u32 records pin
        # ~72 GB of host memory, not ~160 GB
        cap = n + n // 8 + 4096
        hk = torch.empty(cap, dtype=src_k.dtype, pin_memory=True)
        hv = None if src_v is None else torch.empty(cap, dtype=src_v.dtype, pin_memory=True)
        e_steps = max(1, min(args.steps, args.e2e_steps))
        e_ms = 0.0
        out_bytes = 0
        for i in range(e_steps + 1):
            hk[:n].copy_(src_k)  # this rank's unsorted slice (outside the timed region)
            if hv is not None:
                hv[:n].copy_(src_v)
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            dk = hk[:n].to(dev, non_blocking=True)
            dv = None if hv is None else hv[:n].to(dev, non_blocking=True)
            rk, rv, st = dist_sort(dk, dv, ops=ops)
            m = rk.numel()
            ok_h = hk[:m] if m <= cap else torch.empty(m, dtype=rk.dtype, pin_memory=True)
            ok_h.copy_(rk, non_blocking=True)  # (the H2D above is done: same stream)
            ov_h = None
            if rv is not None:
                ov_h = hv[:m] if m <= cap else torch.empty(m, dtype=rv.dtype, pin_memory=True)
                ov_h.copy_(rv, non_blocking=True)
            torch.cuda.synchronize()
            t = torch.tensor([(time.perf_counter() - t0) * 1e3], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            if i > 0:
                e_ms += float(t.item())
            out_bytes = ok_h.numel() * ok_h.element_size() + (0 if ov_h is None else ov_h.numel() * ov_h.element_size())
            del dk, dv, rk, rv
        e_ms /= e_steps
        e2e = {"value": round(n * world / (e_ms / 1e3) / 1e9, 4), "unit": UNIT,
               "h2d_bytes_per_step": n * (kb + vb), "d2h_bytes_per_step": int(out_bytes),
               "ms_per_step": round(e_ms, 2), "steps": e_steps, "per_rank": True,
               "path": "per rank: pinned host slice -> H2D, distributed.dist_sort (NCCL all-to-all), D2H"}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        from oracle import oracle as ora

        ns, dts = cpu_bounded_sample(cfgd, seed=1, budget_s=args.cpu_budget)
        cpu = {"value": round(ns / dts / 1e9, 6), "unit": UNIT, "cores": ora.max_threads(),
               "kind": "port",
               "sample": f"{ns} records of the {args.config} workload sorted by the oracle "
                         f"(C++ restatement of the reference dt_sort) in {dts:.2f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
            "dtype": "u32" if kb == 4 else "u64",
            "data": "synthetic (seeded generator on device: torch, or libdts k_gen_rmat for c5)",
            "config": {"workload": args.config, "desc": cfgd["desc"], "n_per_gpu": n,
                       "key_bytes": kb, "val_bytes": vb, "parallelism": f"keyrange{world}" if multi else "single",
                       "l2": "inputs (n*(k+v) bytes) exceed the 126 MB L2; no flush needed",
                       "timed": ("CUDA events around each stream-ordered sort (ends when its last kernel "
                                 "does); per-step input restore outside; kernel shares from 3 profiled steps after"),
                       "checked": cert},
            "roofline": roof, "pipeline_roofline": pipe, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clk,
        }
        print(json.dumps(line), flush=True)


def free_port() -> int:
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def self_launch(args) -> int:
    """Re-exec this script as N torchrun ranks (one process per GPU).  Aborts
    when fewer than N GPUs are visible (a run on fewer GPUs would print a
    line for the wrong N)."""
    if args.impl == "ours" and not args.gloo_selftest:
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}",
                  file=sys.stderr)
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__)]
    # (torchrun's own parser would claim options such as --n: the ranks read
    # this script's arguments from the environment instead)
    env = dict(os.environ, DTS_BENCH_ARGV=json.dumps(sys.argv[1:]))
    return subprocess.call(cmd, env=env)


def run_gloo_selftest(args, cfgd, rank, world):
    """CPU check of the multi-rank launch (tests/test_bench_launch.py): the
    ranks join a gloo group, run distributed.dist_sort on a small seeded
    input through a host ops double, take the max over ranks of the step
    time and rank 0 prints the bench line shape with n_gpus = world."""
    import torch
    import torch.distributed as dist

    from paper_2401_00710_b200.distributed import dist_sort

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from dist_hostops import HostOps  # test double: no GPU in a gloo self-test

    dist.init_process_group("gloo")
    try:
        n = args.n or 4096
        rng = np.random.default_rng(1000 + rank)
        keys = torch.from_numpy(rng.integers(0, 10**9, size=n, dtype=np.uint32).view(np.int32))
        vals = torch.arange(rank * n, (rank + 1) * n, dtype=torch.int32)
        dist.barrier()
        t0 = time.perf_counter()
        rk, rv, st = dist_sort(keys, vals, ops=HostOps(), samples_per_rank=256)
        t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        got = torch.tensor([rk.numel()], dtype=torch.int64)
        dist.all_reduce(got)
        ok = bool((rk.to(torch.int64) & 0xFFFFFFFF).diff().ge(0).all()) if rk.numel() > 1 else True
        okt = torch.tensor([int(ok)], dtype=torch.int64)
        dist.all_reduce(okt, op=dist.ReduceOp.MIN)
        if rank == 0:
            print(json.dumps({"metric": METRIC, "value": round(n * world / float(t) / 1e9, 6),
                              "unit": UNIT, "n_gpus": world, "steps": 1, "warmup": 0,
                              "ms_per_step": round(float(t) * 1e3, 3), "selftest": "gloo",
                              "records_out": int(got), "sorted": bool(okt.item())}), flush=True)
    finally:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--force-dist", action="store_true",
                    help="run the multi-GPU path (dist_sort) even at world size 1 (testing)")
    ap.add_argument("--gloo-selftest", action="store_true",
                    help="CPU test of the multi-rank launch (gloo, host ops double; no GPU)")
    argv = json.loads(os.environ["DTS_BENCH_ARGV"]) if "DTS_BENCH_ARGV" in os.environ else None
    args = ap.parse_args(argv)
    cfgd = dict(CONFIGS[args.config])
    if args.n:
        cfgd["n"] = args.n
    if "WORLD_SIZE" not in os.environ and (args.gpus > 1 or (args.force_dist and args.impl == "ours")):
        # `python bench.py --gpus N` outside torchrun: launch N ranks (one per
        # GPU) under torch.distributed.run on 127.0.0.1 and relay rank 0's line
        sys.exit(self_launch(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "ours" and world != args.gpus and not args.gloo_selftest:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.gloo_selftest:
        run_gloo_selftest(args, cfgd, rank, world)
        return
    if args.impl == "reference":
        run_reference(args, cfgd, rank, world)
        return
    use_dist = world > 1 or args.force_dist
    if use_dist:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, cfgd, rank, world, local_rank)
    finally:
        if use_dist:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
