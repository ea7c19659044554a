"""bench.py -- A16Wx low-bit-weight matmul on B200 (the hot path of Tilus, arXiv 2504.12984).

Metric (BASELINE.json): "A16Wx matmul HBM GB/s & TFLOP/s vs bit width, batch 1/16/128,
Llama-70B layers".  Workload (BASELINE.json configs[2]): the four Llama-3.3-70B linear
layers (qkv 8192->10240, o 8192->8192, gate_up 8192->57344, down 28672->8192) in the
four formats u3, i5, f6e3m2, u8, group 128, uint formats with zero points.

A STEP is one pass of the whole hot path over one batch: 16 tl_matmul calls (4 layers x
4 formats) at batch M (default 1 = decode).  `value` = algorithmic bytes of the step
(packed weights + scales/zeros + A + Y) / device time, in GB/s.  Each step
streams ~2.5 GB of weights, far more than the 126 MB L2, so no flush is needed between
steps (inputs larger than L2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--M 1] [--impl ours|reference]

Multi-GPU (torchrun, one process per GPU): weak scaling -- rank r owns its own
column shard (the full layer width of the single-GPU problem) of a P-times wider
layer, computes it with no communication, and (only with --gather) all-gathers Y over
NCCL.  Time is the max over ranks of the device time.
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
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as wl  # noqa: E402

METRIC = "A16Wx matmul HBM GB/s & TFLOP/s vs bit width, batch 1/16/128, Llama-70B layers"
WORKLOAD = "llama-3.3-70b linear layers (qkv,o,gate_up,down) x {u3,i5,f6e3m2,u8}, group 128 (BASELINE configs[2])"


def alg_bytes(fmt: str, M: int, K: int, N: int, G: int) -> int:
    """Algorithmic bytes of one matmul: packed codes + scales (+zeros) + A + Y."""
    b = int(fmt[1])
    zp = 1 if fmt[0] == "u" else 0
    return K * N * b // 8 + (K // G) * N * 2 * (1 + zp) + 2 * M * K + 2 * M * N


def load_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"], "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback"}


class ClockSampler:
    """NVML sampler of SM clock + throttle reasons, run DURING the timed region."""

    REASONS = {
        0x0000000000000001: "gpu_idle", 0x0000000000000002: "applications_clocks_setting",
        0x0000000000000004: "sw_power_cap", 0x0000000000000008: "hw_slowdown", 0x0000000000000010: "sync_boost",
        0x0000000000000020: "sw_thermal_slowdown", 0x0000000000000040: "hw_thermal_slowdown",
        0x0000000000000080: "hw_power_brake_slowdown", 0x0000000000000100: "display_clock_setting",
    }

    def __init__(self, index: int, period_s: float = 0.002):
        self.index, self.period = index, period_s
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover - no NVML
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            time.sleep(self.period)

    def _sample(self):
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for bit, name in self.REASONS.items():
                if r & bit and name != "gpu_idle":
                    self.reasons.add(name)
        except Exception:
            pass

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self._stop.set()
            self._t.join()
            self._sample()

    def summary(self) -> dict:
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------------------------------
def _cpu_task(task):
    """One oracle evaluation (worker process): dequant + fp64 matmul of a column sample."""
    from threadpoolctl import threadpool_limits

    from oracle import dequant, matmul_fp64, parse_wtype
    fmt, lname, K, cols, G, M, rep = task
    with threadpool_limits(limits=1):
        seed = wl.stable_seed("cpu", fmt, lname, rep)
        codes = wl.gen_codes(fmt, K, cols, seed)
        s = wl.gen_scales(fmt, K, cols, G, seed)
        z = wl.gen_zeros(fmt, K, cols, G, seed)
        A = wl.gen_activations(M, K, seed)
        t0 = time.perf_counter()
        matmul_fp64(A, dequant(parse_wtype(fmt), codes, s, z, G))
        return alg_bytes(fmt, M, K, cols, G), time.perf_counter() - t0


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown CPU"


_CPU_POOL = None


def cpu_baseline(formats, layers, G, M, budget_s=12.0, impl_line=False):
    """The oracle as it stands, on ALL the host cores: independent column samples of every (format,
    layer) evaluated by one single-threaded worker process per core; throughput = algorithmic bytes
    of all samples / wall time of the parallel section (bounded to ~budget_s)."""
    import concurrent.futures as cf
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    cols = 64
    # calibrate (budget_s > 0): one pass over the pairs on one core gives the per-pass time
    one, t_pass, reps = None, 0.0, 1
    if budget_s > 0:
        t0 = time.perf_counter()
        one = [_cpu_task((fmt, lname, K, cols, G, M, 0)) for fmt in formats for lname, (K, N) in layers.items()]
        t_pass = time.perf_counter() - t0
        reps = max(1, min(200, int(budget_s * cores / max(t_pass, 1e-3))))
    tasks = [(fmt, lname, K, cols, G, M, r) for r in range(1, reps + 1) for fmt in formats
             for lname, (K, N) in layers.items()]
    global _CPU_POOL
    try:
        if _CPU_POOL is None:  # one pool per process, reused by every call (the reference arm's steps)
            import atexit
            _CPU_POOL = cf.ProcessPoolExecutor(max_workers=cores, mp_context=mp.get_context("spawn"))
            atexit.register(_CPU_POOL.shutdown, wait=True)
            list(_CPU_POOL.map(_cpu_task, tasks[:cores], chunksize=1))  # start-up of the workers, untimed
        ex = _CPU_POOL
        w0 = time.perf_counter()
        res = list(ex.map(_cpu_task, tasks, chunksize=max(1, len(tasks) // (4 * cores))))
        wall = time.perf_counter() - w0
        used = cores
    except Exception:  # no process pool on this host: a single-core pass
        if one is None:
            t0 = time.perf_counter()
            one = [_cpu_task((fmt, lname, K, cols, G, M, 0)) for fmt in formats for lname, (K, N) in layers.items()]
            t_pass = time.perf_counter() - t0
        res, wall, used, reps = one, t_pass, 1, 0
    tot_bytes = sum(b for b, _ in res)
    return {"value": tot_bytes / wall / 1e9, "unit": "GB/s", "cores": used, "kind": "oracle",
            "sample": f"{max(reps, 1)} pass(es) over {len(formats)}x{len(layers)} (format, layer) pairs, "
                      f"{cols} columns each, M={M}, numpy fp64, one single-threaded worker per core on "
                      f"{used} core(s) of {_cpu_model()}; {wall:.1f} s wall"}


def run_reference(args):
    """--impl reference: the oracle timed as it stands on the host cores, same metric/config."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    formats, layers = args.formats, {k: wl.LLAMA33_70B[k] for k in args.layers}
    for _ in range(args.warmup):
        cpu_baseline(formats, layers, 128, args.M, budget_s=0.0)
    t0 = time.perf_counter()
    vals = []
    for _ in range(args.steps):
        vals.append(cpu_baseline(formats, layers, 128, args.M, budget_s=0.0))
    dt = time.perf_counter() - t0
    v = statistics.median([x["value"] for x in vals])
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "M": args.M, "formats": formats, "layers": list(layers),
                       "group": 128, "sample": "64 columns per (format, layer)"},
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": vals[0]["cores"], "kind": "oracle",
                             "sample": vals[0]["sample"]},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2504_12984_b200 as P
    from paper_2504_12984_b200.dist import gather_columns

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        if args.gpus != world:
            raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    G = 128
    M = args.M
    layers = {k: wl.LLAMA33_70B[k] for k in args.layers}
    # resident model weights, prepared once before the timed region: the decode kernel's weight
    # stream may overlap the previous launch's tail (programmatic dependent launch, header)
    FLAGS = P.TL_FLAG_STATIC_WEIGHTS

    # ---- one-time weight preparation (untimed) ----
    probs = []
    for fmt in args.formats:
        w = P.wtype(fmt)
        for lname, (K, N) in layers.items():
            seed = wl.stable_seed("bench", fmt, lname, rank)
            codes = wl.gen_codes_torch(fmt, K, N, seed, dev)
            bs = P.tl_pack(w, K, N, codes)
            del codes
            wt = P.tl_transform_weights(w, K, N, bs)
            del bs
            s = wl.gen_scales_torch(fmt, K, N, G, seed, dev)
            z = wl.gen_zeros_torch(fmt, K, N, G, seed, dev)
            probs.append({"fmt": fmt, "layer": lname, "K": K, "N": N, "w": w, "wt": wt, "s": s, "z": z})
    torch.cuda.synchronize()
    ws_bytes = max(P.tl_matmul_workspace_bytes(p["w"], max(M, 128), p["N"], p["K"], G) for p in probs)
    ws = torch.zeros(ws_bytes, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def make_io(m):
        for p in probs:
            p["A"] = wl.gen_activations_torch(m, p["K"], wl.stable_seed("A", p["layer"], m, rank), dev)
            p["Y"] = torch.empty((m, p["N"]), dtype=torch.float16, device=dev)

    def step(m, events=None):
        for i, p in enumerate(probs):
            if events is not None:
                events[i][0].record(stream)
            P.tl_matmul_ex(p["w"], m, p["N"], p["K"], G, p["A"], p["wt"], p["s"], p["z"], p["Y"], ws, flags=FLAGS)
            if events is not None:
                events[i][1].record(stream)
            if args.gather:
                gather_columns(p["Y"], world * p["N"], world)

    def timed(m, steps, warmup, per_launch=True, sampler=None):
        """Device time of `steps` back-to-back steps.  The step's launches are captured once in a
        CUDA graph (no host launch overhead inside the timed region: the library's calls are
        graph-capturable -- no syncs, no allocations); per-launch times come from a second graph
        with external event-record nodes between the launches, replayed with a sync after each."""
        make_io(m)
        for _ in range(warmup):
            step(m)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step(m)
        for _ in range(warmup):
            g.replay()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ctx = sampler if sampler is not None else _Null()
        with ctx:
            t0.record(stream)
            for _ in range(steps):
                g.replay()
            t1.record(stream)
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = t0.elapsed_time(t1)
        launch_ms = None
        if per_launch:
            evs = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(len(probs) + 1)]
            g2 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g2):
                evs[0].record()
                for i, p in enumerate(probs):
                    P.tl_matmul_ex(p["w"], m, p["N"], p["K"], G, p["A"], p["wt"], p["s"], p["z"], p["Y"], ws,
                                   flags=FLAGS)
                    evs[i + 1].record()
            g2.replay()
            torch.cuda.synchronize()
            launch_ms = []
            for _ in range(max(3, min(steps, 10))):
                g2.replay()
                torch.cuda.synchronize()
                launch_ms.append([evs[i].elapsed_time(evs[i + 1]) for i in range(len(probs))])
            del g2
        del g
        ms_max = ms
        if world > 1:
            t = torch.tensor([ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_max = float(t.item())
        return ms_max, launch_ms

    peaks = load_peaks()
    sampler = ClockSampler(local)
    ms, launch_ms = timed(M, args.steps, args.warmup, per_launch=True, sampler=sampler)
    step_bytes = sum(alg_bytes(p["fmt"], M, p["K"], p["N"], G) for p in probs)
    step_flops = sum(2 * M * p["K"] * p["N"] for p in probs)
    ms_per_step = ms / args.steps
    value = world * step_bytes / (ms_per_step * 1e-3) / 1e9

    # per-(format, layer) detail and the dominant kernel's roofline
    path_names = {1: "gemv", 2: "tc", 3: "tcd"}
    details = []
    fam_bytes, fam_ms = {}, {}
    for i, p in enumerate(probs):
        lm = statistics.mean(row[i] for row in launch_ms)
        b = alg_bytes(p["fmt"], M, p["K"], p["N"], G)
        path, _ = P.tl_matmul_plan(p["w"], M, p["N"], p["K"], G)
        fam = path_names.get(path, str(path))
        fam_bytes[fam] = fam_bytes.get(fam, 0) + b
        fam_ms[fam] = fam_ms.get(fam, 0.0) + lm
        details.append({"fmt": p["fmt"], "layer": p["layer"], "M": M, "us": round(lm * 1e3, 2),
                        "GBps": round(b / (lm * 1e-3) / 1e9, 1),
                        "hbm_frac": round(b / (lm * 1e-3) / 1e9 / peaks["hbm_gbs"], 3), "path": fam})
    dom = max(fam_ms, key=fam_ms.get)
    if len(fam_ms) == 1:
        # every launch of the step is the same kernel: its achieved bandwidth is the step's own
        # device time (one graph replay, launches overlapped by programmatic dependent launch);
        # the per-launch event nodes of the breakdown graph serialise the launches and add gaps
        achieved = step_bytes / (ms_per_step * 1e-3) / 1e9
        dom_share = 1.0
    else:
        achieved = fam_bytes[dom] / (fam_ms[dom] * 1e-3) / 1e9
        dom_share = fam_ms[dom] / sum(fam_ms.values())
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(f"{dom}_M{M}")
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": round(achieved / peaks["hbm_gbs"], 4), "traffic": traffic, "kernel": dom,
                "peak_source": peaks["source"], "share_of_step": round(dom_share, 3),
                "traffic_scope": "DRAM read+write bytes per step of this kernel's launches (ncu launch list, "
                                 "profiles/traffic.json); algorithmic bytes per step = %d" % step_bytes}

    # ---- extra batch sizes (reported, not part of `value`) ----
    extra = []
    extra_steps = []
    if not args.no_extra:
        for m2 in [x for x in (16, 64, 128) if x != M]:
            n2 = max(3, min(args.steps, 10))
            ms2, lms2 = timed(m2, n2, 2, per_launch=True)
            # the whole 16-launch step at this batch (one graph, launches overlapped): the throughput a
            # caller sees; the per-launch rows below come from the serialising event graph
            sb = sum(alg_bytes(p["fmt"], m2, p["K"], p["N"], G) for p in probs)
            sf = sum(2 * m2 * p["K"] * p["N"] for p in probs)
            st = ms2 / n2 * 1e-3
            extra_steps.append({"M": m2, "step_us": round(st * 1e6, 1), "GBps": round(sb / st / 1e9, 1),
                                "TFLOPs": round(sf / st / 1e12, 1),
                                "tensor_frac_fp16": round(sf / st / 1e12 / peaks["bf16_tflops"], 3)})
            for i, p in enumerate(probs):
                lm = statistics.mean(row[i] for row in lms2)
                b = alg_bytes(p["fmt"], m2, p["K"], p["N"], G)
                fl = 2 * m2 * p["K"] * p["N"]
                extra.append({"fmt": p["fmt"], "layer": p["layer"], "M": m2, "us": round(lm * 1e3, 2),
                              "GBps": round(b / (lm * 1e-3) / 1e9, 1),
                              "TFLOPs": round(fl / (lm * 1e-3) / 1e12, 2),
                              "tensor_frac_fp16": round(fl / (lm * 1e-3) / 1e12 / peaks["bf16_tflops"], 3)})
        make_io(M)

    # ---- end to end through the public C-ABI with host buffers: every step, ONE host->device copy of
    # the step's activations (all 16 layers' A, pinned), the 16 matmuls, ONE device->host copy of the
    # 16 outputs (tl_matmul_batch_hostio) ----
    e2e = None
    if not args.no_e2e:
        make_io(M)
        a_elems = sum(M * p["K"] for p in probs)
        y_elems = sum(M * p["N"] for p in probs)
        A_host = torch.empty(a_elems, dtype=torch.float16, pin_memory=True)
        off = 0
        for p in probs:
            A_host[off:off + M * p["K"]].copy_(p["A"].reshape(-1).cpu())
            off += M * p["K"]
        A_dev = torch.empty(a_elems, dtype=torch.float16, device=dev)
        Y_dev = torch.empty(y_elems, dtype=torch.float16, device=dev)
        Y_host = torch.empty(y_elems, dtype=torch.float16, pin_memory=True)
        items = P.batch_items([{"w": p["w"], "group": G, "M": M, "N": p["N"], "K": p["K"], "w_t": p["wt"],
                                "scales": p["s"], "zeros": p["z"], "workspace": ws} for p in probs])

        def step_e2e():
            P.tl_matmul_batch_hostio(items, len(probs), A_host, A_dev, Y_dev, Y_host, flags=FLAGS)

        for _ in range(args.warmup):
            step_e2e()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):
            step_e2e()
        t1.record(stream)
        torch.cuda.synchronize()
        ems = t0.elapsed_time(t1)
        if world > 1:
            t = torch.tensor([ems], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": round(world * step_bytes / (ems / args.steps * 1e-3) / 1e9, 1), "unit": "GB/s",
               "h2d_bytes_per_step": sum(2 * M * p["K"] for p in probs),
               "d2h_bytes_per_step": sum(2 * M * p["N"] for p in probs),
               "ms_per_step": round(ems / args.steps, 4)}

    # ---- north-star coverage: all 37 formats x 70B layers x M in {1, 16} (rank 0 only) ----
    spectrum = run_spectrum(args, P, torch, dev, peaks) if (rank == 0 and not args.no_spectrum) else None

    # ---- BASELINE configs[1] (C2): Llama-3-8B decode layers x 22 formats x M in {1, 16} (rank 0) ----
    c2 = run_c2(args, P, torch, dev, peaks) if (rank == 0 and not args.no_spectrum) else None

    # ---- row f4: int8 activations and MX weights (rank 0 only) ----
    f4 = run_f4(args, P, torch, dev, peaks) if (rank == 0 and not args.no_spectrum) else None

    # ---- C5 (BASELINE configs[4]): Llama-3.3-70B gate_up strong-scaled over the ranks ----
    c5 = None if args.no_c5 else run_c5(args, P, torch, dist, world, rank, dev, peaks)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f16", "data": "synthetic",
            "config": {"workload": WORKLOAD, "M": M, "formats": args.formats, "layers": list(layers), "group": 128,
                       "weights": "uint formats with fp16 zero points; int/float symmetric",
                       "l2": "inputs larger than L2: each step streams %.2f GB of weights (L2 126 MB)" %
                             (step_bytes / 1e9),
                       "parallelism": f"column shards, {world} rank(s), no data-path collective" +
                                      (" + NCCL all-gather of Y" if args.gather else ""),
                       "tflops_at_M": round(step_flops / (ms_per_step * 1e-3) / 1e12, 3)},
            "roofline": roofline,
            "e2e": e2e,
            "gpu_launches": args.steps * len(probs),
            "clocks": sampler.summary(),
            "details": details,
            "details_extra_M": extra,
            "details_extra_M_steps": extra_steps,
            "details_c5": c5,
            "details_spectrum": spectrum,
            "details_f4": f4,
            "details_c2": c2,
        }
        if world == 1 and not args.no_cpu:
            line["cpu_baseline"] = cpu_baseline(args.formats, layers, G, M)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_spectrum(args, P, torch, dev, peaks):
    """North-star coverage (every bit width 1-8, int / uint / float, PAPER.md:518-523 fig:exp_coverage):
    all 37 kernel formats on the four Llama-3.3-70B layers at M = 1 and M = 16 (gate_up at M = 16
    is the paper's coverage shape BS=16, K=8192, N=57344), and gate_up at M = 128 (the batch-128
    target, with the fraction of the dense fp16 peak).  Device time of one tl_matmul_ex per
    (format, layer, M), 10 back-to-back launches after 3 warm-ups; algorithmic GB/s and the fraction
    of the measured HBM copy bandwidth."""
    from oracle import all_kernel_formats
    G = 128
    out = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for f in all_kernel_formats():
        fmt = f.name
        w = P.wtype(fmt)
        for lname, (K, N) in wl.LLAMA33_70B.items():
            seed = wl.stable_seed("spectrum", fmt, lname)
            codes = wl.gen_codes_torch(fmt, K, N, seed, dev)
            wt = P.tl_transform_weights(w, K, N, P.tl_pack(w, K, N, codes))
            del codes
            s = wl.gen_scales_torch(fmt, K, N, G, seed, dev)
            z = wl.gen_zeros_torch(fmt, K, N, G, seed, dev)
            ws = torch.zeros(max(P.tl_matmul_workspace_bytes(w, 16, N, K, G),
                                 P.tl_matmul_workspace_bytes(w, 128, N, K, G)), dtype=torch.uint8, device=dev)
            for M in ((1, 16, 128) if lname == "gate_up" else (1, 16)):
                A = wl.gen_activations_torch(M, K, seed, dev)
                Y = torch.empty((M, N), dtype=torch.float16, device=dev)
                for _ in range(3):
                    P.tl_matmul_ex(w, M, N, K, G, A, wt, s, z, Y, ws, flags=P.TL_FLAG_STATIC_WEIGHTS)
                e0.record()
                for _ in range(10):
                    P.tl_matmul_ex(w, M, N, K, G, A, wt, s, z, Y, ws, flags=P.TL_FLAG_STATIC_WEIGHTS)
                e1.record()
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) / 10 * 1e3
                b = alg_bytes(fmt, M, K, N, G)
                rec = {"fmt": fmt, "layer": lname, "M": M, "us": round(us, 2),
                       "GBps": round(b / (us * 1e-6) / 1e9, 1),
                       "hbm_frac": round(b / (us * 1e-6) / 1e9 / peaks["hbm_gbs"], 3)}
                if M == 128:  # tensor-bound for b <= 7: the fraction of the dense fp16 peak
                    fl = 2 * M * K * N
                    rec["TFLOPs"] = round(fl / (us * 1e-6) / 1e12, 1)
                    rec["tensor_frac_fp16"] = round(fl / (us * 1e-6) / 1e12 / peaks["bf16_tflops"], 3)
                out.append(rec)
            del wt, s, z, ws
    return out


def run_c2(args, P, torch, dev, peaks):
    """BASELINE configs[1] / SURVEY C2: the Llama-3-8B decode linear layers (q, k, v, o, gate_up, down)
    at M = 1 and 16 for the 22 formats of P:521's coverage (uint1..8, int1..8, f3e1m1, f4e2m1,
    f5e2m2, f6e3m2, f7e3m3, f8e4m3), group 128: device time of one tl_matmul_ex (10 back-to-back
    launches after 3 warm-ups), algorithmic GB/s and the fraction of the measured HBM bandwidth.
    The 8B layers are 0.5-121 MB: the smaller ones sit below the per-launch floor."""
    G = 128
    out = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for fmt in wl.CONFIG1_FORMATS:
        w = P.wtype(fmt)
        for lname, (K, N) in wl.LLAMA3_8B.items():
            seed = wl.stable_seed("c2", fmt, lname)
            wt = P.tl_transform_weights(w, K, N, P.tl_pack(w, K, N, wl.gen_codes_torch(fmt, K, N, seed, dev)))
            s = wl.gen_scales_torch(fmt, K, N, G, seed, dev)
            z = wl.gen_zeros_torch(fmt, K, N, G, seed, dev)
            ws = torch.zeros(P.tl_matmul_workspace_bytes(w, 16, N, K, G), dtype=torch.uint8, device=dev)
            for M in (1, 16):
                A = wl.gen_activations_torch(M, K, seed, dev)
                Y = torch.empty((M, N), dtype=torch.float16, device=dev)
                for _ in range(3):
                    P.tl_matmul_ex(w, M, N, K, G, A, wt, s, z, Y, ws, flags=P.TL_FLAG_STATIC_WEIGHTS)
                e0.record()
                for _ in range(10):
                    P.tl_matmul_ex(w, M, N, K, G, A, wt, s, z, Y, ws, flags=P.TL_FLAG_STATIC_WEIGHTS)
                e1.record()
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) / 10 * 1e3
                b = alg_bytes(fmt, M, K, N, G)
                out.append({"fmt": fmt, "layer": lname, "M": M, "us": round(us, 2),
                            "GBps": round(b / (us * 1e-6) / 1e9, 1),
                            "hbm_frac": round(b / (us * 1e-6) / 1e9 / peaks["hbm_gbs"], 3)})
            del wt, s, z, ws
    return out


def run_f4(args, P, torch, dev, peaks):
    """SURVEY §8(f) row f4 measured on the 70B layers at M = 1 and 16 (one tl_matmul per (case, layer, M),
    10 back-to-back launches after 3 warm-ups, device time):
      * int8 activations (TL_ACT_I8; u3 / i5 / f6e3m2 / u8 weights, G = 128): the staging kernel plus
        the fp16 path; algorithmic bytes count A at one byte per element;
      * MX weights (group 32 with E8M0 scales converted once by tl_mx_scales_to_f16): fp4 e2m1,
        fp6 e2m3, fp6 e3m2, fp8 e4m3 and MXINT8 (int8 x 2^-6); algorithmic bytes = codes + one fp16
        scale per 32 weights + A + Y."""
    out = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def clock(fn):
        for _ in range(3):
            fn()
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 10 * 1e3

    for lname in ("qkv", "gate_up"):
        K, N = wl.LLAMA33_70B[lname]
        for fmt in ("u3", "i5", "f6e3m2", "u8"):
            G = 128
            w = P.wtype(fmt)
            seed = wl.stable_seed("f4-a8", fmt, lname)
            wt = P.tl_transform_weights(w, K, N, P.tl_pack(w, K, N, wl.gen_codes_torch(fmt, K, N, seed, dev)))
            s = wl.gen_scales_torch(fmt, K, N, G, seed, dev)
            z = wl.gen_zeros_torch(fmt, K, N, G, seed, dev)
            for M in (1, 16):
                ws = torch.zeros(P.tl_matmul_workspace_bytes(w, M, N, K, G, P.TL_ACT_I8), dtype=torch.uint8,
                                 device=dev)
                A8 = torch.randint(-128, 128, (M, K), dtype=torch.int8, device=dev)
                Y = torch.empty((M, N), dtype=torch.float16, device=dev)
                us = clock(lambda: P.tl_matmul_ex(w, M, N, K, G, A8, wt, s, z, Y, ws, flags=P.TL_FLAG_STATIC_WEIGHTS))
                b = alg_bytes(fmt, M, K, N, G) - M * K
                out.append({"case": "a8", "fmt": fmt, "layer": lname, "M": M, "us": round(us, 2),
                            "GBps": round(b / (us * 1e-6) / 1e9, 1),
                            "hbm_frac": round(b / (us * 1e-6) / 1e9 / peaks["hbm_gbs"], 3)})
            del wt, s, z
        for name, fmt, adj, center in (("mxfp4", "f4e2m1", 0, 119), ("mxfp6_e2m3", "f6e2m3", 0, 120),
                                       ("mxfp6_e3m2", "f6e3m2", 0, 117), ("mxfp8_e4m3", "f8e4m3", 0, 115),
                                       ("mxint8", "i8", -6, 121)):
            G = 32
            w = P.wtype(fmt)
            seed = wl.stable_seed("f4-mx", fmt, lname)
            wt = P.tl_transform_weights(w, K, N, P.tl_pack(w, K, N, wl.gen_codes_torch(fmt, K, N, seed, dev)))
            e8 = torch.randint(center - 3, center + 4, (K // G, N), dtype=torch.int32, device=dev).to(torch.uint8)
            s = P.tl_mx_scales_to_f16(e8, adj)
            for M in (1, 16):
                ws = torch.zeros(P.tl_matmul_workspace_bytes(w, M, N, K, G), dtype=torch.uint8, device=dev)
                A = wl.gen_activations_torch(M, K, seed, dev)
                Y = torch.empty((M, N), dtype=torch.float16, device=dev)
                us = clock(lambda: P.tl_matmul_ex(w, M, N, K, G, A, wt, s, None, Y, ws, flags=P.TL_FLAG_STATIC_WEIGHTS))
                b = alg_bytes(fmt, M, K, N, G)
                path, _ = P.tl_matmul_plan(w, M, N, K, G)
                out.append({"case": name, "fmt": fmt, "layer": lname, "M": M, "us": round(us, 2),
                            "GBps": round(b / (us * 1e-6) / 1e9, 1),
                            "hbm_frac": round(b / (us * 1e-6) / 1e9 / peaks["hbm_gbs"], 3), "path": path})
            del wt, s
    return out


def run_c5(args, P, torch, dist, world, rank, dev, peaks):
    """gate_up (K=8192, N=57344) column-sharded over the `world` ranks
    (strong scaling: rank r owns columns column_shard(N, world, r), 57344/P of them), uint4 with
    zeros and int6, M in {1, 16, 128}.  `sharded_us`: the max over ranks of the device time of the
    rank's tl_matmul (no communication); `gathered_us`: tl_matmul followed by
    the NCCL all-gather of the Y shards into Y[M, N] (north star (5)), same timing.  With one rank
    the gathered variant is the plain matmul."""
    from paper_2504_12984_b200.dist import column_shard, gather_columns
    K, N = wl.LLAMA33_70B["gate_up"]
    G = 128
    n0, n1 = column_shard(N, world, rank)
    Ns = n1 - n0
    out = []
    reps = 20
    for fmt in ("u4", "i6"):
        w = P.wtype(fmt)
        seed = wl.stable_seed("c5", fmt, rank)
        codes = wl.gen_codes_torch(fmt, K, Ns, seed, dev)
        wt = P.tl_transform_weights(w, K, Ns, P.tl_pack(w, K, Ns, codes))
        del codes
        s = wl.gen_scales_torch(fmt, K, Ns, G, seed, dev)
        z = wl.gen_zeros_torch(fmt, K, Ns, G, seed, dev)
        ws = torch.zeros(P.tl_matmul_workspace_bytes(w, 128, Ns, K, G), dtype=torch.uint8, device=dev)
        for M in (1, 16, 128):
            A = wl.gen_activations_torch(M, K, wl.stable_seed("c5A", M), dev)
            Y = torch.empty((M, Ns), dtype=torch.float16, device=dev)
            res = {}
            fg = None
            variants = ["sharded", "gathered"]
            if args.fused_gather:
                # row f3: the all-gather fused into the epilogue over NVLink peer memory (opt-in)
                from paper_2504_12984_b200.dist import FusedGather, peer_pointers
                fg = FusedGather(M, N, world, rank)
                variants.append("fused")
            for variant in variants:
                def once():
                    if variant == "fused":
                        fg.epoch += 1
                        b = fg.epoch % fg.nbuf
                        ys, fs = peer_pointers(fg.y_bases[b], fg.f_bases, rank, n0)
                        P.tl_matmul_gathered(w, M, Ns, K, G, A, wt, s, z, fg.Yg[b][:, n0:], N, ys, fs, ws,
                                             flags=P.TL_FLAG_STATIC_WEIGHTS)
                        P.tl_gather_wait(fg.flags, world, rank, fg.epoch)
                        return
                    P.tl_matmul_ex(w, M, Ns, K, G, A, wt, s, z, Y, ws, flags=P.TL_FLAG_STATIC_WEIGHTS)
                    if variant == "gathered" and world > 1:
                        gather_columns(Y, N, world)
                for _ in range(3):
                    once()
                torch.cuda.synchronize()
                if world > 1:
                    dist.barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(reps):
                    once()
                e1.record()
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) / reps * 1e3
                if world > 1:
                    t = torch.tensor([us], device=dev, dtype=torch.float64)
                    dist.all_reduce(t, op=dist.ReduceOp.MAX)
                    us = float(t.item())
                res[variant] = us
            byts = alg_bytes(fmt, M, K, N, G)
            out.append({"fmt": fmt, "M": M, "P": world, "shard_cols": Ns, "sharded_us": round(res["sharded"], 2),
                        "gathered_us": round(res["gathered"], 2),
                        "fused_gathered_us": round(res["fused"], 2) if "fused" in res else None,
                        "GBps_total": round(byts / (res["sharded"] * 1e-6) / 1e9, 1),
                        "hbm_frac_per_gpu": round(byts / world / (res["sharded"] * 1e-6) / 1e9 / peaks["hbm_gbs"], 3),
                        "TFLOPs_total": round(2 * M * K * N / (res["sharded"] * 1e-6) / 1e12, 2)})
        del wt, s, z, ws
    return out


def torchrun_argv(n: int, argv: list[str], port: int) -> list[str]:
    """The command that relaunches this script with one process per GPU (the driver's own launch
    form: torch.distributed.run, one node, rendezvous on 127.0.0.1)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
            "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + argv


def _free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--M", type=int, default=1)
    ap.add_argument("--formats", nargs="+", default=wl.CONFIG2["formats"])
    ap.add_argument("--layers", nargs="+", default=list(wl.LLAMA33_70B))
    ap.add_argument("--gather", action="store_true")
    ap.add_argument("--fused-gather", action="store_true",
                    help="details_c5 also times the all-gather fused into the epilogue (row f3, CUDA IPC peers)")
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c5", action="store_true", help="skip the strong-scaled gate_up (configs[4]) block")
    ap.add_argument("--no-spectrum", action="store_true", help="skip the 37-format coverage table")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N`: start the N ranks ourselves (one process per GPU, NCCL)
        import subprocess
        sys.exit(subprocess.call(torchrun_argv(args.gpus, sys.argv[1:], _free_port())))
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
