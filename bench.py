"""Benchmark of the one-pass quaternion LRA hot path (BASELINE.json metric:
"one-pass LRA wall time & sketch quaternion TFLOP/s (% of FP64 peak)").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

A step is one one-pass LRA over the config's synthetic matrix: fused dual
sketch (one read of A) + pseudo-QR rangefinder + core solve X = (Psi H)\\W,
row-sharded across ranks with NCCL all-reduces of W / Grams / Psi H (strong
scaling: the matrix is fixed, N GPUs share it).  `value` is seconds per
one-pass LRA with A resident in HBM; `e2e` is the same through the public API
with A in pinned host memory (H2D inside the timed region) and H, X read back.
"""
from __future__ import annotations

import argparse
import json
import gc
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG_DEFAULT = "C2"
METRIC = "one-pass LRA wall time"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default=CFG_DEFAULT)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--rangefinder", default="pseudo_qr", choices=["pseudo_qr", "pseudo_svd"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    return p.parse_args()


# ------------------------------------------------------------ clocks ---
class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region (NVML,
    every 20 ms; nvidia-smi fallback)."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._ready = threading.Event()
        # NVML is imported and initialised here, before the timed region: a
        # cold `import pynvml` inside it holds the GIL and stalls the thread
        # that launches the kernels (seen as +30 ms steps)
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self._nvml = (pynvml, h, pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self._nvml = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        if self._nvml is not None:
            pynvml, h, mx = self._nvml
            bits = [("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
                    ("sw_power_cap", 0x4)]
            try:
                while not self._stop.is_set():
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append([str(sm), str(mx)] + ["Active" if r & b else "Not Active" for _, b in bits])
                    self._ready.set()
                    self._stop.wait(0.02)
                return
            except Exception:
                pass
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._ready.set()
            self._stop.wait(0.2)

    def __enter__(self):
        if os.environ.get("QLRA_BENCH_NO_CLOCKS"):  # A/B of the sampler's own interference
            return self
        self._t.start()
        self._ready.wait(timeout=10)  # sampling is running before timing starts
        self.samples.clear()          # keep only samples from inside the timed region
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t.is_alive():
            self._t.join(timeout=10)
            if not self.samples and self._nvml is not None:
                # timed region shorter than the sampling period (C1): one
                # sample at its end
                try:
                    pynvml, h, mx = self._nvml
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append([str(sm), str(mx)] + ["Active" if r & b else "Not Active"
                                                              for b in (0x8, 0x40, 0x20, 0x4)])
                except Exception:
                    pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------- CPU legs ---
def cpu_leg(cfg, y_h, w_h, a_rows_h, nthreads, method):
    """The reference hot path as restated by the CPU oracle: the serial
    ordered sketch on a leading row block (extrapolated linearly -- per-row
    cost is exactly constant in qmat_mul_accumulate_ordered) plus the full
    rangefinder and core solve on full-size Y, W."""
    from oracle import oracle as O
    b = a_rows_h.shape[1]
    ys = np.zeros((4, cfg.m, cfg.s))
    ws = np.zeros((4, cfg.l, cfg.n))
    t0 = time.perf_counter()
    O.sketch_update_rows(ys, ws, 0, a_rows_h, 1, 2, cfg.kind, 1.0, nthreads)
    t_sk = (time.perf_counter() - t0) * cfg.m / b
    qb = O.qb_stage(y_h, w_h, 2, method, kind=cfg.kind, nthreads=nthreads)
    return t_sk + qb["rangefinder_s"] + qb["solve_s"], t_sk, qb["rangefinder_s"], qb["solve_s"]


def sample_rows(cfg, nthreads):
    # ~2 s of serial sketch work per thread at ~2 GFLOP/s, at least 32 rows
    per_row = 32.0 * cfg.n * (cfg.s + cfg.l)
    return int(max(32, min(cfg.m, 2.0 * 2e9 * nthreads / per_row)))


def run_reference(args):
    """--impl reference: the reference's CPU path (oracle port; the C++
    reference itself cannot build here -- Eigen absent) on all host threads."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import torch  # noqa: F401  (torch not used on this arm beyond import parity)
    from oracle import oracle as O
    from paper_2404_14783_b200.configs import CONFIGS
    cfg = CONFIGS[args.config]
    nthreads = os.cpu_count() or 1
    method = 0 if args.rangefinder == "pseudo_qr" else 1
    a = cpu_matrix(cfg, nthreads)
    y, w = O.make_sketch(a, cfg.s - 5, cfg.s, cfg.l, 1, 2, cfg.kind, nthreads=nthreads)
    b = sample_rows(cfg, nthreads)
    times = []
    for it in range(args.warmup + args.steps):
        t, *_ = cpu_leg(cfg, y, w, np.ascontiguousarray(a[:, :b]), nthreads, method)
        if it >= args.warmup:
            times.append(t)
    v = float(np.mean(times))
    line = {"metric": METRIC, "value": v, "unit": "s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{cfg.name} {cfg.m}x{cfg.n} fp64 quaternion, s={cfg.s}, l={cfg.l}, "
                                   f"{args.rangefinder}", "parallelism": "cpu"},
            "cpu_baseline": {"value": v, "unit": "s", "cores": nthreads, "kind": "port",
                             "sample": f"sketch on leading {b}/{cfg.m} rows (extrapolated); "
                                       f"rangefinder + solve full size"},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_matrix(cfg, nthreads):
    """The config's A regenerated on the CPU with the same RNG (C1-C3 only)."""
    from oracle import oracle as O
    from paper_2404_14783_b200.configs import substream_key
    ds = cfg.data_seed
    rank = {"C1": 50, "C2": 400, "C3": 200}[cfg.name]
    g1 = O.gen_test_matrix(O.GAUSSIAN, cfg.m, rank, substream_key(ds, 1), nthreads=nthreads)
    g2 = O.gen_test_matrix(O.GAUSSIAN, rank, cfg.n, substream_key(ds, 2), nthreads=nthreads)
    if cfg.name == "C2":
        g1 = g1 * (np.arange(1, rank + 1, dtype=np.float64) ** -2.0)[None, None, :]
    a = O.qmat_mul(g1, g2)
    if cfg.name in ("C1", "C3"):
        a += (1e-3 if cfg.name == "C1" else 1e-6) * O.gen_test_matrix(
            O.GAUSSIAN, cfg.m, cfg.n, substream_key(ds, 3), nthreads=nthreads)
    return a


# ------------------------------------------------------------- ours ---
def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2404_14783_b200 import qlra as Q
    from paper_2404_14783_b200.configs import CONFIGS, build_matrix

    cfg = CONFIGS[args.config]
    nccl_id = None
    if world > 1:
        obj = [Q.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    ctx = Q.Context(local, rank, world, nccl_id)
    Q.set_default_context(ctx)
    r0, r1 = Q.shard_rows(cfg.m, world, rank)
    a = build_matrix(cfg, (r0, r1), ctx)
    torch.cuda.synchronize()
    # release the generator's temporaries held in torch's cache (C5: tens of
    # GB), which otherwise crowd the library's stream-ordered pool
    torch.cuda.empty_cache()
    method = Q.PSEUDO_QR if args.rangefinder == "pseudo_qr" else Q.PSEUDO_SVD
    opts = Q.OnePassOptions(r=cfg.s - 5, s=cfg.s, l=cfg.l, rangefinder=method, embedding=cfg.kind)
    stream = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    sk_events = []
    host_ms = []
    dev_allocs = []

    used = {"rangefinder": args.rangefinder}

    def step(a_dev):
        nonlocal method
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        h0 = time.perf_counter()
        st = Q.make_sketch(a_dev, opts.r, opts.s, opts.l, opts.omega_seed, opts.psi_seed, cfg.kind,
                           ctx=ctx, row0=r0, m_global=cfg.m)
        host_ms.append(1e3 * (time.perf_counter() - h0))
        if os.environ.get("QLRA_BENCH_STEPTIMES"):
            ms_ = torch.cuda.memory_stats()
            dev_allocs.append((ms_.get("num_device_alloc", -1), ms_.get("num_alloc_retries", -1)))
        e1.record(stream)
        sk_events.append((e0, e1))
        try:
            qb = Q.qb_stage(st, method, ctx=ctx)
        except Q.RankError:
            # pseudo-QR refuses kappa(H) beyond its domain exactly as the
            # reference does ("use pseudo_svd", rangefinders.cpp:122-123);
            # follow that advice and record it (C3: kappa(Y) ~ 1e8).
            method = Q.PSEUDO_SVD
            used["rangefinder"] = "pseudo_svd (pseudo_qr raised RankError, as the reference does)"
            qb = Q.qb_stage(st, method, ctx=ctx)
        return st, qb

    for _ in range(args.warmup):
        step(a)
    barrier()
    sk_events.clear()
    # torch's caching allocator only settles after a few steps of this
    # allocation pattern (two generations of Y, W, H, X alive); a reserved
    # segment carved up by later allocations keeps cudaMalloc -- which blocks
    # the host -- out of the timed region
    # (sized for two generations of this config's Y, W, H and X)
    per_step = 32 * ((r1 - r0) * cfg.s * 2 + cfg.l * cfg.n + cfg.s * cfg.n)
    _reserve = torch.empty(int(max(512e6, 2.2 * per_step)) // 8, dtype=torch.float64, device="cuda")
    del _reserve
    ctx.kernel_timing(True)
    launches0 = ctx.launch_count()
    gc.collect()
    gc.disable()  # no collector pause inside the timed region (it stalls the launching thread)
    with ClockSampler(local) as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        vstep_ev = []
        for _ in range(args.steps):
            if os.environ.get("QLRA_BENCH_STEPTIMES"):
                vstep_ev.append(torch.cuda.Event(enable_timing=True))
                vstep_ev[-1].record(stream)
            st, qb = step(a)
        t1.record(stream)
        barrier()
    gc.enable()
    if vstep_ev and rank == 0:
        vstep_ev.append(t1)
        sys.stderr.write("value per step ms: " + " ".join(
            "%.2f" % vstep_ev[i].elapsed_time(vstep_ev[i + 1]) for i in range(len(vstep_ev) - 1)) + "\n")
    launches = ctx.launch_count() - launches0
    if os.environ.get("QLRA_BENCH_STEPTIMES") and rank == 0:
        sys.stderr.write("sketch per step ms: " + " ".join("%.2f" % e0.elapsed_time(e1) for e0, e1 in sk_events) + "\n")
        sys.stderr.write("make_sketch host ms: " + " ".join("%.2f" % v for v in host_ms[-len(sk_events):]) + "\n")
        sys.stderr.write("torch device allocs/retries: " + " ".join("%d/%d" % v for v in dev_allocs) + "\n")
    kst = ctx.kernel_stats()
    ctx.kernel_timing(False)
    ms = t0.elapsed_time(t1) / args.steps
    sk_ms = float(np.mean([e0.elapsed_time(e1) for e0, e1 in sk_events]))
    k_ms = kst["ms"] / max(1, kst["launches"])  # fused sketch kernel, per launch
    tt = torch.tensor([ms, sk_ms, k_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms, sk_ms, k_ms = float(tt[0]), float(tt[1]), float(tt[2])

    # parity sanity on the measured result (second read of A, not timed)
    res, an = Q.residual_fro(a, qb.h, qb.x, ctx)

    # e2e: A from pinned host memory through the public API, H and X back
    e2e = None
    if not args.no_e2e:
        a_host = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
        a_host.copy_(a)
        del a
        torch.cuda.empty_cache()
        h_host = torch.empty((4, r1 - r0, cfg.s), dtype=torch.float64, pin_memory=True)
        x_host = torch.empty((4, cfg.s, cfg.n), dtype=torch.float64, pin_memory=True)

        e2e_opts = Q.OnePassOptions(r=cfg.s - 5, s=cfg.s, l=cfg.l, rangefinder=method, embedding=cfg.kind)

        def e2e_step():
            # public host-in/host-out API (one C-ABI call): A streams from
            # pinned host memory with the H2D overlapped by the sketch, H is
            # copied back while the core solve runs, then X
            Q.one_pass_qb_host(a_host, e2e_opts, ctx=ctx, row0=r0, m_global=cfg.m, h_out=h_host, x_out=x_host)

        for _ in range(args.warmup):
            e2e_step()
        barrier()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        # (sized for two generations of this config's Y, W, H and X)
        per_step = 32 * ((r1 - r0) * cfg.s * 2 + cfg.l * cfg.n + cfg.s * cfg.n)
        _reserve = torch.empty(int(max(512e6, 2.2 * per_step)) // 8, dtype=torch.float64, device="cuda")
        del _reserve
        gc.collect()
        gc.disable()
        s0.record(stream)
        step_ev = []
        for _ in range(args.steps):
            if os.environ.get("QLRA_BENCH_STEPTIMES"):
                step_ev.append(torch.cuda.Event(enable_timing=True))
                step_ev[-1].record(stream)
            e2e_step()
        s1.record(stream)
        barrier()
        gc.enable()
        if step_ev and rank == 0:
            step_ev.append(s1)
            sys.stderr.write("e2e per step ms: " + " ".join(
                "%.2f" % step_ev[i].elapsed_time(step_ev[i + 1]) for i in range(len(step_ev) - 1)) + "\n")
        e2e_ms = torch.tensor([s0.elapsed_time(s1) / args.steps], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
        e2e = {"value": float(e2e_ms) / 1e3, "unit": "s",
               "h2d_bytes_per_step": int(32 * (r1 - r0) * cfg.n),
               "d2h_bytes_per_step": int(32 * ((r1 - r0) * cfg.s + cfg.s * cfg.n))}
        a = a_host.to("cuda")

    peaks = {"dfma_tflops": Q.measure_fp64_peak(0, 300.0, ctx), "dmma_tflops": Q.measure_fp64_peak(1, 300.0, ctx)}
    peak = max(peaks.values())
    # achieved: algorithmic flops of one fused-kernel launch / its mean
    # CUDA-event duration, measured on the launching stream in the timed region
    flops_launch = kst["flops"] / max(1, kst["launches"])
    achieved = flops_launch / (k_ms * 1e-3) / 1e12
    traffic = None
    prof = os.path.join(ROOT, "profiles", "sketch_traffic.json")
    if os.path.exists(prof):
        pt = json.load(open(prof))
        if pt.get("config") == cfg.name and world == 1:
            traffic = pt["dram_bytes_per_launch"]

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        y_h = st.y.cpu().numpy()
        w_h = st.w.cpu().numpy()
        b = sample_rows(cfg, 1)
        a_rows = a[:, :b].cpu().numpy()
        t, t_sk, t_rf, t_so = cpu_leg(cfg, y_h, w_h, a_rows, 1, 0 if method == Q.PSEUDO_QR else 1)
        cpu = {"value": t, "unit": "s", "cores": 1, "kind": "port",
               "sample": f"serial ordered sketch on leading {b}/{cfg.m} rows, extrapolated "
                         f"({t_sk:.1f} s); rangefinder {t_rf:.2f} s + solve {t_so:.2f} s full size",
               "host": platform_cpu()}

    eight = Q.sketch_kernel_name().startswith("sketch8")
    if rank == 0:
        line = {
            "metric": METRIC, "value": ms / 1e3, "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{cfg.name} {cfg.m}x{cfg.n} fp64 quaternion, s={cfg.s}, l={cfg.l}, "
                                   f"{args.rangefinder}",
                       "parallelism": f"row-shard x{world}",
                       "l2": "A (%.2f GB) larger than the 126 MB L2; no flush needed" % (cfg.a_bytes() / 1e9)},
            "sketch_ms": sk_ms, "sketch_tflops": 32.0 * (r1 - r0) * cfg.n * (cfg.s + cfg.l) / (sk_ms * 1e-3) / 1e12,
            "sketch_kernel": Q.sketch_kernel_name(),
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel_ms_per_launch": k_ms, "launches": kst["launches"],
                         "algorithmic_per_launch": {"flops": flops_launch,
                                                    "a_bytes": kst["a_bytes"] / max(1, kst["launches"])},
                         "peak_source": "FP64 measured in this run (DMMA m8n8k4 / DFMA microbenchmarks; "
                                        "MEASURED_PEAKS.json has no FP64 entry): " + json.dumps(peaks),
                         "note": ("FP64 tensor pipe (DMMA); per-unit = 32 flop per quaternion MAC, "
                                  "a launch covers one row panel of A (<= 2 GB; C2: the whole block): "
                                  "32*rows*n*(s+l) flop" + (
                                      "; the 8-product quaternion algorithm executes 16 of those 32 flop "
                                      "per MAC on the DMMA pipe (+ plane sums on the same pipe), so "
                                      "frac > 1 is the algorithm, executed_frac the pipe" if eight else "")),
                         "executed_tflops": achieved * (0.5 if eight else 1.0),
                         "executed_frac": achieved * (0.5 if eight else 1.0) / peak},
            "rangefinder_used": used["rangefinder"], "rel_error": res / an, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    ctx.close()


def platform_cpu():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        model = [l.split(":", 1)[1].strip() for l in out.splitlines() if l.startswith("Model name")]
        return f"{model[0] if model else '?'}; {os.cpu_count()} logical cpus"
    except Exception:
        return "?"


if __name__ == "__main__":
    main()
