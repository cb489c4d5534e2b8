"""Benchmark: image pairs/s of the B200 generator (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

With --gpus N > 1 and no torchrun environment, bench.py re-launches itself
under `python -m torch.distributed.run --nproc-per-node N` (one rank per GPU,
127.0.0.1 rendezvous, NCCL_DEBUG=INFO); `--dry-run` exercises the launcher and
the rank plumbing on CPU (gloo, no GPU work).

One step = one batch of synthetic PIV image pairs generated on the GPU by the
fused kernel (Philox seeding, bilinear advection, distributed binning, splat,
finalize) -- workload C2 (256x256, B=256 per GPU, Lamb-Oseen vortex flow,
reference defaults: ppp 0.06, d in [0.8, 1.2], I0 = 1, rho = 0). Multi-GPU:
one process per GPU (torchrun), each rank renders B=256 pairs of a global
batch of 256*N (weak scaling), no data-path collective; time = max over ranks.

`value` is device-timed (CUDA events around each step on the launching
stream, L2 flushed between steps), `e2e` goes through the C ABI with HOST
buffers (flow uploaded, images copied back each step). `--impl reference`
times the reference CPU implementation (oracle/_ref = /root/reference/pkg
compiled here) on the host cores with all threads.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "image pairs/sec at 256x256, B=256 on 1/2/4/8 B200; % of HBM/SFU roofline"

# Algorithmic Gaussian evaluations per pair (both frames): the reference's
# clipped patch pixels, SURVEY 8(d) table (probe A.7); the SFU-roofline unit.
# c6 (512^2 plain) has c4's particle law without hiding: ~742,881 as well.
EVALS_PER_PAIR = {"c1": 194567, "c2": 194567, "c3": 35215674, "c4": 742881, "c5": 194567, "c6": 742881}
# nominal MUFU issue, used only when profiles/peaks.json (the
# measured ex2 rate, scripts/measure_peaks.py) is absent
MUFU_PER_CLK_SM = 16

CONFIGS = {
    # name: (H, W, B per GPU, ppp, d_range, flow, extra)
    "c1": (256, 256, 1, (0.06, 0.06), (0.8, 1.2), "uniform", {}),
    "c2": (256, 256, 256, (0.06, 0.06), (0.8, 1.2), "vortex", {}),
    "c3": (1024, 1024, 64, (0.1, 0.1), (1.0, 4.0), "vortex", {}),
    "c4": (512, 512, 256, (0.06, 0.06), (0.8, 1.2), "vortex",
           dict(noise=(0.05, 0.02), hide_probability=0.05,
                laser_sheet=dict(thickness=1.0, shape=2.0, efficiency=1.0, out_of_plane=0.1))),
    "c5": (256, 256, 8192, (0.06, 0.06), (0.8, 1.2), "vortex", {}),
    # the paper's own benchmark size (512^2, B=256, defaults)
    "c6": (512, 512, 256, (0.06, 0.06), (0.8, 1.2), "vortex", {}),
}


def vortex(h, w, scale=2.0):
    """Lamb-Oseen vortex; numpy or torch arrays (device evaluation)."""
    def fn(x, y):
        xp = np
        if type(x).__module__.startswith("torch"):
            import torch as xp
        cx, cy = (w - 1) / 2.0, (h - 1) / 2.0
        rc = 0.1 * w
        dx, dy = x - cx, y - cy
        r = xp.sqrt(dx * dx + dy * dy) + 1e-12
        vt = 1.398 * scale * (rc / r) * (1.0 - xp.exp(-(r / rc) ** 2))
        return -vt * dy / r, vt * dx / r
    return fn


def uniform(x, y):
    return 2.0 + 0.0 * x, -1.0 + 0.0 * y


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def load_probe_peaks():
    """profiles/peaks.json (scripts/measure_peaks.py on a B200): ex2 rate, PCIe."""
    try:
        with open(os.path.join(ROOT, "profiles", "peaks.json")) as fh:
            return json.load(fh)
    except Exception:
        return {}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


class ClockSampler:
    """SM clocks + clock-event (throttle) reasons sampled DURING the timed region:
    NVML polled every ~1 ms on a thread (nvidia-smi -lms 20 as a fallback)."""

    NAMES = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
             0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        self.index = index
        self.sm, self.mx, self.reasons = [], [], set()
        self._stop = threading.Event()
        self._thr = None
        self._smi = None
        self._lines: list[str] = []

    def _handle(self, nv):
        try:
            import torch

            pr = torch.cuda.get_device_properties(self.index)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            return nv.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return nv.nvmlDeviceGetHandleByIndex(self.index)

    def _poll(self, nv, h):
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self._stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                self.mx.append(float(mx))
                bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h) if hasattr(
                    nv, "nvmlDeviceGetCurrentClocksEventReasons") else nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                for bit, name in self.NAMES.items():
                    if bits & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.001)

    def __enter__(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = self._handle(nv)
            self._thr = threading.Thread(target=self._poll, args=(nv, h), daemon=True)
            self._thr.start()
        except Exception:
            try:
                self._smi = subprocess.Popen(
                    ["nvidia-smi", "-i", str(self.index),
                     "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                     "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                     "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "20"],
                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                threading.Thread(target=lambda: self._lines.extend(l.strip() for l in self._smi.stdout),
                                 daemon=True).start()
            except Exception:
                self._smi = None
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thr is not None:
            self._thr.join(2)
        if self._smi is not None:
            self._smi.terminate()
            try:
                self._smi.wait(2)
            except Exception:
                self._smi.kill()
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for line in self._lines:
                parts = [p.strip() for p in line.split(",")]
                try:
                    self.sm.append(float(parts[0]))
                    self.mx.append(float(parts[1]))
                except (ValueError, IndexError):
                    continue
                for name, val in zip(names, parts[2:6]):
                    if val.lower() == "active":
                        self.reasons.add(name)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": max(self.mx),
                "reasons": sorted(self.reasons), "samples": len(self.sm)}


def make_cfg(pg, name, per_gpu_batch):
    H, W, B, ppp, dr, flow, extra = CONFIGS[name]
    kw = dict(image_height=H, image_width=W, batch_size=per_gpu_batch, seeding_density_range=ppp,
              diameter_range=dr, seed=0, flow_sources=(pg.FlowSource(function=f"bench_{flow}"),))
    if "noise" in extra:
        kw["noise"] = pg.NoiseConfig(*extra["noise"])
    if "hide_probability" in extra:
        kw["hide_probability"] = extra["hide_probability"]
    if "laser_sheet" in extra:
        kw["laser_sheet"] = pg.LaserSheetConfig(**extra["laser_sheet"])
    return pg.GeneratorConfig(**kw)


def ref_cfg(name, batch, threads):
    from oracle import reference

    pv = reference.load()
    H, W, B, ppp, dr, flow, extra = CONFIGS[name]
    pv.register_flow_function(f"bench_{flow}", vortex(H, W) if flow == "vortex" else uniform)
    kw = dict(image_height=H, image_width=W, batch_size=batch, seeding_density_range=ppp,
              diameter_range=dr, seed=0, threads=threads,
              flow_sources=(pv.FlowSource(function=f"bench_{flow}"),))
    if "noise" in extra:
        kw["noise"] = pv.NoiseConfig(*extra["noise"])
    if "hide_probability" in extra:
        kw["hide_probability"] = extra["hide_probability"]
        kw["frame2_intensity_std"] = 0.05    # stand-in for the laser sheet (no z in the reference)
    return pv, pv.GeneratorConfig(**kw)


def _ref_rate(name: str, threads: int, budget_s: float, batch: int | None = None):
    pv, cfg = ref_cfg(name, batch or min(CONFIGS[name][2], 256), threads)
    from pivgen.pipeline import Sampler

    pairs = 0
    t_total = 0.0
    with Sampler(cfg) as s:
        s.next_batch()                         # warm-up (thread pool, page-in)
        while t_total < budget_s:
            t0 = time.perf_counter()
            s.next_batch()
            t_total += time.perf_counter() - t0
            pairs += cfg.batch_size
    return pv, cfg, pairs, pairs / t_total


def cpu_baseline(name: str, budget_s: float = 15.0):
    """Reference CPU path (oracle/_ref, native Cython kernel) on the host cores:
    all threads (the reported value) plus a single-thread figure."""
    threads = os.cpu_count() or 1
    pv, cfg, pairs, rate = _ref_rate(name, threads, budget_s)
    _, cfg1, pairs1, rate1 = _ref_rate(name, 1, budget_s / 2, batch=min(cfg.batch_size, 64))
    return {"value": rate, "unit": "pairs/s", "cores": threads, "kind": "reference",
            "cpu_model": cpu_model(),
            "sample": f"{pairs} pairs of {name} ({cfg.image_height}x{cfg.image_width}, "
                      f"B={cfg.batch_size}) via pivgen Sampler.next_batch, threads={threads}, "
                      f"backend={pv.active_backend()}",
            "threads_1": {"value": rate1, "unit": "pairs/s",
                          "sample": f"{pairs1} pairs, B={cfg1.batch_size}, threads=1"}}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    name = args.config
    threads = os.cpu_count() or 1
    pv, cfg = ref_cfg(name, min(CONFIGS[name][2], 256), threads)
    from pivgen.pipeline import Sampler

    times = []
    with Sampler(cfg) as s:
        for _ in range(args.warmup):
            s.next_batch()
        for _ in range(args.steps):
            t0 = time.perf_counter()
            s.next_batch()
            times.append(time.perf_counter() - t0)
    total = sum(times)
    value = cfg.batch_size * len(times) / total
    H, W = cfg.image_height, cfg.image_width
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "pairs/s",
        "cpu_model": cpu_model(),
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * total / len(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64/f32 (CPU)", "data": "synthetic (Lamb-Oseen vortex flow)",
        "config": {"workload": f"{name}: {H}x{W}, B={cfg.batch_size} per step (CPU reference)",
                   "global_batch": cfg.batch_size, "image": [H, W], "parallelism": f"{threads} host threads"},
        "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": threads, "kind": "reference",
                         "sample": f"{args.steps} steps x {cfg.batch_size} pairs, pivgen "
                                   f"{pv.__version__} backend={pv.active_backend()}"},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def sfu_roofline(name, pairs_per_s, clk, world):
    """Secondary roofline (BASELINE.json metric: '% of HBM/SFU roofline'): the
    reference's Gaussian evaluations per pair at the achieved rate against the
    MUFU.EX2 issue rate measured by scripts/measure_peaks.py (per clock per
    SM, scaled to the SM clock sampled during this run); the nominal
    16/clk/SM only when no measurement exists."""
    import torch

    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    summ = clk.summary() if clk is not None else {}
    mhz = summ.get("sm_mhz") or summ.get("sm_max_mhz") or 1965.0
    probe = load_probe_peaks()
    per_clk = probe.get("ex2_per_clk_per_sm")
    if per_clk:
        src = (f"measured ex2.approx {per_clk:.2f}/clk/SM (profiles/peaks.json, {probe.get('when', '?')}) "
               f"x {sms} SMs x {mhz:.0f} MHz (sampled)")
    else:
        per_clk = MUFU_PER_CLK_SM
        src = f"nominal {MUFU_PER_CLK_SM} MUFU/clk/SM x {sms} SMs x {mhz:.0f} MHz (sampled)"
    peak = sms * per_clk * float(mhz) * 1e6 * world / 1e12
    achieved = pairs_per_s * EVALS_PER_PAIR[name] / 1e12
    return {"bound": "sfu", "achieved": achieved, "peak": peak, "unit": "Tevals/s", "frac": achieved / peak,
            "evals_per_pair": EVALS_PER_PAIR[name],
            "peak_source": src,
            "note": "algorithmic evaluations = the reference's clipped patch pixels (SURVEY 8(d)); "
                    "the kernel evaluates fewer (tight windows, separable exponentials)"}


def run_ours(args):
    import torch

    import paper_2512_09664_b200 as pg
    from paper_2512_09664_b200 import _lib
    from paper_2512_09664_b200.particles import native_config

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = torch.cuda.device_count()
    if local >= ndev:
        raise SystemExit(f"bench.py: rank {rank} needs cuda:{local} but only {ndev} device(s) are visible "
                         f"(--gpus {args.gpus})")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    name = args.config
    H, W, Bcfg, *_ = CONFIGS[name]
    per_gpu = Bcfg if name != "c5" else Bcfg // world
    global_batch = per_gpu * world if name != "c5" else Bcfg
    pg.register_flow_function("bench_vortex", vortex(H, W))
    pg.register_flow_function("bench_uniform", uniform)
    cfg = make_cfg(pg, name, global_batch)
    lib = _lib.load()
    ncfg = native_config(cfg)
    kernel_label = ("pgb::band_sorted_kernel (screen-tile items, bank-sorted splat records)" if name == "c3" else
                    "pgb::band_kernel<PSF> (screen-tile items, in-kernel prologue tickets; one launch per batch)")
    field = pg.from_function(vortex(H, W) if CONFIGS[name][5] == "vortex" else uniform, H, W)
    flows = field.to_device(dev).unsqueeze(0).contiguous()
    u16 = False
    img1 = torch.empty((per_gpu, H, W), dtype=torch.float32, device=dev)
    img2 = torch.empty_like(img1)
    stats = {"seeding_density": torch.empty(per_gpu, dtype=torch.float64, device=dev),
             "active_count": torch.empty(per_gpu, dtype=torch.int32, device=dev),
             "side": torch.empty(per_gpu, dtype=torch.int32, device=dev),
             "d_max": torch.empty(per_gpu, dtype=torch.float32, device=dev)}
    st = _lib.PgbPairStats(**{k: v.data_ptr() for k, v in stats.items()})
    pair_base = rank * per_gpu
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step(batch_index):
        _lib.check(lib.pgb_generate_batch_dev(ncfg, batch_index, pair_base, per_gpu, flows.data_ptr(),
                                              1, global_batch, _lib.OUT_U16 if u16 else _lib.OUT_F32,
                                              img1.data_ptr(), img2.data_ptr(), st, None,
                                              stream.cuda_stream))

    for w in range(args.warmup):
        step(w)
    torch.cuda.synchronize()
    lib.pgb_overflow_reset()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches0 = lib.pgb_launch_count()
    with ClockSampler(local) as clk:
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t_wall = time.perf_counter()
        for k in range(args.steps):
            flush.zero_()                          # L2 flush between timed steps (not timed)
            starts[k].record(stream)
            step(args.warmup + k)
            ends[k].record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t_wall = time.perf_counter() - t_wall
    launches = lib.pgb_launch_count() - launches0
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = sum(step_ms)
    rank_ms = [total_ms]
    if dist:
        t = torch.zeros(world, dtype=torch.float64, device=dev)
        t[rank] = total_ms
        dist.all_reduce(t, op=dist.ReduceOp.SUM)      # every rank's device time
        rank_ms = [float(v) for v in t.tolist()]
        total_ms = max(rank_ms)
    ovf = lib.pgb_overflow_count()
    value = global_batch * args.steps / (total_ms / 1000.0)

    # ---- end to end through the C ABI with HOST buffers (rank-local) ----------
    host_flow = torch.from_numpy(field.interleaved()).pin_memory()
    h1 = torch.empty((per_gpu, H, W), dtype=torch.float32).pin_memory()
    h2 = torch.empty_like(h1).pin_memory()
    hst = {"seeding_density": np.empty(per_gpu, np.float64), "active_count": np.empty(per_gpu, np.int32),
           "side": np.empty(per_gpu, np.int32), "d_max": np.empty(per_gpu, np.float32)}
    hs = _lib.PgbPairStats(**{k: v.ctypes.data for k, v in hst.items()})

    def e2e_step(b):
        _lib.check(lib.pgb_generate_batch(ncfg, b, pair_base, per_gpu, host_flow.data_ptr(), 1,
                                          global_batch, _lib.OUT_F32, h1.data_ptr(), h2.data_ptr(), hs))

    e2e_steps = max(2, min(args.steps, 10))
    e2e_step(0)
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for k in range(e2e_steps):
        e2e_step(1 + k)
    e2e_s = time.perf_counter() - t0
    if dist:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = global_batch * e2e_steps / e2e_s
    h2d = host_flow.numel() * 4
    d2h = 2 * per_gpu * H * W * 4 + per_gpu * (8 + 4 + 4 + 4)

    if rank == 0:
        peak, peak_kind = load_peaks()
        bytes_per_launch = 2 * per_gpu * H * W * 4
        kernel_s = (total_ms / 1000.0) / args.steps
        achieved = bytes_per_launch / kernel_s / 1e9
        traffic, traffic_src = None, None
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            try:
                with open(tp) as fh:
                    tj = json.load(fh).get(name)
                if tj:
                    # dram__bytes_read.sum + dram__bytes_write.sum of one ncu --set full
                    # capture (L2 is write-back: part of the output leaves later)
                    traffic = float(tj["dram_bytes_per_launch"])
                    traffic_src = "profiles/" + tj.get("source", "traffic.json")
            except Exception:
                traffic = None
        line = {
            "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (Lamb-Oseen vortex flow; Philox-seeded particles)",
            "config": {"workload": f"{name}: {H}x{W}, B={per_gpu} pairs per GPU, ppp {CONFIGS[name][3][1]}, "
                                   f"d in [{CONFIGS[name][4][0]},{CONFIGS[name][4][1]}], {CONFIGS[name][5]} flow"
                                   + (", " + ",".join(sorted(CONFIGS[name][6])) if CONFIGS[name][6] else ""),
                       "global_batch": global_batch, "seq_len": None, "image": [H, W],
                       "parallelism": f"dp{world} (pairs sharded, no collective)",
                       "l2": "flushed between steps (256 MiB write, untimed); per-step CUDA events summed",
                       "output": "float32 images1+images2 in HBM"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "algorithmic_bytes_per_launch": bytes_per_launch,
                         "kernel": kernel_label,
                         "peak_source": peak_kind + " (MEASURED_PEAKS.json hbm_gbs, copy burst)"},
            "roofline_sfu": sfu_roofline(name, value, clk, world),
            "e2e": e2e_line(e2e_value, h2d, d2h, global_batch, world),
            "gpu_launches": int(launches),
            "rank_ms_total": rank_ms,
            "clocks": clk.summary(),
            "wall_s_timed_region": t_wall,
            "overflow_events": int(ovf),
        }
        if world == 1 and not args.no_cpu_baseline:
            try:
                line["cpu_baseline"] = cpu_baseline(name if name != "c5" else "c2")
            except Exception as exc:  # pragma: no cover - reference missing on the box
                line["cpu_baseline"] = {"value": None, "unavailable": str(exc)}
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def e2e_line(value, h2d, d2h, global_batch, world):
    """End-to-end record; with a measured PCIe D2H bandwidth (profiles/peaks.json)
    also the link bound: the images must cross PCIe (per GPU)."""
    out = {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "path": "pgb_generate_batch (C ABI, host buffers: flow H2D + images D2H, pinned)"}
    probe = load_probe_peaks()
    if probe.get("pcie_d2h_gbs"):
        per_gpu_pairs = global_batch / world
        bound = probe["pcie_d2h_gbs"] * 1e9 / (d2h / per_gpu_pairs) * world
        out["link_bound"] = {"value": bound, "unit": "pairs/s", "frac": value / bound,
                             "pcie_d2h_gbs": probe["pcie_d2h_gbs"], "source": "profiles/peaks.json"}
    return out


def spawn_ranks(args) -> int:
    """--gpus N > 1 outside torchrun: re-launch this script with one rank per
    GPU (python -m torch.distributed.run, 127.0.0.1 rendezvous)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")     # NCCL reports nranks in the log
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def run_dry(args):
    """Launcher check without a GPU: gloo ranks, shard bookkeeping, max-over-ranks."""
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    from paper_2512_09664_b200.pipeline import shard_pairs

    name = args.config
    H, W, Bcfg, *_ = CONFIGS[name]
    per_gpu = Bcfg if name != "c5" else Bcfg // world
    global_batch = per_gpu * world if name != "c5" else Bcfg
    shard = shard_pairs(global_batch, rank, world)
    t = torch.zeros(world, dtype=torch.float64)
    t[rank] = float(len(shard))
    if world > 1:
        dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"dry_run": True, "metric": METRIC, "n_gpus": world, "global_batch": global_batch,
                          "pairs_per_rank": [int(v) for v in t.tolist()], "config": name}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--dry-run", action="store_true", help="CPU launcher check (no GPU work)")
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
