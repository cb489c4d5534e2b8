"""Measure the roofline denominators MEASURED_PEAKS.json does not carry and
write them to profiles/peaks.json (run on the GPU box):

  * MUFU.EX2 issue rate (pgb_probe_ex2_dev: 8 independent ex2.approx chains
    per thread, grid = 148 SMs x 8 CTAs x 256 threads), CUDA-event timed, with
    the SM clock sampled by NVML during the run -> ex2/s and ex2/clk/SM;
  * PCIe host<->device copy bandwidth (pinned, 256 MiB, best of 5): the
    ceiling of bench.py's end-to-end number (images leave over PCIe).

    python scripts/measure_peaks.py [--out profiles/peaks.json]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "peaks.json"))
    args = ap.parse_args()
    import torch

    from bench import ClockSampler
    from paper_2512_09664_b200 import _lib

    lib = _lib.load()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    sink = torch.zeros(256, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    blocks, iters = sms * 8, 4096

    def launch():
        _lib.check(lib.pgb_probe_ex2_dev(blocks, iters, sink.data_ptr(), stream.cuda_stream))

    for _ in range(3):
        launch()
    torch.cuda.synchronize()
    times = []
    with ClockSampler(0) as clk:
        for _ in range(20):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            launch()
            b.record(stream)
            b.synchronize()
            times.append(a.elapsed_time(b) / 1e3)
    t = min(times)
    n_ex2 = blocks * 256 * 8 * iters
    summ = clk.summary()
    mhz = summ.get("sm_mhz") or summ.get("sm_max_mhz") or 1965.0
    ex2_s = n_ex2 / t
    per_clk_sm = ex2_s / (sms * mhz * 1e6)

    # PCIe copy bandwidth (pinned host memory)
    nbytes = 256 << 20
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    bw = {}
    for name, (dst, src) in {"d2h": (h, d), "h2d": (d, h)}.items():
        best = 0.0
        for _ in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dst.copy_(src, non_blocking=True)
            torch.cuda.synchronize()
            best = max(best, nbytes / (time.perf_counter() - t0) / 1e9)
        bw[name] = best
    out = {
        "ex2_per_s": ex2_s, "ex2_tera_per_s": ex2_s / 1e12, "ex2_per_clk_per_sm": per_clk_sm,
        "ex2_probe": f"{blocks} CTAs x 256 threads x 8 chains x {iters} iters, best of 20 (CUDA events)",
        "sm_mhz_during_probe": mhz, "clock_reasons": summ.get("reasons"), "sms": sms,
        "pcie_d2h_gbs": bw["d2h"], "pcie_h2d_gbs": bw["h2d"],
        "pcie_probe": "256 MiB pinned copy, best of 5 (wall clock around copy + sync)",
        "gpu": torch.cuda.get_device_name(dev),
        "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
        "median_probe_s": statistics.median(times),
    }
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(out, fh, indent=1)
        fh.write("\n")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
