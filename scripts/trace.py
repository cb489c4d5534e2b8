"""Per-CTA timeline of one band-kernel launch (debug build with -DPGB_TRACE).

  bash scripts/build_variant.sh trace -DPGB_TRACE
  PGB_LIBRARY=build/trace.so PGB_LIB_LENIENT=1 python scripts/trace.py [config] [B]

Events (globaltimer ns, relative to the earliest kernel-entry stamp):
 0 entry, 1 first ticket, 2-7 pair prologue (start, histogram, chunk sums,
 prefix+marks, max-scan, released), 8 prologue loop done, 9 first item staged,
 10 first item particles done, 11 first item stored, 12 exit, 13 items,
34-38 histogram part / cell window events (last one per CTA).
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2512_09664_b200 as pg  # noqa: E402
from paper_2512_09664_b200 import _lib  # noqa: E402
from paper_2512_09664_b200.particles import native_config  # noqa: E402

SLOTS = 40
NAMES = ["entry", "field_chunk_done", "pro_start", "pro_hist", "pro_sums", "pro_prefix", "pro_maxscan",
         "pro_released", "pro_loop_done", "item1_staged", "stage_polled", "stage_loaded", "exit", "(items)", "pro_f64_chain",
         "stage_finished"]
EXTRA = {34: "part_start", 35: "part_labels", 36: "part_published", 37: "window_go", 38: "window_done"}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    B = int(sys.argv[2]) if len(sys.argv) > 2 else bench.CONFIGS[name][2]
    H, W, _, _, _, flow, _ = bench.CONFIGS[name]
    pg.register_flow_function("bench_vortex", bench.vortex(H, W))
    pg.register_flow_function("bench_uniform", bench.uniform)
    field = pg.from_function(bench.vortex(H, W) if flow == "vortex" else bench.uniform, H, W)
    flows = field.to_device().unsqueeze(0).contiguous()
    lib = _lib.load(require_symbols=False)
    lib.pgb_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
    cfg = bench.make_cfg(pg, name, B)
    ncfg = native_config(cfg)
    img1 = torch.empty((B, H, W), dtype=torch.float32, device="cuda")
    img2 = torch.empty_like(img1)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()

    def step(k):
        _lib.check(lib.pgb_generate_batch_dev(ncfg, k, 0, B, flows.data_ptr(), 1, B, _lib.OUT_F32,
                                              img1.data_ptr(), img2.data_ptr(), None, None,
                                              stream.cuda_stream))
    for k in range(5):
        step(k)
    torch.cuda.synchronize()
    if os.environ.get("TRACE_NOFLUSH"):
        step(8)   # the previous launch leaves code, flow and tables in L2
        torch.cuda.synchronize()
    else:
        flush.zero_()
        if os.environ.get("TRACE_CODEWARM"):
            # one single-pair launch after the flush: kernel code back in L2
            _lib.check(lib.pgb_generate_batch_dev(ncfg, 7, 0, 1, flows.data_ptr(), 1, B, _lib.OUT_F32,
                                                  img1.data_ptr(), img2.data_ptr(), None, None,
                                                  stream.cuda_stream))
            torch.cuda.synchronize()
        if os.environ.get("TRACE_IDLE"):
            # idle gap after the flush (no launch): does the L2 drain its dirty lines?
            torch.cuda._sleep(int(os.environ["TRACE_IDLE"]))
            torch.cuda.synchronize()
    lib.pgb_trace_clear()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    step(9)
    e1.record()
    torch.cuda.synchronize()
    buf = np.zeros(2048 * SLOTS, dtype=np.uint64)
    lib.pgb_trace_read(buf.ctypes.data, buf.size)
    t = buf.reshape(2048, SLOTS).astype(np.int64)
    used = t[:, 0] > 0
    t = t[used]
    t0 = t[:, 0].min()
    print(f"{name} B={B}: kernel {e0.elapsed_time(e1) * 1e3:.1f} us (events), {used.sum()} CTAs traced")
    for ev, nm in enumerate(NAMES):
        if ev == 13:
            continue
        col = t[:, ev]
        ok = col > 0
        if not ok.any():
            continue
        r = (col[ok] - t0) / 1e3
        print(f"  {ev:2d} {nm:16s} n={ok.sum():4d}  min {r.min():7.2f}  med {np.median(r):7.2f}  "
              f"max {r.max():7.2f} us")
    for ev, nm in EXTRA.items():
        col = t[:, ev]
        ok = col > 0
        if ok.any():
            r = (col[ok] - t0) / 1e3
            print(f"  {ev:2d} {nm:16s} n={ok.sum():4d}  min {r.min():7.2f}  med {np.median(r):7.2f}  "
                  f"max {r.max():7.2f} us")
    items = t[:, 13]
    print(f"  items per CTA: min {items.min()} med {np.median(items)} max {items.max()}")
    # per-item phases (worker thread 0): own particles done, all particles
    # done (barrier), store done
    for k in range(6):
        c = t[:, 16 + 3 * k:19 + 3 * k]
        ok = c[:, 2] > 0
        if not ok.any():
            break
        c = (c[ok] - t0) / 1e3
        print(f"  item {k}: n={ok.sum():4d}  splat_end med {np.median(c[:, 0]):6.2f}  barrier med "
              f"{np.median(c[:, 1]):6.2f}  store_end med {np.median(c[:, 2]):6.2f} (min {c[:, 2].min():6.2f} max "
              f"{c[:, 2].max():6.2f})  bar-wait med {np.median(c[:, 1] - c[:, 0]):5.2f}  store med "
              f"{np.median(c[:, 2] - c[:, 1]):5.2f} us")
    # SM co-residents (slot 39 = smid + 1): how much of a CTA's store phases
    # overlap its neighbour's store phases
    sm = t[:, 39] - 1
    ov, tot = 0.0, 0.0
    for s_ in np.unique(sm):
        idx = np.where(sm == s_)[0]
        if len(idx) != 2:
            continue
        ph = []
        for i in idx:
            iv = []
            for k in range(6):
                a, b = t[i, 17 + 3 * k], t[i, 18 + 3 * k]
                if b > 0:
                    iv.append((a, b))
            ph.append(iv)
        for a, b in ph[0]:
            tot += b - a
            for c, d in ph[1]:
                ov += max(0, min(b, d) - max(a, c))
    if tot > 0:
        print(f"  store phases of SM co-residents overlapping: {100 * ov / tot:.0f} %")
    pro = (t[:, 2] > 0) & (t[:, 7] > 0)
    if pro.any():
        d = (t[pro][:, 3:8] - t[pro][:, 2:7]) / 1e3
        print("  prologue stage durations (median us): hist %.2f sums %.2f prefix %.2f maxscan %.2f release %.2f"
              % tuple(np.median(d, axis=0)))


if __name__ == "__main__":
    main()
